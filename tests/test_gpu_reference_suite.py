"""GPU: the reference's own test suite (pkg/tests, all 137 tests) passes with
the B200 backend installed into the reference package (SURVEY.md §7 step 2,
§8b drop-in boundary). Needs the reference installed into baseline/_ref (see
tools/reference_suite.py); skipped where it was not installed."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not (REF / "_tests").is_dir(), reason="reference not installed in baseline/_ref")
def test_reference_suite_passes_with_b200_backend_installed():
    out = subprocess.run([sys.executable, str(ROOT / "tools" / "reference_suite.py")],
                         capture_output=True, text=True, timeout=1800, cwd=str(ROOT))
    last = out.stdout.strip().splitlines()[-1]
    info = json.loads(last)
    assert info["exit_code"] == 0, out.stdout[-4000:] + out.stderr[-2000:]
    # the hot path really ran on the GPU
    assert info["b200_kernel_launches"] > 1000, info
