"""Run the reference's OWN test suite with the B200 backend installed.

The drop-in proof of SURVEY.md §7 step 2 / §8b: `install()` rebinds the
reference package's hot-path names (Factorization, run_numeric_iteration,
residual, encode / maintain_gemm / verify_correct / inject_faults,
_Run._snapshot / _restore) to this repository's B200 implementations, then
the reference's unmodified tests run against them.

The reference is installed (not committed) into baseline/_ref:
    python -m pip install --no-index --no-build-isolation --no-deps \\
        --find-links /opt/wheelhouse --target baseline/_ref <copy of /root/reference/pkg>
    mkdir -p baseline/_ref/_tests && cp /root/reference/pkg/tests/*.py baseline/_ref/_tests/
baseline/_ref is git-ignored but travels to the GPU box with the snapshot.

usage: python tools/reference_suite.py [pytest args...]
Prints the pytest summary and, on the last line, one JSON object with the
exit code and the number of B200 kernel launches the suite made (a suite
that never reached the GPU would report 0).
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"


def main(argv: list[str]) -> int:
    if not (REF / "slackwise").is_dir() or not (REF / "_tests").is_dir():
        print(json.dumps({"reference_suite": "unavailable",
                          "why": "baseline/_ref (installed reference + its tests) missing"}))
        return 0
    sys.path.insert(0, str(REF))
    sys.path.insert(0, str(ROOT))
    import pytest

    import paper_2301_03166_b200 as P
    import slackwise
    lib = P._lib.load()
    assert P.install("slackwise"), "install() could not import slackwise"
    # the patched names really are the B200 ones
    assert slackwise.Factorization is P.Factorization
    assert slackwise.simulator.run_numeric_iteration is P.run_numeric_iteration
    assert slackwise.abft.verify_correct is P.verify_correct
    ini = REF / "_tests" / "pytest.ini"  # keep this repo's pytest.ini out of the run
    if not ini.exists():
        ini.write_text("[pytest]\n")
    before = lib.abft_launch_count()
    rc = pytest.main([str(REF / "_tests"), "-q", "-p", "no:cacheprovider", "-c", str(ini),
                      "--rootdir", str(REF / "_tests"), *argv])
    launches = lib.abft_launch_count() - before
    print(json.dumps({"reference_suite": "ran", "exit_code": int(rc),
                      "b200_kernel_launches": int(launches)}))
    return int(rc)


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
