import json
import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a library)")
    config.addinivalue_line("markers", "slow: long-running")


def golden(name: str):
    return json.loads((GOLDEN / name).read_text())


@pytest.fixture(scope="session")
def gpu_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    # GPU tests fail loudly (not skip) when selected without a GPU, so a
    # missing device or library can never pass silently.
    pass


def report_json(rep) -> dict:
    """Product/oracle CorrectionReport -> the golden JSON shape."""
    val = lambda k: getattr(k, "value", k)  # noqa: E731
    return {"detected": {val(k): int(v) for k, v in rep.detected.items()},
            "corrected": {val(k): int(v) for k, v in rep.corrected.items()},
            "uncorrectable": bool(rep.uncorrectable),
            "locations": [[int(a), int(b), val(c), bool(d)] for a, b, c, d in rep.locations]}


def sparse_reports(reps: list) -> list:
    return [[k, r] for k, r in enumerate(reps)
            if r["locations"] or r["uncorrectable"] or any(r["detected"].values())]
