"""Rebind the reference package's hot-path names to the B200 backend.

The reference resolves these names at call time through module globals
(SURVEY.md §8b): simulator.py:24-26 binds Factorization / generate_test_matrix
/ residual; _Run._numeric_step looks up run_numeric_iteration (:416);
_Run._snapshot/_restore copy the host matrix (:420-436); package re-exports
live in __init__.py:5-27. ``install()`` patches all of them so
``simulate_run(engine="numeric")``, ``fault_campaign`` and the module-level
ABFT functions execute on the B200; ``uninstall()`` restores the originals.
"""
from __future__ import annotations

import importlib
import sys

from . import abft as _abft
from . import linalg as _linalg
from . import simulator as _sim

_saved: list = []


def _patch(mod, name, value):
    if hasattr(mod, name):
        _saved.append((mod, name, getattr(mod, name)))
        setattr(mod, name, value)


def _snapshot(run):
    if not run.numeric:
        return None
    f = run.factors
    f.snapshot(0)
    return ("b200", f.k_done, len(f.qr_t))


def _restore(run, snap):
    f = run.factors
    if snap and snap[0] == "b200":
        f.restore(0)
        f.k_done = snap[1]
        f._set_qr_count(min(snap[2], len(f.qr_t)))


def install(package: str = "slackwise") -> bool:
    """Patch ``package`` (default: the reference, ``slackwise``). Returns
    False when the package is not importable (e.g. on a box without it)."""
    try:
        pkg = importlib.import_module(package)
    except ImportError:
        return False
    mods = {name: sys.modules.get(f"{package}.{name}") or importlib.import_module(f"{package}.{name}")
            for name in ("linalg", "abft", "simulator")}
    # the reference's own exception / enum / report classes
    _linalg.ERRORS["dim"] = mods["linalg"].InvalidDimensionError
    _linalg.ERRORS["breakdown"] = mods["linalg"].NumericBreakdownError
    _abft.TYPES["report"] = mods["abft"].CorrectionReport
    _abft.TYPES["error_kind"] = mods["abft"].ErrorKind
    names = {
        "Factorization": _linalg.Factorization,
        "residual": _linalg.residual,
        "run_numeric_iteration": _sim.run_numeric_iteration,
        "encode": _abft.encode,
        "maintain_gemm": _abft.maintain_gemm,
        "verify_correct": _abft.verify_correct,
        "inject_faults": _abft.inject_faults,
    }
    for mod in (pkg, *mods.values()):
        for name, value in names.items():
            _patch(mod, name, value)
    run_cls = getattr(mods["simulator"], "_Run", None)
    if run_cls is not None:
        _patch(run_cls, "_snapshot", _snapshot)
        _patch(run_cls, "_restore", _restore)
    return True


def uninstall() -> None:
    while _saved:
        mod, name, value = _saved.pop()
        setattr(mod, name, value)
    _linalg.ERRORS["dim"] = _linalg.InvalidDimensionError
    _linalg.ERRORS["breakdown"] = _linalg.NumericBreakdownError
    _abft.TYPES["report"] = _abft.CorrectionReport
    _abft.TYPES["error_kind"] = _abft.ErrorKind
