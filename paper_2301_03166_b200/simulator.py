"""Protected iteration on the B200 — drop-in for the hot-path part of
slackwise.simulator (/root/reference/pkg/src/slackwise/simulator.py):
_tmu_region :86-94, run_numeric_iteration :97-121 (with _protected_tmu
:124-167 executed inside libabft_b200.so).

``run_protected`` is the whole-factorization fast path (one C-ABI call, no
per-iteration host synchronisation unless a report is non-empty): the fault
plans are pre-drawn on the host in exactly the order run_numeric_iteration
would draw them, because the draws do not depend on the data.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .abft import (ChecksumScheme, CorrectionReport, ErrorKind, TYPES, _fault_struct,
                   build_report, draw_plan)
from .linalg import DecompositionKind, Factorization, _value, check

CORRECTNESS_RESIDUAL = 1.0e-8   # simulator.py:33


def _tmu_region(kind, n: int, b: int, k: int):
    """(r0, c0, rows, cols) of the block the trailing update writes."""
    p = k * b
    pe = min(p + b, n)
    kd = _value(kind)
    if kd == "cholesky":
        return p, p, n - p, pe - p
    if kd == "lu":
        return pe, pe, n - pe, n - pe
    return p, pe, n - p, n - pe


def _plan_structs(plan: list):
    arr = (_lib.Fault * max(1, len(plan)))()
    for i, d in enumerate(plan):
        arr[i] = _fault_struct(d, False, d["u"], d["negate"])
    return arr


def run_numeric_iteration(factors: Factorization, k: int, scheme,
                          fault_counts: dict | None = None,
                          rng: np.random.Generator | None = None,
                          correct: bool = True) -> CorrectionReport:
    """simulator.py:97-121: PD/PU + checksum-protected TMU of iteration k with
    the planned faults injected between maintenance and verification."""
    if not isinstance(factors, Factorization):
        raise TypeError("run_numeric_iteration needs a B200 Factorization")
    sch = ChecksumScheme(_value(scheme))
    n, b = factors.n, factors.b
    r0, c0, rows, cols = _tmu_region(factors.kind, n, b, k)
    plan = []
    if rows > 0 and cols > 0 and fault_counts and any(fault_counts.values()):
        plan = draw_plan(rng, fault_counts, r0, c0, rows, cols, b)
    arr = _plan_structs(plan)
    rep = _lib.Report()
    cap = 4096
    locs = (_lib.Location * cap)()
    factors._dirty()
    check(factors._lib.abft_iteration(factors._ctx, int(k), _lib.SCHEME_CODE[sch.value], arr,
                                      len(plan), int(bool(correct)), ctypes.byref(rep), locs, cap))
    if rep.n_locations > cap:
        raise RuntimeError("more ABFT events than the location buffer holds")
    return build_report(rep, locs, cap)


def run_protected(factors: Factorization, scheme, fault_schedule: dict | None = None,
                  rng: np.random.Generator | None = None, correct: bool = True,
                  schemes: list | None = None, out: np.ndarray | None = None) -> list:
    """All remaining iterations in one device call (``out``: stream the
    finished factor into this host array during the call).

    ``fault_schedule``: {k: counts} — equivalent to calling
    run_numeric_iteration(factors, k, scheme, fault_schedule.get(k), rng) for
    every k in order (same rng draws). Returns one CorrectionReport per
    iteration executed.
    """
    n, b, nb = factors.n, factors.b, factors.layout.n_blocks
    k0 = factors.k_done
    flat, iters = [], []
    for k in range(k0, nb):
        counts = (fault_schedule or {}).get(k)
        r0, c0, rows, cols = _tmu_region(factors.kind, n, b, k)
        if rows > 0 and cols > 0 and counts and any(counts.values()):
            for d in draw_plan(rng, counts, r0, c0, rows, cols, b):
                flat.append(d)
                iters.append(k)
    arr = _plan_structs(flat)
    it = (ctypes.c_int64 * max(1, len(iters)))(*iters)
    sch = ChecksumScheme(_value(scheme))
    sarr = None
    if schemes is not None:
        sarr = (ctypes.c_int32 * nb)(*[_lib.SCHEME_CODE[_value(s)] for s in schemes])
    reports = (_lib.Report * nb)()
    cap = 1 << 16
    locs = (_lib.Location * cap)()
    nloc = ctypes.c_int(0)
    factors._dirty()
    if out is not None:
        # the finished factor streams into `out` (n x n, Fortran order; pinned
        # memory overlaps the copies with the factorization)
        if out.shape != (n, n) or out.dtype != np.float64 or not out.flags.f_contiguous:
            raise ValueError("out must be an n x n float64 Fortran-ordered array")
        check(factors._lib.abft_stream_out(factors._ctx, _lib.dptr(out), n))
    try:
        check(factors._lib.abft_factorize(factors._ctx, _lib.SCHEME_CODE[sch.value], sarr, arr, it,
                                          len(flat), int(bool(correct)), reports, locs, cap,
                                          ctypes.byref(nloc)))
    finally:
        if out is not None:
            factors._lib.abft_stream_out(factors._ctx, None, 0)
        factors._streamed_in = None  # the streamed input was consumed by this call
    out, pos = [], 0
    for k in range(k0, nb):
        r = reports[k]
        sub = (_lib.Location * max(1, r.n_locations))()
        for i in range(r.n_locations):
            sub[i] = locs[pos + i]
        pos += r.n_locations
        out.append(build_report(r, sub, r.n_locations))
    return out
