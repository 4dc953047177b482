"""Single-precision factorizations (the s* variants of the north star:
sgetrf, spotrf, sgeqrf) on the B200.

Same Python surface and semantics as the fp64 drop-in (Factorization,
run_numeric_iteration, run_protected, residual; linalg.py:159-368,
simulator.py:97-167): the working matrix is fp32 and the trailing updates /
panel solves run on the tcgen05 tensor cores (kind::tf32, 3xTF32 split for
fp32 accuracy, csrc/sgemm_tc05.cu); block checksums stay fp64 and the
verification threshold is the reference's with eps32. The reference itself
is fp64-only (linalg.py:180, abft.py:163), so fp32 parity is unpinned
(SURVEY.md §8c); the tests compare fault outcomes with the fp64 oracle.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .abft import ChecksumScheme, build_report, draw_plan
from .linalg import BlockLayout, DecompositionKind, ERRORS, _value, check
from .simulator import _plan_structs, _tmu_region


class SFactorization:
    """fp32 Factorization (LU = sgetrf without pivoting, Cholesky = spotrf,
    left-looking as the reference, QR = sgeqrf compact-WY with the
    Householder panel factored in fp64 from the widened fp32 panel)."""

    def __init__(self, kind, a0: np.ndarray, b: int, device: int | None = None,
                 keep_input: bool = False, spd_on_device: bool = False):
        self.kind = DecompositionKind(_value(kind))
        n = a0.shape[0]
        if a0.ndim != 2 or a0.shape != (n, n):
            raise ERRORS["dim"]("square input required")
        self.n, self.b = n, int(b)
        self.layout = BlockLayout(n, self.b)
        self.device = 0 if device is None else int(device)
        lib = _lib.load()
        ctx = ctypes.c_void_p()
        check(lib.abft_s_create(ctypes.byref(ctx), _lib.KIND_CODE[self.kind.value], n, self.b,
                                self.device))
        self._ctx, self._lib = ctx, lib
        if keep_input:
            check(lib.abft_s_keep_input(ctx, 1))
        self.set_matrix(a0)
        if spd_on_device:  # a <- a a^T + n I on the tensor cores (linalg.py:74-75)
            check(lib.abft_s_make_spd(ctx))

    def __del__(self):
        ctx = getattr(self, "_ctx", None)
        if ctx:
            try:
                self._lib.abft_s_destroy(ctx)
            except Exception:
                pass
            self._ctx = None

    def set_matrix(self, a: np.ndarray) -> None:
        host = np.asfortranarray(np.asarray(a, dtype=np.float32))
        check(self._lib.abft_s_set_matrix(self._ctx, _lib.fptr(host), self.n))

    def stream_input(self, a: np.ndarray) -> None:
        """abft_s_set_matrix_streamed: the host matrix (n x n float32, Fortran
        order; pinned for asynchronous copies) moves to the device block column
        by block column inside the next run_protected call, overlapped with
        the factorization. The array is held until that call returns."""
        if a.shape != (self.n, self.n) or a.dtype != np.float32 or not a.flags.f_contiguous:
            raise ValueError("a must be an n x n float32 Fortran-ordered array")
        check(self._lib.abft_s_set_matrix_streamed(self._ctx, _lib.fptr(a), self.n))
        self._streamed_in = a

    def set_input_chunks(self, chunk: int = -1, split: int = -1, right_chunk: int = -1) -> None:
        """abft_s_set_input_chunks (-1: built-in; chunk 0: wait for all input)."""
        check(self._lib.abft_s_set_input_chunks(self._ctx, int(chunk), int(split), int(right_chunk)))

    def reset(self) -> None:
        check(self._lib.abft_s_reset(self._ctx))

    @property
    def k_done(self) -> int:
        return int(self._lib.abft_s_k_done(self._ctx))

    @property
    def complete(self) -> bool:
        return self.k_done >= self.layout.n_blocks

    @property
    def m(self) -> np.ndarray:
        out = np.empty((self.n, self.n), dtype=np.float32, order="F")
        check(self._lib.abft_s_get_matrix(self._ctx, _lib.fptr(out), self.n))
        return out

    def snapshot(self, slot: int = 0) -> None:
        """Device snapshot (one slot) for the recompute recovery policy."""
        check(self._lib.abft_s_snapshot(self._ctx))

    def restore(self, slot: int = 0) -> None:
        check(self._lib.abft_s_restore(self._ctx))

    def stream_ptr(self) -> int:
        return int(self._lib.abft_s_stream(self._ctx))

    def run_numeric_iteration(self, k: int, scheme, fault_counts: dict | None = None,
                              rng: np.random.Generator | None = None, correct: bool = True):
        """simulator.py:97-121 in fp32."""
        sch = ChecksumScheme(_value(scheme))
        r0, c0, rows, cols = _tmu_region(self.kind, self.n, self.b, k)
        plan = []
        if rows > 0 and cols > 0 and fault_counts and any(fault_counts.values()):
            plan = draw_plan(rng, fault_counts, r0, c0, rows, cols, self.b)
        arr = _plan_structs(plan)
        rep = _lib.Report()
        cap = 4096
        locs = (_lib.Location * cap)()
        check(self._lib.abft_s_iteration(self._ctx, int(k), _lib.SCHEME_CODE[sch.value], arr,
                                         len(plan), int(bool(correct)), ctypes.byref(rep), locs, cap))
        return build_report(rep, locs, cap)

    def run_protected(self, scheme, fault_schedule: dict | None = None,
                      rng: np.random.Generator | None = None, correct: bool = True,
                      schemes: list | None = None, out: np.ndarray | None = None) -> list:
        """All remaining iterations in one device call (run_protected);
        ``out`` (n x n float32, Fortran order) receives the finished factor,
        streamed column block by column block during the call."""
        nb, k0 = self.layout.n_blocks, self.k_done
        flat, iters = [], []
        for k in range(k0, nb):
            counts = (fault_schedule or {}).get(k)
            r0, c0, rows, cols = _tmu_region(self.kind, self.n, self.b, k)
            if rows > 0 and cols > 0 and counts and any(counts.values()):
                for d in draw_plan(rng, counts, r0, c0, rows, cols, self.b):
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
        if out is not None:
            if out.shape != (self.n, self.n) or out.dtype != np.float32 or not out.flags.f_contiguous:
                raise ValueError("out must be an n x n float32 Fortran-ordered array")
            check(self._lib.abft_s_stream_out(self._ctx, _lib.fptr(out), self.n))
        try:
            check(self._lib.abft_s_factorize(self._ctx, _lib.SCHEME_CODE[sch.value], sarr, arr, it,
                                             len(flat), int(bool(correct)), reports, locs, cap,
                                             ctypes.byref(nloc)))
        finally:
            if out is not None:
                self._lib.abft_s_stream_out(self._ctx, None, 0)
            self._streamed_in = None  # the streamed input was consumed by this call
        out, pos = [], 0
        for k in range(k0, nb):
            r = reports[k]
            sub = (_lib.Location * max(1, r.n_locations))()
            for i in range(r.n_locations):
                sub[i] = locs[pos + i]
            pos += r.n_locations
            out.append(build_report(r, sub, r.n_locations))
        return out

    def elapsed_ms(self) -> float:
        v = ctypes.c_double(0.0)
        check(self._lib.abft_s_last_elapsed_ms(self._ctx, ctypes.byref(v)))
        return float(v.value)

    def residual(self, a: np.ndarray | None = None) -> float:
        """residual(a, factors) (linalg.py:362-368); a=None uses the kept input."""
        out = ctypes.c_double(0.0)
        if a is None:
            check(self._lib.abft_s_residual(self._ctx, None, self.n, ctypes.byref(out)))
        else:
            host = np.asfortranarray(np.asarray(a, dtype=np.float32))
            check(self._lib.abft_s_residual(self._ctx, _lib.fptr(host), self.n, ctypes.byref(out)))
        return float(out.value)
