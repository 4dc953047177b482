"""B200-backed blocked factorizations — drop-in for slackwise.linalg's hot path.

Mirrors the reference names and semantics
(/root/reference/pkg/src/slackwise/linalg.py):
  DecompositionKind :24, TaskKind :30, InvalidDimensionError :37,
  NumericBreakdownError :41, BlockLayout :46, generate_test_matrix :63,
  compute_flops :85, Factorization :159-359, residual :362.
The working matrix lives in HBM inside a C-ABI context (libabft_b200.so);
``Factorization.m`` is a lazily synchronised host mirror, as the reference's
tests read ``factors.m`` directly (pkg/tests/test_linalg.py:45-50).
"""
from __future__ import annotations

import ctypes
import enum
import math
from dataclasses import dataclass

import numpy as np

from . import _lib


class DecompositionKind(str, enum.Enum):
    CHOLESKY = "cholesky"
    LU = "lu"
    QR = "qr"


class TaskKind(str, enum.Enum):
    PD = "pd"
    PU = "pu"
    TMU = "tmu"
    TRANSFER = "transfer"


class InvalidDimensionError(ValueError):
    pass


class NumericBreakdownError(ArithmeticError):
    """Non-positive / zero / non-finite pivot (linalg.py:41-43)."""


# Exception classes raised for library error codes; ``install()`` rebinds
# these to the reference package's own classes so its tests catch them.
ERRORS = {"dim": InvalidDimensionError, "breakdown": NumericBreakdownError}


def _value(x) -> str:
    return getattr(x, "value", x)


def check(rc: int) -> None:
    """Map a C-ABI return code onto the reference's exception types."""
    if rc == _lib.OK:
        return
    msg = _lib.last_error()
    if rc == _lib.E_DIM:
        raise ERRORS["dim"](msg)
    if rc in (_lib.E_BREAKDOWN, _lib.E_INCOMPLETE):
        raise ERRORS["breakdown"](msg)
    if rc == _lib.E_RANGE:
        raise IndexError(msg)
    if rc == _lib.E_INVALID:
        raise ValueError(msg)
    raise RuntimeError(f"libabft_b200 error {rc}: {msg}")


@dataclass(frozen=True)
class BlockLayout:
    """linalg.py:46-60."""
    n: int
    b: int

    def __post_init__(self):
        if not (1 <= self.b <= self.n):
            raise ERRORS["dim"](f"block size {self.b} outside [1, {self.n}]")

    @property
    def n_blocks(self) -> int:
        return math.ceil(self.n / self.b)

    def block_slice(self, i: int) -> slice:
        return slice(i * self.b, min((i + 1) * self.b, self.n))


def generate_test_matrix(kind, n: int, seed: int) -> np.ndarray:
    """linalg.py:63-78. Bit-identical to the reference (same PCG64 stream,
    same numpy operations); returned in Fortran order."""
    if n < 1:
        raise ERRORS["dim"]("matrix order must be >= 1")
    k = _value(kind)
    a = np.random.default_rng(seed).uniform(-1.0, 1.0, size=(n, n))
    if k == "cholesky":
        a = a @ a.T + n * np.eye(n)
    elif k == "lu":
        a[np.diag_indices(n)] = np.abs(a).sum(axis=1) + 1.0
    return np.asfortranarray(a)


def compute_flops(kind, task, n: int, b: int, k: int) -> float:
    """Closed-form per-task flop model (linalg.py:85-118); the TFLOP/s
    convention (n^3/3, 2n^3/3, 4n^3/3 in total) used by bench.py."""
    layout = BlockLayout(n, b)
    if not 0 <= k < layout.n_blocks:
        raise ERRORS["dim"](f"iteration {k} out of range for {layout.n_blocks} blocks")
    kd, t = _value(kind), _value(task)
    nk = n - k * b
    if kd == "cholesky" and t in ("pd", "pu", "tmu"):
        return {"pd": b ** 3 / 3.0, "pu": 0.0, "tmu": 2.0 * k * b * b * nk}[t]
    if kd == "lu" and t in ("pd", "pu", "tmu"):
        return {"pd": b * b * nk - b ** 3 / 3.0, "pu": b * b * max(nk - b, 0),
                "tmu": 2.0 * b * max(nk - b, 0) ** 2}[t]
    if kd == "qr" and t in ("pd", "pu", "tmu"):
        tmu = 4.0 * b * max(nk - b, 0) * (nk + b) if nk > b else 0.0
        return {"pd": 2.0 * b * b * (nk - b / 3.0), "pu": 0.0, "tmu": tmu}[t]
    raise ValueError(f"no flop model for {kind}/{task}")


def touched_elements(kind, task, n: int, b: int, k: int) -> float:
    """Elements written by a task (linalg.py:134-147), for the cost model."""
    kd, t = _value(kind), _value(task)
    nk = n - k * b
    if kd == "cholesky":
        return {"pd": float(b * b), "pu": float(max(nk - b, 0) * b), "tmu": float(nk * b)}[t]
    if kd == "lu":
        return {"pd": float(nk * b), "pu": float(max(nk - b, 0) * b),
                "tmu": float(max(nk - b, 0) ** 2)}[t]
    return {"pd": float(nk * b), "pu": 0.0,
            "tmu": float(max(nk - b, 0) * (nk + b)) if nk > b else 0.0}[t]


def algorithmic_flops(kind, n: int) -> float:
    """Whole-factorization flops (LAPACK convention, test_linalg.py:81-86)."""
    return {"cholesky": n ** 3 / 3.0, "lu": 2.0 * n ** 3 / 3.0, "qr": 4.0 * n ** 3 / 3.0}[_value(kind)]


class _QRFactors:
    """``qr_t`` (list of T) / ``_qr_vs`` (dict k -> V) views over the device
    panels (linalg.py:294-308). Supports len / indexing / ``del x[n:]`` and
    dict-style keys so the reference simulator's snapshot logic works."""

    def __init__(self, f: "Factorization", which: str):
        self._f, self._which = f, which

    def _count(self) -> int:
        return int(_lib.load().abft_qr_panels(self._f._ctx)) if self._f.kind == DecompositionKind.QR else 0

    def _get(self, k: int) -> np.ndarray:
        f = self._f
        p = k * f.b
        w = min(p + f.b, f.n) - p
        if self._which == "t":
            out = np.zeros((w, w), order="F")
            check(_lib.load().abft_get_qr_panel(f._ctx, k, None, 1, _lib.dptr(out), w))
        else:
            out = np.zeros((f.n - p, w), order="F")
            check(_lib.load().abft_get_qr_panel(f._ctx, k, _lib.dptr(out), f.n - p, None, 1))
        return out

    # list-like
    def __len__(self):
        return self._count()

    def __getitem__(self, k):
        if isinstance(k, slice):
            return [self._get(i) for i in range(self._count())[k]]
        n = self._count()
        if k < 0:
            k += n
        if not 0 <= k < n:
            raise (IndexError if self._which == "t" else KeyError)(k)
        return self._get(k)

    def __delitem__(self, k):
        if isinstance(k, slice) and k.step in (None, 1) and k.stop is None:
            start = k.start or 0
            self._f._set_qr_count(min(start, self._count()))
            return
        if self._which == "v":   # dict-style deletion of trailing panels
            self._f._set_qr_count(min(int(k), self._count()))
            return
        raise TypeError("only `del qr_t[n:]` is supported")

    def __iter__(self):
        for i in range(self._count()):
            yield self[i]

    # dict-like (for _qr_vs)
    def keys(self):
        return list(range(self._count()))

    def __contains__(self, k):
        return 0 <= k < self._count()

    def items(self):
        return [(k, self._get(k)) for k in range(self._count())]

    def values(self):
        return [self._get(k) for k in range(self._count())]

    def append(self, _):
        raise TypeError("QR panels are produced on the device")


class Factorization:
    """In-progress blocked factorization over a device-resident working
    matrix (linalg.py:159-359).

    Cholesky is left-looking, LU (no pivoting) and QR (compact WY)
    right-looking, exactly as the reference; the task kernels are the B200
    ones in libabft_b200.so.
    """

    def __init__(self, kind, a0: np.ndarray, b: int, device: int | None = None,
                 keep_input: bool = False, pivoting: bool = False):
        """``pivoting`` (LU only): partial pivoting with LAPACK dgetrf
        semantics (P a0 = L U; ``piv``) -- an option of the drop-in, the
        reference factors unpivoted (linalg.py:230-238)."""
        self.kind = DecompositionKind(_value(kind))
        self.a0 = a0
        self.b = int(b)
        n = a0.shape[0]
        if a0.ndim != 2 or a0.shape != (n, n):
            raise ERRORS["dim"]("square input required")
        self.layout = BlockLayout(n, self.b)
        self.device = 0 if device is None else int(device)
        lib = _lib.load()
        ctx = ctypes.c_void_p()
        check(lib.abft_create(ctypes.byref(ctx), _lib.KIND_CODE[self.kind.value], n, self.b,
                              self.device))
        self._ctx = ctx
        self._lib = lib
        if keep_input:  # device copy of the input for reset()/residual without a0
            check(lib.abft_keep_input(ctx, 1))
        host = np.asfortranarray(np.asarray(a0, dtype=np.float64))
        check(lib.abft_set_matrix(ctx, _lib.dptr(host), n))
        self.pivoting = bool(pivoting)
        if self.pivoting:
            check(lib.abft_set_pivoting(ctx, 1))
        self._m_cache: np.ndarray | None = None
        self.qr_t = _QRFactors(self, "t")
        self._qr_vs = _QRFactors(self, "v")

    @property
    def piv(self) -> np.ndarray:
        """Row interchanges of the pivoted LU (0-based, LAPACK ipiv - 1: row i
        was swapped with piv[i], in order); the identity when unpivoted."""
        out = np.empty(self.n, dtype=np.int32)
        check(self._lib.abft_get_pivots(self._ctx, out.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))))
        return out

    def __del__(self):
        ctx = getattr(self, "_ctx", None)
        if ctx:
            try:
                self._lib.abft_destroy(ctx)
            except Exception:
                pass
            self._ctx = None

    # -- state ------------------------------------------------------------
    @property
    def n(self) -> int:
        return self.a0.shape[0]

    @property
    def k_done(self) -> int:
        return int(self._lib.abft_k_done(self._ctx))

    @k_done.setter
    def k_done(self, k: int) -> None:
        check(self._lib.abft_set_k_done(self._ctx, int(k)))

    @property
    def complete(self) -> bool:
        return self.k_done >= self.layout.n_blocks

    @property
    def m(self) -> np.ndarray:
        """Host mirror of the device working matrix (Fortran order)."""
        if self._m_cache is None:
            out = np.empty((self.n, self.n), order="F")
            check(self._lib.abft_get_matrix(self._ctx, _lib.dptr(out), self.n))
            self._m_cache = out
        return self._m_cache

    @m.setter
    def m(self, value: np.ndarray) -> None:
        host = np.asfortranarray(np.asarray(value, dtype=np.float64))
        if host.shape != (self.n, self.n):
            raise ERRORS["dim"]("square input required")
        k, q = self.k_done, len(self.qr_t)
        check(self._lib.abft_set_matrix(self._ctx, _lib.dptr(host), self.n))
        self.k_done = k
        self._set_qr_count(q)
        self._m_cache = None

    def _dirty(self) -> None:
        self._m_cache = None

    def stream_input(self, a: np.ndarray) -> None:
        """abft_set_matrix_streamed: the host matrix (n x n float64, Fortran
        order; pinned for asynchronous copies) moves to the device block column
        by block column inside the next run_protected call, overlapped with
        the factorization (LU / QR factor their first panels as they arrive).
        The array is held until that call returns."""
        if a.shape != (self.n, self.n) or a.dtype != np.float64 or not a.flags.f_contiguous:
            raise ValueError("a must be an n x n float64 Fortran-ordered array")
        check(self._lib.abft_set_matrix_streamed(self._ctx, _lib.dptr(a), self.n))
        self._streamed_in = a
        self._m_cache = None

    def set_input_chunks(self, chunk: int = -1, split: int = -1, right_chunk: int = -1) -> None:
        """abft_set_input_chunks (-1: built-in; chunk 0: wait for all input)."""
        check(self._lib.abft_set_input_chunks(self._ctx, int(chunk), int(split), int(right_chunk)))

    def _set_qr_count(self, q: int) -> None:
        # panels beyond q are re-produced by the next PD(k) (del qr_t[n:])
        check(self._lib.abft_set_qr_panels(self._ctx, int(q)))

    def _qr_v(self, k: int) -> np.ndarray:
        return self._qr_vs[k]

    # -- tasks (linalg.py:192-258) -----------------------------------------
    def _task(self, k: int, task: str) -> None:
        self._dirty()
        check(self._lib.abft_task(self._ctx, int(k), _lib.TASK_CODE[task]))

    def task_tmu(self, k: int) -> None:
        self._task(k, "tmu")

    def task_pd(self, k: int) -> None:
        self._task(k, "pd")

    def task_pu(self, k: int) -> None:
        if self.kind != DecompositionKind.QR:
            self._task(k, "pu")

    def task_order(self) -> tuple:
        if self.kind == DecompositionKind.CHOLESKY:
            return (TaskKind.TMU, TaskKind.PD, TaskKind.PU)
        if self.kind == DecompositionKind.LU:
            return (TaskKind.PD, TaskKind.PU, TaskKind.TMU)
        return (TaskKind.PD, TaskKind.TMU)

    def run_iteration(self, k: int) -> None:
        """linalg.py:312-324 (order enforced)."""
        if k != self.k_done:
            raise ERRORS["dim"](f"expected iteration {self.k_done}, got {k}")
        if k >= self.layout.n_blocks:
            raise ERRORS["dim"]("factorization already complete")
        for task in self.task_order():
            self._task(k, _value(task))
        self.k_done = k + 1

    def run_all(self) -> "Factorization":
        while not self.complete:
            self.run_iteration(self.k_done)
        return self

    # -- device snapshots (replace _Run._snapshot/_restore, simulator.py:420-436)
    def snapshot(self, slot: int = 0) -> None:
        check(self._lib.abft_snapshot(self._ctx, slot))

    def restore(self, slot: int = 0) -> None:
        self._dirty()
        check(self._lib.abft_restore(self._ctx, slot))

    # -- reconstruction (linalg.py:340-359) ----------------------------------
    def reconstruct(self) -> np.ndarray:
        if not self.complete:
            raise ERRORS["breakdown"]("factorization incomplete")
        out = np.empty((self.n, self.n), order="F")
        check(self._lib.abft_reconstruct(self._ctx, _lib.dptr(out), self.n))
        return out

    def elapsed_ms(self) -> float:
        """Device time of the last iteration / factorize call (CUDA events)."""
        v = ctypes.c_double(0.0)
        check(self._lib.abft_last_elapsed_ms(self._ctx, ctypes.byref(v)))
        return float(v.value)


def residual(a: np.ndarray, factors: Factorization) -> float:
    """Relative Frobenius reconstruction error (linalg.py:362-368), computed
    on the device (reconstruct GEMM + deterministic reductions)."""
    host = np.asfortranarray(np.asarray(a, dtype=np.float64))
    out = ctypes.c_double(0.0)
    check(factors._lib.abft_residual(factors._ctx, _lib.dptr(host), host.shape[0],
                                     ctypes.byref(out)))
    return float(out.value)
