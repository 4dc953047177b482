"""Block-checksum ABFT — drop-in for slackwise.abft on the B200.

Same names, arguments and error behaviour as the reference
(/root/reference/pkg/src/slackwise/abft.py): ChecksumScheme :36,
ErrorKind :42, InjectedFault :48, CorrectionReport :60, RegionChecksums :87,
encode :118, maintain_gemm :138, verify_correct :174, inject_faults :283,
sample_fault_plan :310, checksum_flops :340. The arithmetic (block sums,
operand maintenance, threshold/classify/repair, injection) runs in the sm_100a
kernels of libabft_b200.so; only RNG draws and bookkeeping stay on the host.
"""
from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .linalg import DecompositionKind, TaskKind, _value, check, compute_flops

CHECK_TOLERANCE_FACTOR = 50.0   # abft.py:29
INDEX_SNAP_TOLERANCE = 1e-2     # abft.py:33


class ChecksumScheme(str, enum.Enum):
    NONE = "none"
    SINGLE = "single"
    FULL = "full"


class ErrorKind(str, enum.Enum):
    D0 = "0d"
    D1 = "1d"
    D2 = "2d"


@dataclass(frozen=True)
class InjectedFault:
    kind: ErrorKind
    row: int
    col: int
    magnitude: float
    iteration: int = 0
    task: TaskKind = TaskKind.TMU
    orientation: str = "col"
    extent: int = 1


@dataclass
class CorrectionReport:
    detected: dict = field(default_factory=lambda: {k: 0 for k in ErrorKind})
    corrected: dict = field(default_factory=lambda: {k: 0 for k in ErrorKind})
    uncorrectable: bool = False
    locations: list = field(default_factory=list)

    @property
    def total_detected(self) -> int:
        return sum(self.detected.values())

    @property
    def total_corrected(self) -> int:
        return sum(self.corrected.values())

    @property
    def clean(self) -> bool:
        return self.total_detected == 0 and not self.uncorrectable

    def merge(self, other: "CorrectionReport") -> None:
        for k in self.detected:
            self.detected[k] += other.detected[k]
            self.corrected[k] += other.corrected[k]
        self.uncorrectable = self.uncorrectable or other.uncorrectable
        self.locations.extend(other.locations)


# Classes used to build reports; install() rebinds them to the reference's
# so callers compare against their own enum members.
TYPES = {"report": CorrectionReport, "error_kind": ErrorKind}


def build_report(rep: _lib.Report, locs, n: int) -> CorrectionReport:
    """Translate the C-ABI report/locations (already in reference order)."""
    ek = TYPES["error_kind"]
    kinds = list(ek)
    out = TYPES["report"]()
    for i, k in enumerate(kinds):
        out.detected[k] = int(rep.detected[i])
        out.corrected[k] = int(rep.corrected[i])
    out.uncorrectable = bool(rep.uncorrectable)
    for i in range(min(n, rep.n_locations)):
        L = locs[i]
        out.locations.append((int(L.row), int(L.col), kinds[L.kind], bool(L.flag)))
    return out


class RegionChecksums:
    """Checksums of an aligned region (abft.py:87-115), held as dense arrays:
    col sums (nbr x cols), row sums (rows x nbc). ``col_plain[bi, bj]``
    style access returns the per-block vector like the reference's dicts."""

    def __init__(self, r0: int, c0: int, shape, b: int, scheme):
        scheme = ChecksumScheme(_value(scheme))
        if scheme == ChecksumScheme.NONE:
            raise ValueError("cannot encode with scheme 'none'")
        self.r0, self.c0 = int(r0), int(c0)
        self.rows, self.cols = (int(x) for x in shape)
        self.b = int(b)
        self.scheme = scheme
        nbr, nbc = -(-self.rows // self.b), -(-self.cols // self.b)
        self.cp = np.zeros((nbr, self.cols), order="F")
        self.cw = np.zeros((nbr, self.cols), order="F")
        self.rp = np.zeros((self.rows, nbc), order="F")
        self.rw = np.zeros((self.rows, nbc), order="F")

    def row_blocks(self) -> list:
        return [slice(i, min(i + self.b, self.rows)) for i in range(0, self.rows, self.b)]

    def col_blocks(self) -> list:
        return [slice(j, min(j + self.b, self.cols)) for j in range(0, self.cols, self.b)]

    def view(self, m: np.ndarray) -> np.ndarray:
        return m[self.r0:self.r0 + self.rows, self.c0:self.c0 + self.cols]

    def _blockdict(self, arr, cols_side: bool) -> dict:
        out = {}
        for bi, rs in enumerate(self.row_blocks()):
            for bj, cs in enumerate(self.col_blocks()):
                out[bi, bj] = arr[bi, cs] if cols_side else arr[rs, bj]
        return out

    @property
    def col_plain(self) -> dict:
        return self._blockdict(self.cp, True)

    @property
    def col_weighted(self) -> dict:
        return self._blockdict(self.cw, True)

    @property
    def row_plain(self) -> dict:
        return self._blockdict(self.rp, False) if self.scheme == ChecksumScheme.FULL else {}

    @property
    def row_weighted(self) -> dict:
        return self._blockdict(self.rw, False) if self.scheme == ChecksumScheme.FULL else {}


def _fortran(x: np.ndarray) -> np.ndarray:
    return np.asfortranarray(np.asarray(x, dtype=np.float64))


def encode(m: np.ndarray, b: int, scheme, r0: int = 0, c0: int = 0,
           shape=None) -> RegionChecksums:
    """abft.py:118-135 (block sums computed by the device checksum kernel)."""
    if shape is None:
        shape = (m.shape[0] - r0, m.shape[1] - c0)
    cs = RegionChecksums(r0, c0, shape, b, scheme)
    reg = _fortran(cs.view(m))
    lib = _lib.load()
    check(lib.abft_region_encode(_lib.dptr(reg), max(cs.rows, 1), cs.rows, cs.cols, cs.b,
                                 _lib.SCHEME_CODE[cs.scheme.value], _lib.dptr(cs.cp),
                                 _lib.dptr(cs.cw), _lib.dptr(cs.rp), _lib.dptr(cs.rw)))
    return cs


def maintain_gemm(cs: RegionChecksums, left: np.ndarray, right: np.ndarray) -> None:
    """abft.py:138-158: carry the sums through region -= left @ right from the
    operands (device GEMMs over the operand block sums)."""
    left = _fortran(left)
    right = _fortran(right)
    kdim = left.shape[1]
    lib = _lib.load()
    check(lib.abft_region_maintain(cs.rows, cs.cols, kdim, cs.b,
                                   _lib.SCHEME_CODE[cs.scheme.value], _lib.dptr(left),
                                   max(left.shape[0], 1), _lib.dptr(right), max(kdim, 1),
                                   _lib.dptr(cs.cp), _lib.dptr(cs.cw), _lib.dptr(cs.rp),
                                   _lib.dptr(cs.rw)))


def verify_correct(m: np.ndarray, cs: RegionChecksums, correct: bool = True):
    """abft.py:174-276: threshold, classify and repair on the device; the
    repaired region is written back into ``m``."""
    reg = _fortran(cs.view(m))
    lib = _lib.load()
    rep = _lib.Report()
    cap = max(16, reg.size)
    locs = (_lib.Location * cap)()
    check(lib.abft_region_verify(_lib.dptr(reg), max(cs.rows, 1), cs.rows, cs.cols, cs.b,
                                 _lib.SCHEME_CODE[cs.scheme.value], int(bool(correct)), cs.r0,
                                 cs.c0, _lib.dptr(cs.cp), _lib.dptr(cs.cw), _lib.dptr(cs.rp),
                                 ctypes.byref(rep), locs, cap))
    if correct and rep.n_locations:
        cs.view(m)[...] = reg
    return build_report(rep, locs, cap)


def _fault_struct(f, absolute: bool, u: float = 0.0, negate: bool = False) -> _lib.Fault:
    s = _lib.Fault()
    s.kind = ("0d", "1d", "2d").index(_value(f.kind) if not isinstance(f, dict) else f["kind"])
    get = (lambda k: f[k]) if isinstance(f, dict) else (lambda k: getattr(f, k))
    s.orientation = 0 if get("orientation") == "col" else 1
    s.row = int(get("row"))
    s.col = int(get("col"))
    s.extent = int(get("extent"))
    s.absolute = 1 if absolute else 0
    s.u = float(u)
    s.negate = 1 if negate else 0
    s.magnitude = float(get("magnitude")) if absolute else 0.0
    return s


def inject_faults(m: np.ndarray, plan) -> None:
    """abft.py:283-307 (device kernel; IndexError outside the matrix)."""
    plan = list(plan)
    if not plan:
        return
    n_rows, n_cols = m.shape
    for f in plan:
        if not (0 <= f.row < n_rows and 0 <= f.col < n_cols):
            raise IndexError(f"fault at ({f.row}, {f.col}) outside matrix")
    arr = (_lib.Fault * len(plan))(*[_fault_struct(f, True) for f in plan])
    host = _fortran(m)
    check(_lib.load().abft_inject(_lib.dptr(host), max(n_rows, 1), n_rows, n_cols, arr, len(plan),
                                  0.0))
    m[...] = host


def draw_plan(rng, counts: dict, r0: int, c0: int, rows: int, cols: int, b: int):
    """The data-independent draws of sample_fault_plan (abft.py:314-332),
    in the reference's exact order. Returns dicts with u/negate instead of a
    magnitude; the device applies mag = (u*1e-3)*max(scale, 1)."""
    norm = {ErrorKind(_value(k)): int(v) for k, v in (counts or {}).items()}
    plan = []
    for kind in ErrorKind:
        for _ in range(norm.get(kind, 0)):
            r = r0 + int(rng.integers(rows))
            c = c0 + int(rng.integers(cols))
            u = float(rng.uniform(0.5, 2.0))
            negate = bool(rng.random() < 0.5)
            extent = min(b, 4, rows, cols) if kind != ErrorKind.D0 else 1
            extent = max(extent, 1)
            if kind == ErrorKind.D1:
                r = r0 + (r - r0) - (r - r0) % b
            r = min(r, r0 + rows - extent)
            c = min(c, c0 + cols - extent)
            plan.append({"kind": kind.value, "row": r, "col": c, "u": u, "negate": negate,
                         "extent": extent, "orientation": "col"})
    return plan


def sample_fault_plan(rng, counts: dict, r0: int, c0: int, rows: int, cols: int, b: int,
                      scale: float, iteration: int) -> list:
    """abft.py:310-333 (host RNG; identical draws and magnitudes)."""
    out = []
    for d in draw_plan(rng, counts, r0, c0, rows, cols, b):
        mag = d["u"] * 1e-3 * max(scale, 1.0)
        if d["negate"]:
            mag = -mag
        out.append(InjectedFault(kind=ErrorKind(d["kind"]), row=d["row"], col=d["col"],
                                 magnitude=mag, iteration=iteration, orientation="col",
                                 extent=d["extent"]))
    return out


def checksum_flops(scheme, kind, task, n: int, b: int, k: int,
                   component: str = "update") -> float:
    """Checksum cost model (abft.py:340-360); host arithmetic."""
    if _value(scheme) == "none":
        return 0.0
    flops = compute_flops(kind, task, n, b, k)
    if flops == 0.0:
        return 0.0
    sides = 2.0 if _value(scheme) == "full" else 1.0
    if component == "update":
        return sides * 2.0 * flops / b
    if component == "verify":
        from .linalg import touched_elements
        return sides * 2.0 * touched_elements(kind, task, n, b, k)
    raise ValueError(f"unknown checksum component {component!r}")
