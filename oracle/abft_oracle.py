"""numpy restatement of the reference hot path (test infrastructure only).

Reference: /root/reference/pkg/src/slackwise/{linalg,abft,simulator}.py.
Kinds, schemes and error kinds are plain strings here ("cholesky"/"lu"/"qr",
"none"/"single"/"full", "0d"/"1d"/"2d") so the oracle has no dependency on the
product package. Checksum bookkeeping is vectorised over blocks (one padded
reshape per region) instead of the reference's per-block Python loops; the
decision logic (thresholds, classification, repair order, location order) is
restated line by line.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# abft.py:29, :33
CHECK_TOLERANCE_FACTOR = 50.0
INDEX_SNAP_TOLERANCE = 1e-2
EPS64 = float(np.finfo(np.float64).eps)
EPS32 = float(np.finfo(np.float32).eps)

# fp32 (s*) restatement of the threshold rule (the reference
# has no fp32 path, parity unpinned). tau32 = 2048 * max(max|blk|, 1) * eps32
# = max(max|blk|, 1) / 4096, which sits 2.05x below the reference's smallest
# fault (0.5e-3 * max(max|region|, 1), abft.py:319-321), so every injected
# fault trips the check; the snap tolerance of SINGLE's index recovery is 0.25
# (the fp32 data's rounding moves dw / dp by ~1e-4 of a fault; the sampler's
# 1-D / 2-D streak ratios have fractional parts 0.59-0.61 and never snap).
# Mirrors TAU32_MULT / SNAP_TOL32 in paper_2301_03166_b200/csrc/abft_kernels.cuh.
TAU32_MULT = 2048.0
SNAP_TOL32 = 0.25
PRECISIONS = ("f64", "f32")


def threshold(b: int, bmax, precision: str = "f64"):
    """_block_threshold (abft.py:161-163), in the reference's operation order;
    ``precision="f32"`` is the s* restatement above."""
    if precision == "f32":
        return TAU32_MULT * np.maximum(bmax, 1.0) * EPS32
    return CHECK_TOLERANCE_FACTOR * b * np.maximum(bmax, 1.0) * EPS64

ALL_KINDS = ("cholesky", "lu", "qr")
ERROR_KINDS = ("0d", "1d", "2d")   # ErrorKind iteration order, abft.py:42-45


class BreakdownError(ArithmeticError):
    """NumericBreakdownError (linalg.py:41-43)."""


# ---------------------------------------------------------------------------
# inputs and flop convention
# ---------------------------------------------------------------------------

def generate_test_matrix(kind: str, n: int, seed: int) -> np.ndarray:
    """linalg.py:63-78: PCG64 uniform(-1, 1); SPD a a^T + n I; LU diagonal =
    absolute row sum + 1; QR raw; Fortran order."""
    x = np.random.default_rng(seed).uniform(-1.0, 1.0, size=(n, n))
    if kind == "cholesky":
        x = x @ x.T + n * np.eye(n)
    elif kind == "lu":
        x[np.diag_indices(n)] = np.abs(x).sum(axis=1) + 1.0
    return np.asfortranarray(x)


def algorithmic_flops(kind: str, n: int) -> float:
    """LAPACK convention pinned by pkg/tests/test_linalg.py:81-86."""
    return {"cholesky": n ** 3 / 3.0, "lu": 2.0 * n ** 3 / 3.0,
            "qr": 4.0 * n ** 3 / 3.0}[kind]


def region_of(kind: str, n: int, b: int, k: int):
    """_tmu_region (simulator.py:86-94): (r0, c0, rows, cols)."""
    p = k * b
    pe = min(p + b, n)
    return {"cholesky": (p, p, n - p, pe - p),
            "lu": (pe, pe, n - pe, n - pe)}.get(kind, (p, pe, n - p, n - pe))


# ---------------------------------------------------------------------------
# checksums (abft.py:87-158)
# ---------------------------------------------------------------------------

def _blocked(x: np.ndarray, b: int) -> np.ndarray:
    """Zero-pad to whole b x b blocks and view as [bi, i, bj, j]."""
    rows, cols = x.shape
    nbr, nbc = -(-rows // b), -(-cols // b)
    pad = np.zeros((nbr * b, nbc * b))
    pad[:rows, :cols] = x
    return pad.reshape(nbr, b, nbc, b)


def block_sums(x: np.ndarray, b: int):
    """Per-block plain / index-weighted column sums (nbr x cols), row sums
    (rows x nbc) and max|x| (nbr x nbc) of a region (abft.py:124-134, :162).
    Weights restart at 0 in every block (abft.py:126, :132). Works one block
    row at a time on strided views (no copy of the region), like the
    reference's per-block loops but vectorised across the block row."""
    rows, cols = x.shape
    nbr, nbc = -(-rows // b), -(-cols // b)
    cp = np.zeros((nbr, cols))
    cw = np.zeros((nbr, cols))
    rp = np.zeros((rows, nbc))
    rw = np.zeros((rows, nbc))
    bmax = np.zeros((nbr, nbc))
    wfull = np.arange(b, dtype=np.float64)
    full_c = (cols // b) * b
    for bi in range(nbr):
        r0, r1 = bi * b, min(bi * b + b, rows)
        blk = x[r0:r1, :]
        cp[bi] = blk.sum(axis=0)
        cw[bi] = wfull[:r1 - r0] @ blk
        if full_c:
            v3 = blk[:, :full_c].reshape(r1 - r0, full_c // b, b)
            rp[r0:r1, :full_c // b] = v3.sum(axis=2)
            rw[r0:r1, :full_c // b] = v3 @ wfull
            bmax[bi, :full_c // b] = np.abs(v3).max(axis=(0, 2))
        if full_c < cols:
            tail = blk[:, full_c:]
            rp[r0:r1, nbc - 1] = tail.sum(axis=1)
            rw[r0:r1, nbc - 1] = tail @ wfull[:cols - full_c]
            bmax[bi, nbc - 1] = np.abs(tail).max()
    return cp, cw, rp, rw, bmax


@dataclass
class Checksums:
    """RegionChecksums (abft.py:87-115) as dense arrays."""
    r0: int
    c0: int
    rows: int
    cols: int
    b: int
    scheme: str
    cp: np.ndarray
    cw: np.ndarray
    rp: np.ndarray | None
    rw: np.ndarray | None


def encode(m: np.ndarray, b: int, scheme: str, r0: int = 0, c0: int = 0,
           shape=None) -> Checksums:
    """abft.py:118-135."""
    if scheme == "none":
        raise ValueError("cannot encode with scheme 'none'")
    if shape is None:
        shape = (m.shape[0] - r0, m.shape[1] - c0)
    rows, cols = shape
    cp, cw, rp, rw, _ = block_sums(m[r0:r0 + rows, c0:c0 + cols], b)
    full = scheme == "full"
    return Checksums(r0, c0, rows, cols, b, scheme, cp, cw,
                     rp if full else None, rw if full else None)


def maintain(cs: Checksums, left: np.ndarray, right: np.ndarray) -> None:
    """maintain_gemm (abft.py:138-158): update from the operands of
    region -= left @ right, never from the result."""
    b = cs.b
    rows, kdim = left.shape
    nbr = -(-rows // b)
    padl = np.zeros((nbr * b, kdim))
    padl[:rows] = left
    lt = padl.reshape(nbr, b, kdim)
    w = np.arange(b, dtype=np.float64)
    cs.cp = cs.cp - lt.sum(axis=1) @ right                      # (1^T L_i) R_j
    cs.cw = cs.cw - np.einsum("i,aik->ak", w, lt) @ right       # (w^T L_i) R_j
    if cs.scheme == "full":
        cols = right.shape[1]
        nbc = -(-cols // b)
        padr = np.zeros((kdim, nbc * b))
        padr[:, :cols] = right
        rt = padr.reshape(kdim, nbc, b)
        cs.rp = cs.rp - left @ rt.sum(axis=2)                   # L_i (R_j 1)
        cs.rw = cs.rw - left @ np.einsum("j,knj->kn", w, rt)    # L_i (R_j w)


# ---------------------------------------------------------------------------
# verification (abft.py:161-276)
# ---------------------------------------------------------------------------

@dataclass
class OracleReport:
    """CorrectionReport (abft.py:60-84) with string kinds."""
    detected: dict = field(default_factory=lambda: {k: 0 for k in ERROR_KINDS})
    corrected: dict = field(default_factory=lambda: {k: 0 for k in ERROR_KINDS})
    uncorrectable: bool = False
    locations: list = field(default_factory=list)

    def to_json(self) -> dict:
        return {"detected": dict(self.detected), "corrected": dict(self.corrected),
                "uncorrectable": bool(self.uncorrectable),
                "locations": [[int(r), int(c), k, bool(f)] for r, c, k, f in self.locations]}


def _snap_index(dw: float, dp: float, limit: int, tol: float = INDEX_SNAP_TOLERANCE):
    """_recovered_index (abft.py:208-213); Python round() is half-to-even."""
    ratio = dw / dp
    idx = round(ratio)
    if abs(ratio - idx) <= tol and 0 <= idx < limit:
        return int(idx)
    return None


def verify(m: np.ndarray, cs: Checksums, correct: bool = True,
           precision: str = "f64") -> OracleReport:
    """verify_correct (abft.py:174-205) with _handle_single / _handle_full.
    ``precision="f64"`` is the reference; "f32" is the s* restatement of the
    threshold and snap rules (TAU32_MULT, SNAP_TOL32 above)."""
    rep = OracleReport()
    b = cs.b
    view = m[cs.r0:cs.r0 + cs.rows, cs.c0:cs.c0 + cs.cols]
    cp, cw, rp, _, bmax = block_sums(view, b)
    tau = threshold(b, bmax, precision)                                 # _block_threshold
    snap_tol = SNAP_TOL32 if precision == "f32" else INDEX_SNAP_TOLERANCE
    nbr, nbc = bmax.shape
    d_col = cp - cs.cp
    d_w = cw - cs.cw
    col_tau = np.repeat(tau, b, axis=1)[:, :cs.cols]
    bad_c = np.abs(d_col) > col_tau
    full = cs.scheme == "full"
    if full:
        d_row = rp - cs.rp
        row_tau = np.repeat(tau, b, axis=0)[:cs.rows, :]
        bad_r = np.abs(d_row) > row_tau
    for bi in range(nbr):
        rs, re_ = bi * b, min(bi * b + b, cs.rows)
        for bj in range(nbc):
            c_s, c_e = bj * b, min(bj * b + b, cs.cols)
            bc = np.flatnonzero(bad_c[bi, c_s:c_e])
            br = np.flatnonzero(bad_r[rs:re_, bj]) if full else np.zeros(0, int)
            if bc.size == 0 and br.size == 0:
                continue
            blk = view[rs:re_, c_s:c_e]
            corner = (cs.r0 + rs, cs.c0 + c_s)
            if not full:
                fixes = []
                for j in bc:
                    idx = _snap_index(d_w[bi, c_s + j], d_col[bi, c_s + j], re_ - rs, snap_tol)
                    if idx is None:
                        fixes = None
                        break
                    fixes.append((idx, int(j), d_col[bi, c_s + j]))
                if fixes is None:
                    kind = "1d" if bc.size == 1 else "2d"
                    rep.detected[kind] += 1
                    rep.uncorrectable = True
                    rep.locations.append((*corner, kind, False))
                    continue
                for idx, j, delta in fixes:
                    rep.detected["0d"] += 1
                    if correct:
                        blk[idx, j] -= delta
                        rep.corrected["0d"] += 1
                    rep.locations.append((corner[0] + idx, corner[1] + j, "0d", correct))
                continue
            # _classify (abft.py:166-171)
            if br.size <= 1 and bc.size <= 1:
                kind = "0d"
            elif br.size <= 1 or bc.size <= 1:
                kind = "1d"
            else:
                kind = "2d"
            if kind == "0d":
                rep.detected["0d"] += 1
                if br.size == 0 or bc.size == 0:
                    rep.uncorrectable = True
                    rep.locations.append((*corner, "0d", False))
                    continue
                i, j = int(br[0]), int(bc[0])
                if correct:
                    blk[i, j] -= d_col[bi, c_s + j]
                    rep.corrected["0d"] += 1
                rep.locations.append((corner[0] + i, corner[1] + j, "0d", correct))
            elif kind == "1d":
                rep.detected["1d"] += 1
                if bc.size == 1:
                    j = int(bc[0])
                    if correct:
                        blk[br, j] -= d_row[rs + br, bj]
                        rep.corrected["1d"] += 1
                else:
                    i = int(br[0])  # IndexError when br is empty (abft.py:267)
                    if correct:
                        blk[i, bc] -= d_col[bi, c_s + bc]
                        rep.corrected["1d"] += 1
                rep.locations.append((*corner, "1d", correct))
            else:
                rep.detected["2d"] += 1
                rep.uncorrectable = True
                rep.locations.append((*corner, "2d", False))
    return rep


# ---------------------------------------------------------------------------
# fault injection (abft.py:283-333)
# ---------------------------------------------------------------------------

def draw_fault_plan(rng, counts: dict, r0: int, c0: int, rows: int, cols: int, b: int):
    """The data-independent draws of sample_fault_plan (abft.py:314-332), in
    the same order: integers(rows), integers(cols), uniform(0.5, 2), random()."""
    plan = []
    for kind in ERROR_KINDS:
        for _ in range(int(counts.get(kind, 0))):
            r = r0 + int(rng.integers(rows))
            c = c0 + int(rng.integers(cols))
            u = float(rng.uniform(0.5, 2.0))
            neg = bool(rng.random() < 0.5)
            ext = max(min(b, 4, rows, cols) if kind != "0d" else 1, 1)
            if kind == "1d":
                r = r0 + (r - r0) - (r - r0) % b
            r = min(r, r0 + rows - ext)
            c = min(c, c0 + cols - ext)
            plan.append({"kind": kind, "row": r, "col": c, "u": u, "negate": neg,
                         "extent": ext, "orientation": "col"})
    return plan


def magnitude(u: float, negate: bool, scale: float) -> float:
    """abft.py:319-321."""
    mag = u * 1e-3 * max(scale, 1.0)
    return -mag if negate else mag


def inject(m: np.ndarray, faults) -> None:
    """inject_faults (abft.py:283-307); faults carry 'magnitude'."""
    nr, nc = m.shape
    for f in faults:
        r, c, mag = f["row"], f["col"], f["magnitude"]
        if not (0 <= r < nr and 0 <= c < nc):
            raise IndexError(f"fault at ({r}, {c}) outside matrix")
        ext = max(2, f.get("extent", 1))
        if f["kind"] == "0d":
            m[r, c] += mag
        elif f["kind"] == "1d":
            if f.get("orientation", "col") == "col":
                e = min(r + ext, nr)
                m[r:e, c] += mag * (1.0 + 0.1 * np.arange(e - r))
            else:
                e = min(c + ext, nc)
                m[r, c:e] += mag * (1.0 + 0.1 * np.arange(e - c))
        else:
            er_, ec_ = min(r + ext, nr), min(c + ext, nc)
            ramp = np.add.outer(np.arange(er_ - r) * 0.1, np.arange(ec_ - c) * 0.07) + 1.0
            m[r:er_, c:ec_] += mag * ramp


# ---------------------------------------------------------------------------
# numeric engine (linalg.py:159-359)
# ---------------------------------------------------------------------------

class OracleFactorization:
    def __init__(self, kind: str, a0: np.ndarray, b: int):
        n = a0.shape[0]
        if a0.shape != (n, n) or not (1 <= b <= n):
            raise ValueError("bad dimensions")
        self.kind, self.n, self.b = kind, n, b
        self.nb = -(-n // b)
        self.m = np.array(a0, dtype=np.float64, order="F", copy=True)
        self.qr_t: list = []
        self.qr_vs: dict = {}
        self.k_done = 0

    def _span(self, k):
        p = k * self.b
        return p, min(p + self.b, self.n)

    # -- TMU operands (simulator.py:135-157 / linalg.py:192-213) --
    def tmu_operands(self, k):
        """(left, right, target view) of region -= left @ right, or None."""
        n, m = self.n, self.m
        p, pe = self._span(k)
        if self.kind == "cholesky":
            if k == 0:
                return None
            return m[p:n, 0:p], m[p:pe, 0:p].T, m[p:n, p:pe]
        if self.kind == "lu":
            if pe >= n:
                return None
            return m[pe:n, p:pe], m[p:pe, pe:n], m[pe:n, pe:n]
        if pe >= n or k >= len(self.qr_t):
            return None
        v, t = self.qr_vs[k], self.qr_t[k]
        c = m[p:n, pe:n]
        return v, t.T @ (v.T @ c), c

    def tmu(self, k):
        ops = self.tmu_operands(k)
        if ops is not None:
            left, right, tgt = ops
            tgt -= left @ right

    def pd(self, k):
        n, b = self.n, self.b
        p, pe = self._span(k)
        w = pe - p
        if self.kind == "cholesky":          # linalg.py:219-229 (Crout)
            d = self.m[p:pe, p:pe]
            for j in range(w):
                piv = d[j, j] - d[j, :j] @ d[j, :j]
                if piv <= 0.0 or not np.isfinite(piv):
                    raise BreakdownError(f"non-positive pivot at column {p + j}")
                d[j, j] = math.sqrt(piv)
                if j + 1 < w:
                    d[j + 1:, j] = (d[j + 1:, j] - d[j + 1:, :j] @ d[j, :j]) / d[j, j]
            d[np.triu_indices(w, 1)] = 0.0
        elif self.kind == "lu":              # linalg.py:230-238 (dgetf2, no pivot)
            pan = self.m[p:n, p:pe]
            for j in range(w):
                piv = pan[j, j]
                if piv == 0.0 or not np.isfinite(piv):
                    raise BreakdownError(f"zero pivot at column {p + j}")
                pan[j + 1:, j] /= piv
                if j + 1 < w:
                    pan[j + 1:, j + 1:w] -= np.outer(pan[j + 1:, j], pan[j, j + 1:w])
        else:
            self._householder(k)

    def _householder(self, k):
        """_qr_panel (linalg.py:260-300)."""
        n = self.n
        p, pe = self._span(k)
        w = pe - p
        pan = self.m[p:n, p:pe]
        v = np.zeros((n - p, w))
        tau = np.zeros(w)
        for j in range(w):
            x = pan[j:, j].copy()
            nx = np.linalg.norm(x)
            if nx == 0.0:
                v[j, j] = 1.0
                continue
            alpha = -math.copysign(nx, x[0] if x[0] != 0 else 1.0)
            vj = x.copy()
            vj[0] -= alpha
            vn2 = vj @ vj
            if vn2 == 0.0:
                v[j, j] = 1.0
                pan[j, j] = alpha
                continue
            beta = 2.0 / vn2
            pan[j:, j + 1:] -= beta * np.outer(vj, vj @ pan[j:, j + 1:])
            pan[j, j] = alpha
            pan[j + 1:, j] = 0.0
            v[j:, j] = vj / vj[0]
            tau[j] = beta * vj[0] * vj[0]
        t = np.zeros((w, w))
        for j in range(w):
            t[j, j] = tau[j]
            if j:
                t[:j, j] = -tau[j] * (t[:j, :j] @ (v[:, :j].T @ v[:, j]))
        self.qr_t.append(t)
        self.qr_vs[k] = v

    def pu(self, k):
        """linalg.py:242-258 (solves through LAPACK dgesv)."""
        n = self.n
        p, pe = self._span(k)
        if pe >= n or self.kind == "qr":
            return
        if self.kind == "cholesky":
            self.m[pe:n, p:pe] = np.linalg.solve(self.m[p:pe, p:pe], self.m[pe:n, p:pe].T).T
            self.m[p:pe, pe:n] = 0.0
        else:
            l11 = np.tril(self.m[p:pe, p:pe], -1) + np.eye(pe - p)
            self.m[p:pe, pe:n] = np.linalg.solve(l11, self.m[p:pe, pe:n])

    def order(self):
        """task_order (linalg.py:326-331)."""
        return {"cholesky": ("tmu", "pd", "pu"), "lu": ("pd", "pu", "tmu")}.get(
            self.kind, ("pd", "tmu"))

    def run_all(self):
        for k in range(self.k_done, self.nb):
            for task in self.order():
                getattr(self, task)(k)
            self.k_done = k + 1
        return self

    def reconstruct(self) -> np.ndarray:
        """linalg.py:340-359."""
        m, n = self.m, self.n
        if self.kind == "cholesky":
            low = np.tril(m)
            return low @ low.T
        if self.kind == "lu":
            return (np.tril(m, -1) + np.eye(n)) @ np.triu(m)
        out = np.triu(m)
        for k in range(len(self.qr_t) - 1, -1, -1):
            p = k * self.b
            v, t = self.qr_vs[k], self.qr_t[k]
            out[p:n, :] -= v @ (t @ (v.T @ out[p:n, :]))
        return out


def residual(a: np.ndarray, f: OracleFactorization) -> float:
    """linalg.py:362-368."""
    diff = np.linalg.norm(a - f.reconstruct())
    na = np.linalg.norm(a)
    return float(diff if na == 0.0 else diff / na)


# ---------------------------------------------------------------------------
# protected iteration (simulator.py:97-167)
# ---------------------------------------------------------------------------

def protected_iteration(f: OracleFactorization, k: int, scheme: str,
                        counts: dict | None = None, rng=None,
                        correct: bool = True, precision: str = "f64") -> OracleReport:
    rep = OracleReport()
    for task in f.order():
        if task != "tmu":
            getattr(f, task)(k)
            continue
        r0, c0, rows, cols = region_of(f.kind, f.n, f.b, k)
        live = rows > 0 and cols > 0
        cs = encode(f.m, f.b, scheme, r0, c0, (rows, cols)) if (scheme != "none" and live) else None
        ops = f.tmu_operands(k)
        if ops is not None:
            left, right, tgt = ops
            if cs is not None:
                maintain(cs, left, right)
            tgt -= left @ right
        if live and counts and any(counts.values()):
            scale = float(np.abs(f.m[r0:r0 + rows, c0:c0 + cols]).max(initial=0.0))
            plan = draw_fault_plan(rng, counts, r0, c0, rows, cols, f.b)
            for flt in plan:
                flt["magnitude"] = magnitude(flt["u"], flt["negate"], scale)
            inject(f.m, plan)
        if cs is not None:
            rep = verify(f.m, cs, correct, precision)
    f.k_done = k + 1
    return rep
