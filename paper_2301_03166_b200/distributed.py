"""Multi-GPU ABFT factorization: 1-D block-cyclic columns over one process
per GPU.

The reference (/root/reference/pkg/src/slackwise/) is a single-process
simulator; its protected iteration (simulator.py:97-167) and factorization
(linalg.py:159-359) are distributed here the way the survey plans it:

* rank g owns global column blocks j with j mod G == g (contiguous locally),
  so every b x b checksum block, its verification and its repair are local;
* LU / QR: the owner of panel k factors it and the panel (plus L11^{-1} or
  T) is **broadcast** from k mod G; every rank then updates its own trailing
  columns with the fused-checksum trailing-update GEMM;
* Cholesky is right-looking (default): the owner of panel k verifies,
  factors and **broadcasts** it (with its block-row checksums), every rank
  applies the rank-b update to its own trailing column blocks and maintains
  their checksums from the operands (abft.py:138-158 one panel at a time);
  with the cross-rank look-ahead the owner of panel k does that mid-update.
  ABFT_DIST_CHOL=left keeps the reference's left-looking form (linalg.py:
  192-200: partial panel products **sum-reduced** to the owner);
* the fault plan is drawn on every rank from the same seeded Generator in
  sample_fault_plan's order (abft.py:310-333); the magnitude scale
  max|region| (simulator.py:159-160) is an all-reduce MAX over ranks;
* events come back in global coordinates and are merged into the
  reference's order (iteration, block row, block column, column).

Transport: torch.distributed. With the NCCL backend the collectives run on
the context's CUDA stream directly on device buffers; any other backend
(gloo: the CPU-side test harness and the two-ranks-on-one-GPU GPU tests) is
staged through host memory. The compute is the same sm_100a library either
way; there is no CPU compute path.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _lib
from .abft import ChecksumScheme, CorrectionReport, TYPES, draw_plan
from .linalg import DecompositionKind, BlockLayout, ERRORS, _value, check
from .simulator import _plan_structs, _tmu_region

EVENT_FIELDS = ("iter", "block_row", "block_col", "seq", "row", "col", "kind", "flag",
                "detected_kind", "corrected", "uncorrectable")


# ---------------------------------------------------------------------------
# host-side layout logic (pure Python; tested on CPU with gloo)
# ---------------------------------------------------------------------------
def owner_of(k: int, world: int) -> int:
    """Rank owning global column block k."""
    return k % world


def local_blocks(nb: int, rank: int, world: int) -> list:
    """Global column blocks stored (in this order) by `rank`."""
    return list(range(rank, nb, world))


def local_columns(n: int, b: int, rank: int, world: int) -> int:
    nb = -(-n // b)
    return sum(min(b, n - j * b) for j in local_blocks(nb, rank, world))


def scatter_columns(a: np.ndarray, b: int, rank: int, world: int) -> np.ndarray:
    """The owned column blocks of a global matrix, concatenated (n x ncl)."""
    n = a.shape[0]
    nb = -(-n // b)
    cols = [a[:, j * b:min((j + 1) * b, n)] for j in local_blocks(nb, rank, world)]
    return np.asfortranarray(np.concatenate(cols, axis=1)) if cols else np.zeros((n, 0), order="F")


def assemble_columns(parts: list, n: int, b: int) -> np.ndarray:
    """Inverse of scatter_columns over all ranks (parts[r] = rank r's n x ncl_r)."""
    world = len(parts)
    nb = -(-n // b)
    out = np.empty((n, n), order="F")
    for r, part in enumerate(parts):
        off = 0
        for j in local_blocks(nb, r, world):
            w = min(b, n - j * b)
            out[:, j * b:j * b + w] = part[:, off:off + w]
            off += w
    return out


def scatter_input(a0, n: int, b: int, group=None, root: int = 0, device: int = 0) -> np.ndarray:
    """The rank's own column blocks of a global matrix that only `root`
    holds (the others pass None): root cuts every rank's blocks and sends
    them point to point (NCCL: device buffers; other backends: host), so no
    rank but root ever materialises the n x n input (8.6 GB at N = 32768)."""
    import torch
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    native = dist.get_backend(group) == "nccl"
    dev = torch.device("cuda", device) if native else torch.device("cpu")
    gr = (lambda r: r) if group is None else (lambda r: dist.get_global_rank(group, r))
    if rank == root:
        a = np.asarray(a0)
        if a.shape != (n, n):
            raise ERRORS["dim"]("square input of order n required on the root rank")
        for r in range(world):
            if r == root:
                continue
            part = scatter_columns(a, b, r, world)
            # row-major (ncl x n) storage of the Fortran (n x ncl) block
            t = torch.from_numpy(np.ascontiguousarray(part.T)).to(dev)
            dist.send(t, gr(r), group=group)
        return scatter_columns(a, b, root, world)
    ncl = local_columns(n, b, rank, world)
    t = torch.empty((ncl, n), dtype=torch.float64, device=dev)
    dist.recv(t, gr(root), group=group)
    return np.asfortranarray(t.cpu().numpy().T)


def merge_events(per_rank: list) -> list:
    """Events of all ranks (dicts with EVENT_FIELDS) in the reference's
    location order: iteration, block row, block column, column
    (abft.py:60-84 / verify_correct's loops, abft.py:174-205)."""
    allev = [e for evs in per_rank for e in evs]
    allev.sort(key=lambda e: (e["iter"], e["block_row"], e["block_col"], e["seq"]))
    return allev


def reports_from_events(events: list, k0: int, nb: int) -> list:
    """One CorrectionReport per iteration k0..nb-1 from merged events."""
    kinds = list(TYPES["error_kind"])
    reps = []
    by_k = {}
    for e in events:
        by_k.setdefault(e["iter"], []).append(e)
    for k in range(k0, nb):
        rep = TYPES["report"]()
        for kk in kinds:
            rep.detected[kk] = 0
            rep.corrected[kk] = 0
        for e in by_k.get(k, []):
            dk = kinds[e["detected_kind"]]
            rep.detected[dk] += 1
            if e["corrected"]:
                rep.corrected[dk] += 1
            if e["uncorrectable"]:
                rep.uncorrectable = True
            rep.locations.append((e["row"], e["col"], kinds[e["kind"]], bool(e["flag"])))
        reps.append(rep)
    return reps


# ---------------------------------------------------------------------------
# transport
# ---------------------------------------------------------------------------
class _Transport:
    """torch.distributed collectives on the context stream (NCCL: device
    buffers; other backends: staged through host memory)."""

    def __init__(self, group, stream_ptr: int, device: int, comm_ptr: int | None = None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist, self.group = torch, dist, group
        self.native = dist.get_backend(group) == "nccl"
        dev = torch.device("cuda", device)
        self.stream = torch.cuda.ExternalStream(stream_ptr, device=dev)
        self.comm = torch.cuda.ExternalStream(comm_ptr, device=dev) if comm_ptr else self.stream

    def _global(self, r: int) -> int:
        return r if self.group is None else self.dist.get_global_rank(self.group, r)

    def _run(self, t, fn, comm: bool = False):
        torch = self.torch
        with torch.cuda.stream(self.comm if comm else self.stream):
            if self.native:
                fn(t)
            else:
                h = t.cpu()
                fn(h)
                t.copy_(h)

    def broadcast(self, t, src: int, comm: bool = False) -> None:
        self._run(t, lambda x: self.dist.broadcast(x, self._global(src), group=self.group), comm)

    def reduce_sum(self, t, dst: int) -> None:
        if self.native:
            self._run(t, lambda x: self.dist.reduce(x, self._global(dst), group=self.group))
        else:
            self._run(t, lambda x: self.dist.all_reduce(x, group=self.group))

    def allreduce_max(self, t) -> None:
        self._run(t, lambda x: self.dist.all_reduce(x, op=self.dist.ReduceOp.MAX, group=self.group))


# ---------------------------------------------------------------------------
# distributed factorization
# ---------------------------------------------------------------------------
class DistributedFactorization:
    """Factorization(kind, a0, b) (linalg.py:159-188) distributed over the
    ranks of a torch.distributed process group, one GPU per rank.

    Every rank passes the same global input ``a0`` (the reference's
    generate_test_matrix is deterministic per seed) and keeps only its
    column blocks on its GPU.
    """

    def __init__(self, kind, a0: np.ndarray | None, b: int, group=None, device: int | None = None,
                 keep_input: bool = False, root: int | None = None, n: int | None = None):
        """``root``: only that rank passes the global ``a0`` (the others pass
        None and the order ``n``); it is scattered by column blocks
        (scatter_input). Otherwise every rank passes the same ``a0``."""
        import torch
        import torch.distributed as dist
        self.kind = DecompositionKind(_value(kind))
        if root is not None and a0 is None:
            if n is None:
                raise ERRORS["dim"]("the order n is required on non-root ranks")
        else:
            n = a0.shape[0]
            if a0.ndim != 2 or a0.shape != (n, n):
                raise ERRORS["dim"]("square input required")
        self.n, self.b = n, int(b)
        self.layout = BlockLayout(n, self.b)
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.device = torch.cuda.current_device() if device is None else int(device)
        lib = _lib.load()
        self._lib = lib
        ctx = ctypes.c_void_p()
        check(lib.abft_dist_create(ctypes.byref(ctx), _lib.KIND_CODE[self.kind.value], n, self.b,
                                   self.device, self.rank, self.world))
        self._ctx = ctx
        if keep_input:  # device copy of the local input for reset()
            check(lib.abft_dist_keep_input(ctx, 1))
        if root is not None:
            self.local_input = scatter_input(a0, n, self.b, group, root, self.device)
            check(lib.abft_dist_set_local(ctx, _lib.dptr(self.local_input), n))
        else:
            host = np.asfortranarray(np.asarray(a0, dtype=np.float64))
            check(lib.abft_dist_set_matrix(ctx, _lib.dptr(host), n))
            self.local_input = None
        self.ncl = int(lib.abft_dist_local_cols(ctx))
        dev = torch.device("cuda", self.device)
        cap = max(int(lib.abft_dist_xbuf_elems(ctx, k)) for k in range(self.layout.n_blocks))
        # two exchange buffers: panel k is consumed while panel k+1 is broadcast
        self._bufs = [torch.zeros(max(cap, 1), dtype=torch.float64, device=dev) for _ in range(2)]
        self._xbuf = self._bufs[0]
        self._scale = torch.zeros(2, dtype=torch.float64, device=dev)
        self._tx = _Transport(group, lib.abft_dist_stream(ctx), self.device,
                              lib.abft_dist_comm_stream(ctx))
        self.lookahead = os.environ.get("ABFT_NO_LOOKAHEAD") != "1"
        self.force_lookahead = False  # exercise the look-ahead machinery on one rank (tests)
        self._prefetched = set()

    def __del__(self):
        ctx = getattr(self, "_ctx", None)
        if ctx:
            try:
                self._lib.abft_dist_destroy(ctx)
            except Exception:
                pass
            self._ctx = None

    @property
    def k_done(self) -> int:
        return int(self._lib.abft_dist_k_done(self._ctx))

    def set_matrix(self, a: np.ndarray) -> None:
        """Load a new global input (owned column blocks are copied)."""
        host = a if a.flags.f_contiguous else np.asfortranarray(a, dtype=np.float64)
        self._prefetched.clear()
        check(self._lib.abft_dist_set_matrix(self._ctx, _lib.dptr(host), self.n))

    def reset(self) -> None:
        """Restore the kept input on the device (needs keep_input=True)."""
        self._prefetched.clear()
        check(self._lib.abft_dist_reset(self._ctx))

    def stream_ptr(self) -> int:
        return int(self._lib.abft_dist_stream(self._ctx))

    @property
    def complete(self) -> bool:
        return self.k_done >= self.layout.n_blocks

    # -- one iteration (asynchronous; events are drained by _drain) ----------
    def _iterate(self, k: int, scheme: str, plan: list, correct: bool) -> None:
        lib, ctx = self._lib, self._ctx
        code = _lib.SCHEME_CODE[scheme]
        xe = int(lib.abft_dist_xbuf_elems(ctx, k))
        buf = self._bufs[k % 2]
        xptr = buf.data_ptr()
        check(lib.abft_dist_begin(ctx, k, code, ctypes.c_void_p(xptr)))
        root = ctypes.c_int(0)
        op = int(lib.abft_dist_exchange(ctx, k, ctypes.byref(root)))
        if xe > 0 and op and k not in self._prefetched:
            view = buf[:xe]
            if op == 2:  # left-looking Cholesky: partial panel products
                self._tx.reduce_sum(view, root.value)
            else:        # the panel (LU / QR: k; right-looking Cholesky: k-1)
                self._tx.broadcast(view, root.value)
        self._prefetched.discard(k)
        nplan = len(plan)
        # look-ahead: the next exchanged panel (LU / QR: panel k+1; right-looking
        # Cholesky: panel k) is factored mid-update by its owner and broadcast
        # on the comm stream while the trailing update of k runs
        nb = self.layout.n_blocks
        xe1 = int(lib.abft_dist_xbuf_elems(ctx, k + 1)) if k + 1 < nb else 0
        root1 = ctypes.c_int(0)
        op1 = int(lib.abft_dist_exchange(ctx, k + 1, ctypes.byref(root1))) if k + 1 < nb else 0
        la = (self.lookahead and (self.world > 1 or self.force_lookahead)
              and op1 == 1 and nplan == 0 and xe1 > 0)
        nxt = self._bufs[(k + 1) % 2]
        if la:
            check(lib.abft_dist_lookahead(ctx, k, ctypes.c_void_p(nxt.data_ptr())))
        sptr = ctypes.c_void_p(self._scale.data_ptr())
        check(lib.abft_dist_update(ctx, k, code, ctypes.c_void_p(xptr), nplan,
                                   sptr if nplan else None))
        if la:
            self._tx.broadcast(nxt[:xe1], root1.value, comm=True)
            check(lib.abft_dist_comm_done(ctx))
            self._prefetched.add(k + 1)
        if nplan:
            self._tx.allreduce_max(self._scale[:1])
        arr = _plan_structs(plan)
        check(lib.abft_dist_finish(ctx, k, code, arr, nplan, int(bool(correct)),
                                   sptr if nplan else None))

    def _drain(self) -> list:
        """Synchronize; gather and merge every rank's events (all ranks)."""
        import torch.distributed as dist
        cap = 1 << 16
        locs = (_lib.Location * cap)()
        iters = (ctypes.c_int64 * cap)()
        nout = ctypes.c_int(0)
        rc = self._lib.abft_dist_events(self._ctx, locs, iters, cap, ctypes.byref(nout))
        msg = _lib.last_error() if rc else ""
        evs = []
        for i in range(min(nout.value, cap)):
            L = locs[i]
            evs.append({"iter": int(iters[i]), "block_row": int(L.block_row),
                        "block_col": int(L.block_col), "seq": int(L.seq), "row": int(L.row),
                        "col": int(L.col), "kind": int(L.kind), "flag": int(L.flag),
                        "detected_kind": int(L.detected_kind), "corrected": int(L.corrected),
                        "uncorrectable": int(L.uncorrectable)})
        gathered = [None] * self.world
        dist.all_gather_object(gathered, (rc, msg, evs), group=self.group)
        for grc, gmsg, _ in gathered:
            if grc != 0:
                _lib_raise(grc, gmsg)
        return merge_events([g[2] for g in gathered])

    # -- reference-shaped drivers -------------------------------------------
    def run_numeric_iteration(self, k: int, scheme, fault_counts: dict | None = None,
                              rng: np.random.Generator | None = None,
                              correct: bool = True) -> CorrectionReport:
        """simulator.py:97-121 for iteration k, distributed."""
        sch = ChecksumScheme(_value(scheme)).value
        r0, c0, rows, cols = _tmu_region(self.kind, self.n, self.b, k)
        plan = []
        if rows > 0 and cols > 0 and fault_counts and any(fault_counts.values()):
            plan = draw_plan(rng, fault_counts, r0, c0, rows, cols, self.b)
        self._iterate(k, sch, plan, correct)
        return reports_from_events(self._drain(), k, k + 1)[0]

    def run_protected(self, scheme, fault_schedule: dict | None = None,
                      rng: np.random.Generator | None = None, correct: bool = True,
                      schemes: list | None = None) -> list:
        """All remaining iterations (simulator.run_protected semantics): one
        CorrectionReport per iteration, identical on every rank. The host
        loop only enqueues work; it synchronizes once at the end."""
        nb, k0 = self.layout.n_blocks, self.k_done
        self._prefetched.clear()
        for k in range(k0, nb):
            sch = ChecksumScheme(_value(schemes[k] if schemes is not None else scheme)).value
            counts = (fault_schedule or {}).get(k)
            r0, c0, rows, cols = _tmu_region(self.kind, self.n, self.b, k)
            plan = []
            if rows > 0 and cols > 0 and counts and any(counts.values()):
                plan = draw_plan(rng, counts, r0, c0, rows, cols, self.b)
            self._iterate(k, sch, plan, correct)
        return reports_from_events(self._drain(), k0, nb)

    def elapsed_ms(self) -> float:
        v = ctypes.c_double(0.0)
        check(self._lib.abft_dist_elapsed_ms(self._ctx, ctypes.byref(v)))
        return float(v.value)

    # -- results -----------------------------------------------------------------
    def local_matrix(self) -> np.ndarray:
        out = np.empty((self.n, self.ncl), order="F")
        check(self._lib.abft_dist_get_matrix(self._ctx, _lib.dptr(out), self.n))
        return out

    def gather(self, dst: int = 0) -> np.ndarray | None:
        """The packed factor on rank `dst` (None elsewhere)."""
        import torch
        import torch.distributed as dist
        width = max(local_columns(self.n, self.b, r, self.world) for r in range(self.world))
        loc = np.zeros((width, self.n))       # row-major rows = local columns
        loc[:self.ncl] = self.local_matrix().T
        dev = torch.device("cuda", self.device) if self._tx.native else torch.device("cpu")
        t = torch.from_numpy(loc).to(dev)
        gl = self._tx._global(dst)
        if self.rank == dst:
            bufs = [torch.empty_like(t) for _ in range(self.world)]
            dist.gather(t, bufs, dst=gl, group=self.group)
            parts = []
            for r, bt in enumerate(bufs):
                ncl = local_columns(self.n, self.b, r, self.world)
                parts.append(np.asfortranarray(bt.cpu().numpy()[:ncl].T))
            return assemble_columns(parts, self.n, self.b)
        dist.gather(t, None, dst=gl, group=self.group)
        return None

    def residual(self, a0: np.ndarray) -> float:
        """residual(a, factors) (linalg.py:362-368): the factor is gathered
        to rank 0's GPU (8.6 GB fits one B200 at N=32768, §8e) and the
        reconstruction runs on the single-GPU path; the value is broadcast."""
        import torch.distributed as dist
        full = self.gather(0)
        val = [None]
        if self.rank == 0:
            lib = self._lib
            ctx = ctypes.c_void_p()
            check(lib.abft_create(ctypes.byref(ctx), _lib.KIND_CODE[self.kind.value], self.n,
                                  self.b, self.device))
            try:
                check(lib.abft_set_matrix(ctx, _lib.dptr(full), self.n))
                check(lib.abft_set_k_done(ctx, self.layout.n_blocks))
                if self.kind == DecompositionKind.QR:
                    for k in range(self.layout.n_blocks):
                        p = k * self.b
                        w = min(p + self.b, self.n) - p
                        V = np.zeros((self.n - p, w), order="F")
                        T = np.zeros((w, w), order="F")
                        check(lib.abft_dist_get_qr_panel(self._ctx, k, _lib.dptr(V), self.n - p,
                                                         _lib.dptr(T), w))
                        check(lib.abft_set_qr_panel(ctx, k, _lib.dptr(V), self.n - p,
                                                    _lib.dptr(T), w))
                host = np.asfortranarray(np.asarray(a0, dtype=np.float64))
                out = ctypes.c_double(0.0)
                check(lib.abft_residual(ctx, _lib.dptr(host), self.n, ctypes.byref(out)))
                val[0] = float(out.value)
            finally:
                lib.abft_destroy(ctx)
        dist.broadcast_object_list(val, src=self._tx._global(0), group=self.group)
        return float(val[0])


def _lib_raise(rc: int, msg: str) -> None:
    if rc == _lib.E_DIM:
        raise ERRORS["dim"](msg)
    if rc in (_lib.E_BREAKDOWN, _lib.E_INCOMPLETE):
        raise ERRORS["breakdown"](msg)
    if rc == _lib.E_RANGE:
        raise IndexError(msg)
    if rc == _lib.E_INVALID:
        raise ValueError(msg)
    raise RuntimeError(f"libabft_b200 error {rc}: {msg}")
