"""Worker processes for the multi-rank tests (spawned, one per rank).

GPU mode: every rank drives the sm_100a library on cuda:0 (the test boxes
have one GPU) with the gloo backend — the same DistributedFactorization code
the NCCL path runs, with the exchange staged through host memory.
CPU mode: only the host-side logic (event merge over all_gather_object).
"""
from __future__ import annotations

import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def _init(rank: int, world: int, init_file: str):
    import torch.distributed as dist
    os.environ.setdefault("GLOO_SOCKET_IFNAME", "lo")
    dist.init_process_group("gloo", init_method=f"file://{init_file}", rank=rank,
                            world_size=world)
    return dist


def gpu_cases(rank: int, world: int, init_file: str, cases: list, out: str) -> None:
    import numpy as np
    import torch
    torch.cuda.set_device(0)
    dist = _init(rank, world, init_file)
    import paper_2301_03166_b200 as P
    from paper_2301_03166_b200.distributed import DistributedFactorization
    results = []
    for c in cases:
        a = P.generate_test_matrix(c["kind"], c["n"], c["seed"])
        root = c.get("root")  # input only on this rank, scattered by column blocks
        if c.get("chol_left"):  # the reference's left-looking form (sum-reduce exchange)
            os.environ["ABFT_DIST_CHOL"] = "left"
        if root is not None:
            f = DistributedFactorization(c["kind"], a if rank == root else None, c["b"],
                                         keep_input=bool(c.get("reset")), root=root, n=c["n"])
        else:
            f = DistributedFactorization(c["kind"], a, c["b"], keep_input=bool(c.get("reset")))
        os.environ.pop("ABFT_DIST_CHOL", None)
        f.lookahead = not c.get("no_lookahead", False)
        if c.get("reset"):  # a throw-away factorization, then restore the kept input
            f.run_protected("none", {}, None)
            f.reset()
        rng = np.random.default_rng(c["seed"])
        sched = {int(k): v for k, v in c.get("schedule", {}).items()}
        if c.get("per_iteration"):
            reps = [f.run_numeric_iteration(k, c["scheme"], sched.get(k), rng)
                    for k in range(f.layout.n_blocks)]
        else:
            reps = f.run_protected(c["scheme"], sched, rng)
        locs = [[(int(r), int(cc), getattr(kk, "value", kk), bool(fl))
                 for r, cc, kk, fl in rep.locations] for rep in reps]
        res = f.residual(a)
        full = f.gather(0)
        if rank == 0:
            np.save(os.path.join(out, f"{c['name']}.npy"), full)
        results.append({"name": c["name"], "locations": locs, "residual": res,
                        "detected": [{getattr(k, "value", k): v for k, v in r.detected.items()}
                                     for r in reps],
                        "uncorrectable": [bool(r.uncorrectable) for r in reps]})
        del f
    with open(os.path.join(out, f"rank{rank}.json"), "w") as fh:
        json.dump(results, fh)
    dist.barrier()
    dist.destroy_process_group()


def cpu_merge(rank: int, world: int, init_file: str, out: str) -> None:
    dist = _init(rank, world, init_file)
    from paper_2301_03166_b200.distributed import merge_events, reports_from_events
    # each rank owns different block columns of the same iterations
    mine = [{"iter": k, "block_row": br, "block_col": bc, "seq": s, "row": 10 * br + s,
             "col": 100 * bc + s, "kind": 0, "flag": 1, "detected_kind": 0, "corrected": 1,
             "uncorrectable": 0}
            for k in range(3) for br in range(2) for bc in range(rank, 4, world) for s in range(2)]
    gathered = [None] * world
    dist.all_gather_object(gathered, mine)
    merged = merge_events(gathered)
    reps = reports_from_events(merged, 0, 3)
    with open(os.path.join(out, f"rank{rank}.json"), "w") as fh:
        json.dump({"order": [(e["iter"], e["block_row"], e["block_col"], e["seq"]) for e in merged],
                   "counts": [sum(r.detected.values()) for r in reps],
                   "locations": [r.locations for r in reps]}, fh, default=str)
    dist.barrier()
    dist.destroy_process_group()


def cpu_scatter(rank: int, world: int, init_file: str, out: str) -> None:
    """scatter_input over gloo: only the root holds the global matrix."""
    import numpy as np
    dist = _init(rank, world, init_file)
    from paper_2301_03166_b200.distributed import scatter_columns, scatter_input
    n, b, root = 70, 16, world - 1
    a = np.asfortranarray(np.arange(n * n, dtype=np.float64).reshape(n, n)) if rank == root else None
    local = scatter_input(a, n, b, None, root)
    ref = scatter_columns(np.asfortranarray(np.arange(n * n, dtype=np.float64).reshape(n, n)), b,
                          rank, world)
    with open(os.path.join(out, f"rank{rank}.json"), "w") as fh:
        json.dump({"ok": bool(local.shape == ref.shape and np.array_equal(local, ref)),
                   "fortran": bool(local.flags.f_contiguous)}, fh)
    dist.barrier()
    dist.destroy_process_group()


def nccl_single(rank: int, world: int, init_file: str, out: str) -> None:
    """World-size-1 NCCL group: the native transport (device tensors on the
    context / comm streams) and the look-ahead machinery against the
    single-GPU path, bit for bit."""
    import numpy as np
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"file://{init_file}", rank=rank,
                            world_size=world, device_id=torch.device("cuda", 0))
    import paper_2301_03166_b200 as P
    from paper_2301_03166_b200.distributed import DistributedFactorization
    res = {}
    for kind in ("lu", "qr", "cholesky"):
        n, b, seed = 768, 128, 13
        a = P.generate_test_matrix(kind, n, seed)
        sched = {1: {"0d": 1}, 3: {"0d": 1}}
        f = DistributedFactorization(kind, a, b)
        f.force_lookahead = True
        reps = f.run_protected("full", sched, np.random.default_rng(seed))
        full = f.gather(0)
        f1 = P.Factorization(kind, a, b)
        reps1 = P.run_protected(f1, "full", sched, np.random.default_rng(seed))
        res[kind] = {
            "same_reports": [r.locations for r in reps] == [r.locations for r in reps1],
            "max_diff": float(np.max(np.abs(full - f1.m))),
            "residual": f.residual(a),
            "residual1": P.residual(a, f1),
        }
    import json
    with open(os.path.join(out, "nccl.json"), "w") as fh:
        json.dump(res, fh, default=str)
    dist.barrier()
    dist.destroy_process_group()


def breakdown(rank: int, world: int, init_file: str, out: str) -> None:
    """A zero pivot in a panel owned by rank 1 surfaces as the reference's
    NumericBreakdownError on every rank (linalg.py:234-235)."""
    import torch
    torch.cuda.set_device(0)
    dist = _init(rank, world, init_file)
    import paper_2301_03166_b200 as P
    from paper_2301_03166_b200.distributed import DistributedFactorization
    a = P.generate_test_matrix("lu", 256, 0)
    a[70, 70] = 0.0
    a[70, :] = 0.0  # row 70 identically zero: the pivot of column 70 (panel 1) is 0
    f = DistributedFactorization("lu", a, 64)
    try:
        f.run_protected("full")
        res = "no error"
    except P.NumericBreakdownError as e:
        res = f"NumericBreakdownError: {e}"
    except Exception as e:  # noqa: BLE001
        res = f"{type(e).__name__}: {e}"
    with open(os.path.join(out, f"brk{rank}.txt"), "w") as fh:
        fh.write(res)
    dist.barrier()
    dist.destroy_process_group()
