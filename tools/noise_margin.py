"""Threshold margins of the ABFT checks on the B200 path (diagnostic).

(1) Clean runs: the largest |delta| / tau among checks that did not trip
    (abft_noise_stats), per kind / precision / size and scheme. A value well
    below 1 is the false-positive margin of the threshold rule.
(2) Detection sweep: criterion-5 protocol (k_fault = rng.integers(0, nb - 1),
    one 0-D fault) over many seeds; every fault must be located at its
    planned (row, col) and corrected.

usage: python tools/noise_margin.py [--out gpurun_out/noise.jsonl] [--quick]
"""
from __future__ import annotations

import argparse
import copy
import ctypes
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2301_03166_b200 as P  # noqa: E402
from paper_2301_03166_b200 import _lib  # noqa: E402
from paper_2301_03166_b200.abft import draw_plan  # noqa: E402
from paper_2301_03166_b200.simulator import _tmu_region  # noqa: E402


def noise_read(lib, reset=True):
    out = (ctypes.c_double * 4)()
    assert lib.abft_noise_read(out, int(reset)) == 0
    return [float(x) for x in out]


def make(precision, kind, n, b, a):
    if precision == "f32":
        return P.SFactorization(kind, a, b)
    return P.Factorization(kind, a, b)


def run_all(f, precision, scheme, sched, rng):
    if precision == "f32":
        return f.run_protected(scheme, sched, rng)
    return P.run_protected(f, scheme, sched, rng)


def clean(lib, precision, kind, n, b, seed, out):
    a = P.generate_test_matrix(kind, n, seed)
    for scheme in ("full", "single"):
        f = make(precision, kind, n, b, a)
        noise_read(lib)
        t = time.time()
        reps = run_all(f, precision, scheme, None, np.random.default_rng(seed))
        stats = noise_read(lib)
        nev = sum(len(r.locations) for r in reps)
        rec = {"test": "clean", "precision": precision, "kind": kind, "n": n, "b": b,
               "scheme": scheme, "events": nev, "max_dcol_over_tau": stats[0],
               "max_drow_over_tau": stats[1], "max_dw_over_tau": stats[2],
               "s": round(time.time() - t, 2)}
        print(json.dumps(rec), flush=True)
        out.write(json.dumps(rec) + "\n")
        del f


def sweep(lib, precision, kind, n, b, seeds, out):
    a_cache = {}
    for scheme in ("full", "single"):
        ok = total = 0
        misses, snaps = [], []
        for seed in seeds:
            if seed not in a_cache:
                a_cache[seed] = P.generate_test_matrix(kind, n, seed)
            a = a_cache[seed]
            nb = -(-n // b)
            rng = np.random.default_rng(seed)
            k_fault = int(rng.integers(0, nb - 1))
            r0, c0, rows, cols = _tmu_region(P.DecompositionKind(kind), n, b, k_fault)
            if rows <= 0 or cols <= 0:
                continue
            plan = draw_plan(copy.deepcopy(rng), {P.ErrorKind.D0: 1}, r0, c0, rows, cols, b)
            want = (plan[0]["row"], plan[0]["col"])
            f = make(precision, kind, n, b, a)
            noise_read(lib)
            reps = run_all(f, precision, scheme, {k_fault: {P.ErrorKind.D0: 1}}, rng)
            snap = noise_read(lib)[3]
            locs = [(r, c, kk.value, fl) for rep in reps for r, c, kk, fl in rep.locations]
            total += 1
            if locs == [(want[0], want[1], "0d", True)]:
                ok += 1
                if scheme == "single":
                    snaps.append(snap)
            else:
                misses.append({"seed": seed, "k": k_fault, "want": want, "got": locs[:4],
                               "snap_distance": snap})
            del f
        rec = {"test": "detect", "precision": precision, "kind": kind, "n": n, "b": b,
               "scheme": scheme, "runs": total, "located_and_corrected": ok,
               "misses": misses[:10],
               "snap_distance_located": (np.percentile(snaps, [50, 90, 99, 100]).tolist()
                                         if snaps else None)}
        print(json.dumps(rec), flush=True)
        out.write(json.dumps(rec) + "\n")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/noise.jsonl")
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--what", default="clean,sweep")
    ap.add_argument("--seeds", type=int, default=100)
    ap.add_argument("--kinds", default="lu,cholesky,qr")
    ap.add_argument("--sweep-n", type=int, default=2048)
    args = ap.parse_args()
    lib = _lib.load()
    assert lib.abft_noise_stats(1) == 0
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    what = args.what.split(",")
    with open(args.out, "a") as out:
        if "clean" in what:
            sizes = [("f32", 4096, 128)] if args.quick else [("f32", 16384, 128), ("f64", 16384, 256)]
            for precision, n, b in sizes:
                for kind in ("lu", "cholesky", "qr"):
                    clean(lib, precision, kind, n, b, 0, out)
        if "sweep" in what:
            nseeds = 8 if args.quick else args.seeds
            for kind in args.kinds.split(","):
                sweep(lib, "f32", kind, args.sweep_n, 128, range(nseeds), out)
        if "big" in what:
            for kind in ("lu", "cholesky", "qr"):
                sweep(lib, "f32", kind, 16384, 128, range(3), out)


if __name__ == "__main__":
    main()
