"""Run-mode measurements on one B200 (SURVEY §8d configs C2 and C5-style
sweeps): LU N=8192 original vs r2h vs sr vs bsr, and a bsr reclamation-ratio
sweep, with measured task times and NVML energy. One JSON line per run."""
import argparse
import dataclasses
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2301_03166_b200 as P
from paper_2301_03166_b200 import governor as G

ap = argparse.ArgumentParser()
ap.add_argument("--kind", default="lu")
ap.add_argument("--n", type=int, default=8192)
ap.add_argument("--b", type=int, default=256)
ap.add_argument("--seed", type=int, default=0)
ap.add_argument("--rate-scale", type=float, default=2e4)
ap.add_argument("--sweep", action="store_true")
args = ap.parse_args()
a = P.generate_test_matrix(args.kind, args.n, args.seed)
table = G.scaled_rate_table(args.rate_scale)
G.run_mode(args.kind, a, args.b, "original", seed=args.seed)  # warm-up
runs = [(m, 0.5) for m in G.MODES]
if args.sweep:
    runs += [("bsr", r) for r in (0.0, 0.25, 0.5, 0.75, 1.0)]
for mode, r in runs:
    s, recs = G.run_mode(args.kind, a, args.b, mode, r=r, seed=args.seed, rates=table)
    d = dataclasses.asdict(s)
    d["rate_scale"] = args.rate_scale
    d["f_gpu_mhz"] = [rc.f_gpu_mhz for rc in recs]
    d["abft_modes"] = "".join(rc.abft_mode[0] for rc in recs)
    print(json.dumps(d), flush=True)
