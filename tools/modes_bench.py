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
ap.add_argument("--rate-scale", type=float, default=2e3,
                help="fault-rate scale of the forced-scheme campaign runs")
ap.add_argument("--sweep", action="store_true")
ap.add_argument("--precision", default="f64", choices=["f64", "f32"])
ap.add_argument("--engine", default="iteration", choices=["iteration", "stream"],
                help="stream: the modes on the look-ahead path with the SM-split lever")
ap.add_argument("--repeat", type=int, default=10,
                help="factorizations per configuration (NVML energy counter resolution)")
args = ap.parse_args()
a = P.generate_test_matrix(args.kind, args.n, args.seed)
G.run_mode(args.kind, a, args.b, "original", seed=args.seed, precision=args.precision,
           engine=args.engine)  # warm-up
# (mode, r, forced scheme, rate scale): the reference's rates for the mode
# comparison and the r sweep; forced-scheme campaign runs with scaled rates
runs = [(m, 0.5, None, 1.0) for m in G.MODES]
if args.sweep:
    runs += [("bsr", r, None, 1.0) for r in (0.0, 0.25, 0.75, 1.0)]
    if args.precision == "f32":  # C5: the full reclamation-ratio sweep r = 0..1
        runs += [("bsr", round(0.05 * i, 2), None, 1.0) for i in range(21) if i % 5]
    runs += [("bsr", 1.0, sch, args.rate_scale) for sch in ("none", "single", "full")]
nv = G._Energy(0)
for mode, r, forced, scale in runs:
    e0 = nv.mj()
    for _ in range(args.repeat):
        s, recs = G.run_mode(args.kind, a, args.b, mode, r=r, seed=args.seed,
                             rates=G.scaled_rate_table(scale), forced_scheme=forced,
                             recovery="continue" if forced == "none" else "recompute",
                             precision=args.precision, engine=args.engine)
    e1 = nv.mj()
    d = dataclasses.asdict(s)
    d["energy_j"] = (e1 - e0) / 1e3 / args.repeat if e0 is not None and e1 is not None else None
    d["energy_note"] = f"NVML TotalEnergyConsumption over {args.repeat} factorizations (incl. host gaps)"
    d["rate_scale"] = scale
    d["forced_scheme"] = forced
    d["precision"] = args.precision
    d["f_gpu_mhz"] = [rc.f_gpu_mhz for rc in recs]
    d["abft_modes"] = "".join(rc.abft_mode[0] for rc in recs)
    d["engine"] = args.engine
    d["side_sms"] = [rc.side_sms for rc in recs]
    print(json.dumps(d), flush=True)
