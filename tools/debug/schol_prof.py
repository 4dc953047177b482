"""Per-iteration bracket times of the fp32 Cholesky per-iteration path
(diagnoses run-mode device_ms variance)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_2301_03166_b200 as P
from paper_2301_03166_b200 import governor as G
from paper_2301_03166_b200.single import SFactorization

kind = sys.argv[1] if len(sys.argv) > 1 else "cholesky"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
a = P.generate_test_matrix(kind, n, 0)
for rep in range(3):
    f = SFactorization(kind, a, 128)
    G._profile_enable(f, True)
    tot = np.zeros(4)
    rows = []
    t0 = time.perf_counter()
    for k in range(f.layout.n_blocks):
        b0 = G._profile(f)
        th = time.perf_counter()
        f.run_numeric_iteration(k, "none")
        th = time.perf_counter() - th
        d = np.array(G._profile(f)) - np.array(b0)
        tot += d
        rows.append((k, *d, th * 1e3))
    wall = time.perf_counter() - t0
    print(f"rep {rep}: brackets pd/pu/tmu/abft = {tot.round(2)} sum {tot.sum():.1f} ms wall {wall*1e3:.1f} ms")
    rows.sort(key=lambda r: -sum(r[1:5]))
    for r in rows[:6]:
        print("   k=%d pd %.2f pu %.2f tmu %.2f abft %.2f host %.2f" % r)
