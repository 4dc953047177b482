import sys, numpy as np
sys.path.insert(0, ".")
import oracle as O, paper_2301_03166_b200 as P
sys.path.insert(0, "tests"); from conftest import report_json
kind, scheme, seed, n, b = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
counts = {"0d": 2, "1d": 1, "2d": 1}
rng = np.random.default_rng(seed); rng_o = np.random.default_rng(seed)
nb = -(-n // b); kf = int(rng.integers(0, nb - 1)); rng_o.integers(0, nb - 1)
a = P.generate_test_matrix(kind, n, seed)
f = P.Factorization(kind, a, b); fo = O.OracleFactorization(kind, a, b)
for k in range(nb):
    c = counts if k == kf else None
    r = report_json(P.run_numeric_iteration(f, k, scheme, c, rng))
    ro = O.protected_iteration(fo, k, scheme, c, rng_o).to_json()
    diff = np.abs(f.m - fo.m)
    print(k, "match" if r == ro else f"MISMATCH\n gpu {r}\n orc {ro}", "max|m-m_o| %.2e" % diff.max())
    if diff.max() > 1e-8:
        idx = np.argwhere(diff > 1e-8); print("  bad entries:", idx[:10].tolist(), len(idx))
