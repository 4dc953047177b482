import sys, numpy as np
sys.path.insert(0, ".")
import paper_2301_03166_b200 as P
kind = sys.argv[1] if len(sys.argv) > 1 else "cholesky"
for seed in (2,):
    a = P.generate_test_matrix(kind, 256, seed)
    f = P.Factorization(kind, a, 32)
    rng = np.random.default_rng(seed)
    for k in range(8):
        P.run_numeric_iteration(f, k, "single", {"0d": 1} if k == 2 else None, rng)
    print(kind, "residual", P.residual(a, f))
