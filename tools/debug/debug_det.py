import sys, numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import oracle as O, paper_2301_03166_b200 as P
from conftest import report_json
def run(kind, scheme, seed, n, b, with_oracle):
    counts = {"0d": 2, "1d": 1, "2d": 1}
    rng = np.random.default_rng(seed); nb = -(-n // b); kf = int(rng.integers(0, nb - 1))
    a = P.generate_test_matrix(kind, n, seed); f = P.Factorization(kind, a, b)
    if with_oracle:
        rng_o = np.random.default_rng(seed); rng_o.integers(0, nb - 1); fo = O.OracleFactorization(kind, a, b)
    ms, reps = [], []
    for k in range(nb):
        c = counts if k == kf else None
        reps.append(report_json(P.run_numeric_iteration(f, k, scheme, c, rng)))
        ms.append(f.m.copy())
        if with_oracle:
            ro = O.protected_iteration(fo, k, scheme, c, rng_o).to_json()
            d = np.abs(f.m - fo.m)
            cb = [float(d[:, j*b:(j+1)*b].max()) for j in range(nb)]
            print(f"  k={k} kf={kf} {'ok ' if reps[-1]==ro else 'MISMATCH'} max diff per col block", ["%.0e" % x for x in cb])
            if reps[-1] != ro: print("   gpu", reps[-1], "\n   orc", ro)
    return ms, reps
for seed in range(8):
    m1, r1 = run("cholesky", "single", seed, 256, 32, False)
    m2, r2 = run("cholesky", "single", seed, 256, 32, False)
    same = all(np.array_equal(x, y) for x, y in zip(m1, m2))
    print("seed", seed, "bitwise deterministic:", same, "reports equal:", r1 == r2)
    if not same:
        for k, (x, y) in enumerate(zip(m1, m2)):
            if not np.array_equal(x, y):
                idx = np.argwhere(x != y); print("  first diff at iteration", k, "entries", idx[:5].tolist(), len(idx)); break
for seed in range(8):
    print("oracle compare seed", seed); run("cholesky", "single", seed, 256, 32, True)
