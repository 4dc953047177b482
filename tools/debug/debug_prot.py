import sys, numpy as np
sys.path.insert(0, ".")
import oracle as O, paper_2301_03166_b200 as P
kind = sys.argv[1]; n = int(sys.argv[2]); b = int(sys.argv[3]); reps = int(sys.argv[4])
a = P.generate_test_matrix(kind, n, 1)
fo_ms = []
fo = O.OracleFactorization(kind, a, b)
for k in range(fo.nb):
    O.protected_iteration(fo, k, "none"); fo_ms.append(fo.m.copy())
for scheme in ("none", "single", "full"):
    fails = {}
    for rep in range(reps):
        f = P.Factorization(kind, a, b)
        for k in range(f.layout.n_blocks):
            r = P.run_numeric_iteration(f, k, scheme)
            d = np.abs(f.m - fo_ms[k])
            if d.max() > 1e-10 or not r.clean:
                fails[k] = fails.get(k, 0) + 1
                if sum(fails.values()) <= 3:
                    idx = np.argwhere(d > 1e-10)
                    print(f" {scheme} rep {rep} k={k} maxdiff {d.max():.2e} clean={r.clean} rows {idx[:,0].min() if len(idx) else -1}..{idx[:,0].max() if len(idx) else -1} cols {idx[:,1].min() if len(idx) else -1}..{idx[:,1].max() if len(idx) else -1} nbad {len(idx)}")
                break
    print(kind, scheme, "failures by k:", fails)
