import sys, numpy as np
sys.path.insert(0, ".")
import oracle as O, paper_2301_03166_b200 as P
kind = sys.argv[1]; n = int(sys.argv[2]); b = int(sys.argv[3]); reps = int(sys.argv[4])
a = P.generate_test_matrix(kind, n, 1)
fails = {}
for rep in range(reps):
    f = P.Factorization(kind, a, b); fo = O.OracleFactorization(kind, a, b)
    for k in range(f.layout.n_blocks):
        for task in [t.value for t in f.task_order()]:
            getattr(f, "task_" + task)(k); getattr(fo, task)(k)
            d = np.abs(f.m - fo.m).max()
            if d > 1e-10:
                key = (k, task); fails[key] = fails.get(key, 0) + 1
                if fails[key] == 1:
                    idx = np.argwhere(np.abs(f.m - fo.m) > 1e-10)
                    print(f"rep {rep} k={k} task={task} maxdiff {d:.2e} rows {idx[:,0].min()}..{idx[:,0].max()} cols {idx[:,1].min()}..{idx[:,1].max()} n_bad {len(idx)}")
                f = None
                break
        if f is None: break
        f.k_done = k + 1
print(kind, "failures:", fails)
