import sys, ctypes, json, numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import oracle as O, paper_2301_03166_b200 as P
from paper_2301_03166_b200 import _lib
from conftest import report_json, sparse_reports, golden
def arr(f, which):
    r = ctypes.c_int64(); c = ctypes.c_int64()
    _lib.load().abft_debug_array(f._ctx, which, None, ctypes.byref(r), ctypes.byref(c))
    out = np.zeros((r.value, c.value), order="F")
    _lib.load().abft_debug_array(f._ctx, which, _lib.dptr(out), ctypes.byref(r), ctypes.byref(c))
    return out
runs = golden("multi.json")["runs"]
for run in runs:
    kind, scheme, seed, n, b = run["kind"], run["scheme"], run["seed"], run["n"], run["b"]
    rng = np.random.default_rng(seed); nb = -(-n // b); kf = int(rng.integers(0, nb - 1))
    a = P.generate_test_matrix(kind, n, seed); f = P.Factorization(kind, a, b)
    reps = []
    for k in range(nb):
        c = run["counts"] if k == kf else None
        rep = report_json(P.run_numeric_iteration(f, k, scheme, c, rng))
        reps.append(rep)
        want = dict((kk, r) for kk, r in run["reports"]).get(k, {"detected": {"0d": 0, "1d": 0, "2d": 0}, "corrected": {"0d": 0, "1d": 0, "2d": 0}, "uncorrectable": False, "locations": []})
        if rep != want:
            print("MISMATCH", kind, scheme, seed, n, b, "k", k)
            print(" gpu", rep); print(" ref", want, "k_fault", kf)
            g = arr(f, 0); cs = arr(f, 1); gm = arr(f, 4)
            r0 = k * b
            print(" gcsw rows 2k.. cols p..pe (plain):", g[2*k:2*nb:2, r0:r0+4])
            print(" csm  rows (plain):", cs[0:2*(nb-k):2, 0:4])
            print(" gmax:", gm[k:, k])
            sys.exit(0)
print("no mismatch")
