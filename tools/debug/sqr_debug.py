import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_2301_03166_b200 as P
for n, b in ((512, 128), (1024, 128), (2048, 128), (4096, 128)):
    a = P.generate_test_matrix("qr", n, 1)
    for scheme in ("none", "full"):
        f = P.SFactorization("qr", a, b)
        f.run_protected(scheme)
        r = f.residual(a)
        m = f.m
        _, rr = np.linalg.qr(a)
        dr = np.max(np.abs(np.abs(np.diag(m)) - np.abs(np.diag(rr))) / np.abs(np.diag(rr)))
        f64 = P.Factorization("qr", a, b).run_all()
        print(n, scheme, "res %.2e" % r, "diagR rel %.2e" % dr, "|R32-R64| %.2e" % np.max(np.abs(np.triu(m) - np.triu(f64.m))), flush=True)
