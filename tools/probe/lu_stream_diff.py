"""Where does the chunked streamed LU differ from the iteration-ordered one?"""
import ctypes, os, sys
import numpy as np
import paper_2301_03166_b200 as P

KIND = sys.argv[1] if len(sys.argv) > 1 else "lu"

n, b = 2048, 128
nb = n // b


def run(streamed, sched, scheme="full"):
    a = P.generate_test_matrix(KIND, n, 7)
    f = P.Factorization(KIND, a, b)
    if streamed:
        af = np.asfortranarray(a)
        assert f._lib.abft_set_matrix_streamed(f._ctx, af.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), n) == 0
    P.run_protected(f, scheme, sched, np.random.default_rng(7))
    return f.m


for label, sched, scheme in [("nofault", {}, "full"), ("nofault-none", {}, "none"),
                             ("fault8", {8: {P.ErrorKind.D0: 1}}, "full")]:
    m1 = run(False, sched, scheme)
    m2 = run(True, sched, scheme)
    d = np.abs(m1 - m2)
    bad = np.argwhere(d > 0)
    print(label, "ndiff", len(bad), "max", d.max())
    if len(bad):
        bl = sorted(set((int(r) // b, int(c) // b) for r, c in bad))
        print("  first blocks", bl[:12])
        cols = sorted(set(int(c) // b for r, c in bad))
        print("  block cols", cols)
