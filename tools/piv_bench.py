"""Pivoted vs unpivoted LU (FULL checksums, fault-free) on one B200: device
time of one protected factorization after a warm-up."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2301_03166_b200 as P

for n in (8192, 16384, 32768):
    dom = P.generate_test_matrix("lu", n, 0)
    gen = np.asfortranarray(np.random.default_rng(0).uniform(-1, 1, (n, n))) if n <= 16384 else None
    for name, a, piv in (("unpivoted (reference input)", dom, False), ("pivoted (reference input)", dom, True),
                         ("pivoted (uniform input)", gen, True)):
        if a is None:
            continue
        f = P.Factorization("lu", a, 256, pivoting=piv, keep_input=True)
        P.run_protected(f, "full", {}, None)
        f._lib.abft_reset(f._ctx)
        f.k_done = 0
        torch.cuda.synchronize()
        t = time.perf_counter()
        P.run_protected(f, "full", {}, None)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        print(f"N={n} {name}: {dt * 1e3:.1f} ms {2 * n ** 3 / 3 / dt / 1e12:.2f} TF/s "
              f"residual {P.residual(a, f):.2e}", flush=True)
        del f
        torch.cuda.empty_cache()
