"""Streamed LU / QR e2e (N=32768, KIND=lu|qr): chunk / split sweep in one process
(abft_set_input_chunks), pinned host in/out as bench.run_e2e."""
import ctypes, sys, time, statistics
import numpy as np
import torch
sys.path.insert(0, ".")
import bench

import os
KIND = os.environ.get("KIND", "lu")
n, b = 32768, 256
arm = bench.Arm(KIND, n, b, 0, 0)
FL = {"lu": 2 / 3, "qr": 4 / 3}[KIND] * n ** 3
P, lib, f = arm.P, arm.lib, arm.f
pin_in = torch.empty((n, n), dtype=torch.float64, pin_memory=True).numpy()
pin_in[...] = arm.host.T
src = pin_in.T
pin_out = torch.empty((n, n), dtype=torch.float64, pin_memory=True).numpy().T
P.linalg.check(lib.abft_keep_input(f._ctx, 0))
cfgs = [(16, 40, 0)]
if len(sys.argv) > 1:
    cfgs = [tuple(int(x) for x in c.split(",")) for c in sys.argv[1:]]
for chunk, split, rch in cfgs:
    P.linalg.check(lib.abft_set_input_chunks(f._ctx, chunk, split, rch))
    ts = []
    for i in range(3):
        t0 = time.perf_counter()
        P.linalg.check(lib.abft_set_matrix_streamed(f._ctx, P._lib.dptr(src), n))
        k_fault, rng = bench.fault_plan(n, b, 0)
        reps = P.run_protected(f, "full", {k_fault: {"0d": 1}}, rng, out=pin_out)
        ts.append(time.perf_counter() - t0)
    fixed = sum(r.corrected[P.ErrorKind.D0] for r in reps)
    dev = ctypes_ms = None
    sec = statistics.median(ts[1:])
    lib.abft_profile(f._ctx, 1)
    P.linalg.check(lib.abft_set_matrix_streamed(f._ctx, P._lib.dptr(src), n))
    k_fault, rng = bench.fault_plan(n, b, 0)
    P.run_protected(f, "full", {k_fault: {"0d": 1}}, rng, out=pin_out)
    ms = (ctypes.c_double * 4)()
    lib.abft_profile_read(f._ctx, ms)
    lib.abft_profile(f._ctx, 0)
    el = ctypes.c_double(0)
    lib.abft_last_elapsed_ms(f._ctx, ctypes.byref(el))
    print(f"chunk={chunk} split={split} rch={rch} e2e {sec*1e3:.1f} ms {FL/sec/1e12:.2f} TF/s "
          f"fixed={fixed} | profiled call {el.value:.1f} ms pd/pu/tmu/abft "
          + " ".join(f"{x:.1f}" for x in ms), flush=True)
