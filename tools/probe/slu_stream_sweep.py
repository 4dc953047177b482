"""Streamed sgetrf e2e (N=16384, b=128): wall time vs the call's device time."""
import ctypes, os, sys, time, statistics
import numpy as np
import torch
sys.path.insert(0, ".")
import bench

n, b = 16384, 128
arm = bench.SArm("lu", n, b, 0, 0)
f, lib, P = arm.f, arm.lib, arm.P
pin_in = torch.empty((n, n), dtype=torch.float32, pin_memory=True).numpy()
pin_in[...] = arm.host.T
src = pin_in.T
pin_out = torch.empty((n, n), dtype=torch.float32, pin_memory=True).numpy().T
P.linalg.check(lib.abft_s_keep_input(f._ctx, 0))
cfgs = [(0, -1, 0), (-1, -1, 0), (8, 32, 0), (16, 64, 0), (4, 24, 0)]
if len(sys.argv) > 1:
    cfgs = [tuple(int(x) for x in a.split(",")) + ((0,) if a.count(",") == 1 else ())
            for a in sys.argv[1:]]
for chunk, split, rch in cfgs:
    lib.abft_s_set_input_chunks(f._ctx, chunk, split, rch)
    ts, dev = [], []
    for i in range(4):
        t0 = time.perf_counter()
        P.linalg.check(lib.abft_s_set_matrix_streamed(f._ctx, P._lib.fptr(src), n))
        k_fault, rng = bench.fault_plan(n, b, 0)
        t1 = time.perf_counter()
        reps = f.run_protected("full", {k_fault: {"0d": 1}}, rng, out=pin_out)
        t2 = time.perf_counter()
        el = ctypes.c_double(0)
        lib.abft_s_last_elapsed_ms(f._ctx, ctypes.byref(el))
        if i:
            ts.append((t2 - t0, t2 - t1))
            dev.append(el.value)
    print(f"chunk={chunk} split={split} rch={rch} wall {statistics.median(t[0] for t in ts)*1e3:.1f} ms "
          f"(run_protected {statistics.median(t[1] for t in ts)*1e3:.1f}) device call "
          f"{statistics.median(dev):.1f} ms", flush=True)
