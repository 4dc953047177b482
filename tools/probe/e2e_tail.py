"""How much of the e2e gap is the D2H tail? Streamed input with and without
the streamed output (dgetrf / dgeqrf N=32768; KIND env)."""
import ctypes, os, sys, time, statistics
import torch
sys.path.insert(0, ".")
import bench

KIND = os.environ.get("KIND", "lu")
n, b = 32768, 256
arm = bench.Arm(KIND, n, b, 0, 0)
P, lib, f = arm.P, arm.lib, arm.f
pin_in = torch.empty((n, n), dtype=torch.float64, pin_memory=True).numpy()
pin_in[...] = arm.host.T
src = pin_in.T
pin_out = torch.empty((n, n), dtype=torch.float64, pin_memory=True).numpy().T
P.linalg.check(lib.abft_keep_input(f._ctx, 0))
for label, out in [("in+out", pin_out), ("in only", None), ("in+out", pin_out), ("in only", None)]:
    ts = []
    for i in range(3):
        t0 = time.perf_counter()
        P.linalg.check(lib.abft_set_matrix_streamed(f._ctx, P._lib.dptr(src), n))
        k_fault, rng = bench.fault_plan(n, b, 0)
        P.run_protected(f, "full", {k_fault: {"0d": 1}}, rng, out=out)
        ts.append(time.perf_counter() - t0)
    print(KIND, label, f"{statistics.median(ts[1:]) * 1e3:.1f} ms", flush=True)
