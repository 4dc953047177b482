"""GEMM throughput vs K (trailing-update shapes), for A/B experiments."""
import ctypes, sys, torch
sys.path.insert(0, ".")
from paper_2301_03166_b200 import _lib
lib = _lib.load()
def bench(M, N, K, reps=5, beta=1.0):
    A = torch.randn(M * K, dtype=torch.float64, device="cuda"); B = torch.randn(K * N, dtype=torch.float64, device="cuda")
    C = torch.randn(M * N, dtype=torch.float64, device="cuda")
    f = lambda: lib.abft_dev_dgemm(None, b'N', b'N', M, N, K, -1.0, A.data_ptr(), M, B.data_ptr(), K, beta, C.data_ptr(), M, C.data_ptr(), M)
    f(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"  {M}x{N}x{K} beta={beta}: {2*M*N*K/ms/1e9:.2f} TFLOP/s")
for K in (256, 1024):
    bench(16384, 16384, K)
    bench(16384, 16384, K, beta=0.0)
