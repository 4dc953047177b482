"""Is the fused trailing update's epilogue C load the DMMA-issue limiter?
The LU trailing-update shape through abft_dev_dgemm with beta = 1 (C read
from HBM/L2 in the epilogue) vs beta = 0 (no C read: the kernel skips the
loads), same output writes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2301_03166_b200 import _lib

lib = _lib.load()
st = torch.cuda.current_stream()
m = n = 31744
k = 256
A = torch.randn((k, m), dtype=torch.float64, device="cuda")
B = torch.randn((n, k), dtype=torch.float64, device="cuda")
C = torch.randn((n, m), dtype=torch.float64, device="cuda")
for beta in (1.0, 0.0, 1.0, 0.0):
    def run():
        rc = lib.abft_dev_dgemm(st.cuda_stream, b"N", b"N", m, n, k, -1.0, A.data_ptr(), m,
                                B.data_ptr(), k, beta, C.data_ptr(), m, C.data_ptr(), m)
        assert rc == 0, _lib.last_error()
    for _ in range(2):
        run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(5):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"beta={beta}: {ms:.3f} ms  {2 * m * n * k / ms / 1e9:.1f} TFLOP/s")
