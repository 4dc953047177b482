"""Achieved TFLOP/s of the DMMA GEMM (abft_dev_dgemm) on the factorizations'
update shapes: LU trailing update vs the left-looking Cholesky panel update."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2301_03166_b200 import _lib

lib = _lib.load()
shapes = [("chol panel", "N", "T", 16384, 256, 16384), ("lu  trailing", "N", "N", 16384, 16384, 256), ("lu  trailing", "N", "N", 31744, 31744, 256),
          ("chol panel", "N", "T", 24576, 256, 8192), ("chol panel", "N", "T", 16384, 256, 16384),
          ("chol panel", "N", "T", 8192, 256, 24320), ("chol panel", "N", "T", 2048, 256, 30464),
          ("qr  V^T C", "T", "N", 256, 16384, 16640)]
st = torch.cuda.current_stream()
for name, ta, tb, m, n, k in shapes:
    A = torch.randn((k, m) if ta == "N" else (m, k), dtype=torch.float64, device="cuda")
    B = torch.randn((n, k) if tb == "N" else (k, n), dtype=torch.float64, device="cuda")
    C = torch.randn((n, m), dtype=torch.float64, device="cuda")
    lda = m if ta == "N" else k
    ldb = k if tb == "N" else n
    def run():
        rc = lib.abft_dev_dgemm(st.cuda_stream, ta.encode(), tb.encode(), m, n, k, -1.0, A.data_ptr(), lda,
                                B.data_ptr(), ldb, 1.0, C.data_ptr(), m, C.data_ptr(), m)
        assert rc == 0, _lib.last_error()
    for _ in range(3):
        run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(5):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"{name} {ta}{tb} M={m} N={n} K={k}: {ms:.3f} ms  {2 * m * n * k / ms / 1e9:.1f} TFLOP/s")
