"""GPU check + timing of the DMMA/TMA dgemm against torch (cuBLAS) fp64."""
import ctypes, sys, time
import torch
lib = ctypes.CDLL("paper_2301_03166_b200/libabft_b200.so")
lib.abft_dev_dgemm.argtypes = [ctypes.c_void_p, ctypes.c_char, ctypes.c_char] + [ctypes.c_int64]*3 + \
    [ctypes.c_double, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_double,
     ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64]
lib.abft_last_error.restype = ctypes.c_char_p

def colmajor(rows, cols, ld, off=0):
    buf = torch.randn(ld * cols + off + 8, dtype=torch.float64, device="cuda")
    return buf, off

def view(buf, off, rows, cols, ld):
    return buf[off:off + ld * cols].view(cols, ld)[:, :rows].t()  # rows x cols view, col-major

def run(ta, tb, M, N, K, off_a=0, off_c=0, alpha=-1.0, beta=1.0):
    lda = (M if ta == 'N' else K) + 6
    ldb = (K if tb == 'N' else N) + 4
    ldc = M + 2
    ra, ca = (M, K) if ta == 'N' else (K, M)
    rb, cb = (K, N) if tb == 'N' else (N, K)
    A, oa = colmajor(ra, ca, lda, off_a); B, ob = colmajor(rb, cb, ldb)
    C, oc = colmajor(M, N, ldc, off_c)
    Av = view(A, oa, ra, ca, lda); Bv = view(B, ob, rb, cb, ldb); Cv = view(C, oc, M, N, ldc)
    opA = Av if ta == 'N' else Av.t(); opB = Bv if tb == 'N' else Bv.t()
    ref = beta * Cv + alpha * (opA @ opB)
    rc = lib.abft_dev_dgemm(None, ta.encode(), tb.encode(), M, N, K, alpha, A.data_ptr() + 8 * oa, lda,
                            B.data_ptr() + 8 * ob, ldb, beta, C.data_ptr() + 8 * oc, ldc, C.data_ptr() + 8 * oc, ldc)
    torch.cuda.synchronize()
    if rc != 0:
        print("rc", rc, lib.abft_last_error()); return False
    err = (Cv - ref).abs().max().item() / max(1.0, ref.abs().max().item())
    ok = err < 1e-13 * max(1, K) ** 0.5 * 10
    print(f"{ta}{tb} M={M} N={N} K={K} offA={off_a} offC={off_c}: relerr {err:.2e} {'OK' if ok else 'FAIL'}")
    return ok

ok = True
for ta in "NT":
    for tb in "NT":
        for (M, N, K) in [(128, 128, 16), (200, 130, 37), (1, 1, 1), (513, 257, 300), (256, 256, 4096), (64, 96, 20000)]:
            ok &= run(ta, tb, M, N, K)
        ok &= run(ta, tb, 333, 222, 111, off_a=1, off_c=1)
print("ALL OK" if ok else "SOME FAILED")

def bench(ta, tb, M, N, K, reps=5):
    lda = M if ta == 'N' else K; ldb = K if tb == 'N' else N
    A = torch.randn(lda * (K if ta == 'N' else M), dtype=torch.float64, device="cuda")
    B = torch.randn(ldb * (N if tb == 'N' else K), dtype=torch.float64, device="cuda")
    C = torch.randn(M * N, dtype=torch.float64, device="cuda")
    f = lambda: lib.abft_dev_dgemm(None, ta.encode(), tb.encode(), M, N, K, -1.0, A.data_ptr(), lda, B.data_ptr(), ldb, 1.0, C.data_ptr(), M, C.data_ptr(), M)
    f(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"bench {ta}{tb} {M}x{N}x{K}: {ms:.3f} ms  {2*M*N*K/ms/1e9:.2f} TFLOP/s")
bench('N', 'N', 32512, 32512, 256)
bench('N', 'N', 16384, 16384, 256)
bench('N', 'N', 8192, 8192, 8192)
bench('N', 'T', 8192, 8192, 8192)
bench('T', 'N', 8192, 8192, 8192)
bench('T', 'T', 8192, 8192, 8192)
bench('N', 'T', 16384, 256, 16384)
bench('T', 'N', 256, 16384, 16384)
