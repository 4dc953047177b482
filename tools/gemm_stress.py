import ctypes, sys, torch
sys.path.insert(0, ".")
from paper_2301_03166_b200 import _lib
lib = _lib.load()
st = torch.cuda.Stream()
def case(M, N, K, lda, ldb, ldc, g):
    A = torch.randn(lda * K, dtype=torch.float64, device="cuda", generator=g)
    B = torch.randn(ldb * K, dtype=torch.float64, device="cuda", generator=g)   # 'T': B(k,n)=B[n + k*ldb]
    C = torch.randn(ldc * N, dtype=torch.float64, device="cuda", generator=g)
    return A, B, C
g = torch.Generator(device="cuda").manual_seed(0)
shapes = [(8, 32, 160, 16, 256, 16), (96, 32, 160, 256, 256, 256), (128, 32, 128, 256, 256, 256), (64, 64, 192, 256, 256, 256)]
bufs = [case(*s, g) for s in shapes]
refs = []
for (M, N, K, lda, ldb, ldc), (A, B, C) in zip(shapes, bufs):
    Av = A[:lda*K].view(K, lda)[:, :M].t(); Bv = B[:ldb*K].view(K, ldb)[:, :N]; Cv = C[:ldc*N].view(N, ldc)[:, :M].t()
    refs.append((Cv.clone() - Av @ Bv))
bad = 0
for it in range(int(sys.argv[1])):
    outs = []
    for (M, N, K, lda, ldb, ldc), (A, B, C) in zip(shapes, bufs):
        D = torch.empty(ldc * N, dtype=torch.float64, device="cuda")
        rc = lib.abft_dev_dgemm(ctypes.c_void_p(st.cuda_stream), b'N', b'T', M, N, K, -1.0, A.data_ptr(), lda, B.data_ptr(), ldb, 1.0, C.data_ptr(), ldc, D.data_ptr(), ldc)
        assert rc == 0
        outs.append(D)
    st.synchronize()
    for (M, N, K, lda, ldb, ldc), D, ref in zip(shapes, outs, refs):
        Dv = D[:ldc*N].view(N, ldc)[:, :M].t()
        err = (Dv - ref).abs()
        if err.max().item() > 1e-10:
            bad += 1
            rows = torch.nonzero(err > 1e-10)[:, 0]
            if bad <= 5: print(f"it {it} shape {M}x{N}x{K}: err {err.max().item():.2e} rows {rows.min().item()}..{rows.max().item()} n {len(rows)}")
print("bad", bad)
