import torch, time
torch.backends.cuda.matmul.allow_tf32 = False
for n in (4096, 8192, 16384):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(3): c = a @ b
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    reps = 10 if n < 16384 else 4
    e0.record()
    for _ in range(reps): c = a @ b
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"cuBLAS DGEMM {n}^3: {2*n**3/ms/1e9:.2f} TFLOP/s ({ms:.2f} ms)")
# rank-256 update shape (LU TMU at N=32768, k=0)
n, kk = 32512, 256
a = torch.randn(n, kk, dtype=torch.float64, device="cuda")
b = torch.randn(kk, n, dtype=torch.float64, device="cuda")
c = torch.randn(n, n, dtype=torch.float64, device="cuda")
for _ in range(2): c.addmm_(a, b, alpha=-1)
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5): c.addmm_(a, b, alpha=-1)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"cuBLAS DGEMM rank-256 update {n}x{n}x{kk}: {2*n*n*kk/ms/1e9:.2f} TFLOP/s ({ms:.2f} ms)")
# cusolver dpotrf / dgetrf via torch.linalg
for n in (8192, 16384, 32768):
    a = torch.rand(n, n, dtype=torch.float64, device="cuda") * 2 - 1
    a.diagonal().copy_(a.abs().sum(1) + 1)
    torch.cuda.synchronize()
    for rep in range(2):
        t0 = time.perf_counter(); lu, piv = torch.linalg.lu_factor(a); torch.cuda.synchronize(); t = time.perf_counter() - t0
    print(f"cuSOLVER dgetrf {n}: {2*n**3/3/t/1e12:.2f} TFLOP/s ({t*1e3:.1f} ms)")
    del lu, piv
    s = a @ a.T if n <= 16384 else None
    if s is not None:
        s.diagonal().add_(n)
        for rep in range(2):
            t0 = time.perf_counter(); l = torch.linalg.cholesky(s); torch.cuda.synchronize(); t = time.perf_counter() - t0
        print(f"cuSOLVER dpotrf {n}: {n**3/3/t/1e12:.2f} TFLOP/s ({t*1e3:.1f} ms)")
        for rep in range(2):
            t0 = time.perf_counter(); q = torch.geqrf(a); torch.cuda.synchronize(); t = time.perf_counter() - t0
        print(f"cuSOLVER dgeqrf {n}: {4*n**3/3/t/1e12:.2f} TFLOP/s ({t*1e3:.1f} ms)")
        del s, l, q
    del a
    torch.cuda.empty_cache()
