"""GPU: the tcgen05 fp32 GEMM (kind::tf32, 3xTF32) against a float64
reference of the same op. Bound: |D - D_ref| <= 2e-6 * max(1, sqrt(K/256)) *
(|alpha| |A||B| + |beta||C|) elementwise (fp32 accumulation accuracy; plain
TF32 operands would be ~1e-3)."""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run(ta, tb, m, n, k, alpha=1.0, beta=0.0, seed=0, splits=1):
    import torch
    from paper_2301_03166_b200 import _lib
    lib = _lib.load()
    g = torch.Generator(device="cpu").manual_seed(seed)
    a_shape = (m, k) if ta == "N" else (k, m)
    b_shape = (k, n) if tb == "N" else (n, k)
    # column-major storage = transpose of a row-major torch tensor
    A = torch.randn(a_shape[::-1], generator=g, dtype=torch.float32).cuda()
    B = torch.randn(b_shape[::-1], generator=g, dtype=torch.float32).cuda()
    C = torch.randn((n, m), generator=g, dtype=torch.float32).cuda()
    D = torch.empty((n, m), dtype=torch.float32, device="cuda")
    rc = lib.abft_dev_sgemm_splitk(None, ta.encode(), tb.encode(), m, n, k, alpha, A.data_ptr(),
                                   a_shape[0], B.data_ptr(), b_shape[0], beta,
                                   C.data_ptr() if beta else None, m, D.data_ptr(), m, splits)
    assert rc == 0, _lib.last_error()
    torch.cuda.synchronize()
    An = A.double().cpu().numpy().T
    Bn = B.double().cpu().numpy().T
    opA = An if ta == "N" else An.T
    opB = Bn if tb == "N" else Bn.T
    Cn = C.double().cpu().numpy().T
    ref = alpha * (opA @ opB) + beta * Cn
    mag = abs(alpha) * (np.abs(opA) @ np.abs(opB)) + abs(beta) * np.abs(Cn)
    got = D.double().cpu().numpy().T
    return got, ref, mag


@pytest.mark.parametrize("ta,tb", [("N", "N"), ("N", "T"), ("T", "N"), ("T", "T")])
@pytest.mark.parametrize("m,n,k", [(128, 128, 32), (256, 384, 128), (300, 200, 100), (1000, 517, 256)])
def test_sgemm_tc05_matches_fp64_reference(ta, tb, m, n, k):
    got, ref, mag = _run(ta, tb, m, n, k, alpha=-1.0, beta=1.0)
    err = np.abs(got - ref)
    tol = 2e-6 * max(1.0, (k / 256) ** 0.5)
    assert np.all(err <= tol * mag + 1e-30), float((err / (mag + 1e-30)).max())


def test_sgemm_tc05_large_k_and_alpha():
    got, ref, mag = _run("N", "N", 512, 512, 2048, alpha=0.5, beta=0.0)
    err = np.abs(got - ref)
    assert np.all(err <= 2e-6 * (2048 / 256) ** 0.5 * mag), float((err / mag).max())


@pytest.mark.parametrize("ta,tb", [("N", "N"), ("N", "T"), ("T", "N")])
@pytest.mark.parametrize("m,n,k,splits", [(1000, 128, 4096, 7), (128, 517, 3000, 16),
                                          (300, 200, 100, 3), (256, 256, 64, 5)])
def test_sgemm_tc05_split_k(ta, tb, m, n, k, splits):
    """split-K: K-slices in separate tensor-core chains + fixed-order
    reduction (beta*C added once); splits beyond the k-block count clamp."""
    got, ref, mag = _run(ta, tb, m, n, k, alpha=-1.0, beta=1.0, splits=splits)
    err = np.abs(got - ref)
    tol = 2e-6 * max(1.0, (k / 256) ** 0.5)
    assert np.all(err <= tol * mag + 1e-30), float((err / (mag + 1e-30)).max())


def test_sgemm_tc05_split_k_is_deterministic():
    a = _run("N", "T", 640, 128, 8192, alpha=-1.0, beta=1.0, splits=12)[0]
    b = _run("N", "T", 640, 128, 8192, alpha=-1.0, beta=1.0, splits=12)[0]
    assert np.array_equal(a, b)


@pytest.mark.parametrize("splits", [1, 3])
def test_sgemm_tc05_raw_operands_with_k_tail(splits):
    """'T' A and 'N' B with 16-byte aligned leading dimensions are split in
    shared memory (raw TMA boxes); K = 77 leaves a partial k-block whose
    tail the TMA must zero-fill. Checked against fp64."""
    import torch
    from paper_2301_03166_b200 import _lib
    lib = _lib.load()
    m, n, k, ld = 200, 130, 77, 80
    g = torch.Generator(device="cpu").manual_seed(5)
    At = torch.randn((m, ld), generator=g, dtype=torch.float32)   # column-major k x m, ld 80
    Bt = torch.randn((n, ld), generator=g, dtype=torch.float32)   # column-major k x n, ld 80
    At[:, k:] = float("nan")  # must never be read
    Bt[:, k:] = float("nan")
    C = torch.randn((n, m), generator=g, dtype=torch.float32)
    A, B, Cd = At.cuda(), Bt.cuda(), C.cuda()
    D = torch.empty((n, m), dtype=torch.float32, device="cuda")
    rc = lib.abft_dev_sgemm_splitk(None, b"T", b"N", m, n, k, -1.0, A.data_ptr(), ld, B.data_ptr(),
                                   ld, 1.0, Cd.data_ptr(), m, D.data_ptr(), m, splits)
    assert rc == 0, _lib.last_error()
    torch.cuda.synchronize()
    opA = At[:, :k].double().numpy()          # m x k
    opB = Bt[:, :k].double().numpy().T        # k x n
    ref = -(opA @ opB) + C.double().numpy().T
    mag = np.abs(opA) @ np.abs(opB) + np.abs(C.double().numpy().T)
    got = D.double().cpu().numpy().T
    assert np.all(np.isfinite(got))
    assert np.all(np.abs(got - ref) <= 2e-6 * mag), float((np.abs(got - ref) / mag).max())
