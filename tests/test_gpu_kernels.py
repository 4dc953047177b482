"""GPU: the DMMA/TMA GEMM and the region ABFT kernels against the references."""
import ctypes

import numpy as np
import pytest

import paper_2301_03166_b200 as P
from paper_2301_03166_b200 import _lib
from conftest import golden, report_json

pytestmark = pytest.mark.gpu


def _torch():
    import torch
    assert torch.cuda.is_available(), "GPU test selected but no CUDA device"
    return torch


@pytest.mark.parametrize("ta", "NT")
@pytest.mark.parametrize("tb", "NT")
@pytest.mark.parametrize("shape", [(128, 128, 16), (200, 130, 37), (1, 1, 1), (513, 257, 300),
                                   (256, 256, 4096), (64, 96, 20000), (333, 222, 111)])
def test_dgemm_matches_fp64_reference(ta, tb, shape):
    """D = C - op(A) op(B) vs a plain fp64 torch reference (tolerance: fp64
    accumulation error, 10 * sqrt(K) * eps relative to max|D|)."""
    torch = _torch()
    M, N, K = shape
    lib = _lib.load()
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N * 3 + K)
    def mat(r, c, ld):
        buf = torch.randn(ld * c + 2, dtype=torch.float64, device="cuda", generator=g)
        return buf, buf[:ld * c].view(c, ld)[:, :r].t()
    lda = ((M if ta == "N" else K) + 7) // 2 * 2
    ldb = ((K if tb == "N" else N) + 5) // 2 * 2
    ldc = (M + 3) // 2 * 2
    A, Av = mat(*((M, K) if ta == "N" else (K, M)), lda)
    B, Bv = mat(*((K, N) if tb == "N" else (N, K)), ldb)
    C, Cv = mat(M, N, ldc)
    opA = Av if ta == "N" else Av.t()
    opB = Bv if tb == "N" else Bv.t()
    ref = Cv - opA @ opB
    rc = lib.abft_dev_dgemm(None, ta.encode(), tb.encode(), M, N, K, -1.0, A.data_ptr(), lda,
                            B.data_ptr(), ldb, 1.0, C.data_ptr(), ldc, C.data_ptr(), ldc)
    torch.cuda.synchronize()
    assert rc == 0, _lib.last_error()
    err = (Cv - ref).abs().max().item() / max(1.0, ref.abs().max().item())
    assert err <= 10 * np.sqrt(K) * 2.2e-16


def _rm(n, seed):
    return np.random.default_rng(seed).uniform(-1.0, 1.0, size=(n, n))


@pytest.mark.parametrize("case", [c for c in golden("abft.json")])
def test_region_abft_matches_reference_reports(case):
    """pkg/tests/test_abft.py fixtures through the product's encode /
    inject_faults / verify_correct (device kernels): reports bit-exact with
    the reference; repaired data within 1e-12 (test_abft.py:41)."""
    E = P.ErrorKind
    want = golden("abft.json")[case]
    F = P.InjectedFault
    spec = {
        "single_corrects_0d": (3, "single", {}, [F(E.D0, 10, 37, 0.5)]),
        "single_flags_1d": (4, "single", {}, [F(E.D1, 16, 5, 0.3, extent=4)]),
        "full_corrects_1d_col": (5, "full", {}, [F(E.D1, 16, 5, 0.3, extent=4)]),
        "full_corrects_1d_row": (6, "full", {}, [F(E.D1, 20, 16, 0.4, orientation="row", extent=4)]),
        "full_flags_2d": (7, "full", {}, [F(E.D2, 17, 18, 0.4, extent=3)]),
        "multi_0d_distinct_blocks": (8, "single", {}, [F(E.D0, 16 * i + 3, 16 * i + 7, 0.2 + i) for i in range(4)]),
        "region_offsets": (9, "full", dict(r0=16, c0=32, shape=(48, 32)), [F(E.D0, 40, 50, 0.9)]),
    }
    for sch in ("single", "full"):
        spec[f"q1_two_0d_one_block_{sch}"] = (21, sch, {}, [F(E.D0, 3, 5, 0.5), F(E.D0, 9, 11, -0.7)])
        spec[f"q2_two_0d_one_column_{sch}"] = (22, sch, {}, [F(E.D0, 3, 5, 0.5), F(E.D0, 9, 5, -0.7)])
        spec[f"q3_2d_corner_straddle_{sch}"] = (23, sch, {}, [F(E.D2, 14, 14, 0.5, extent=4)])
    if case == "no_false_positive_20_updates":
        rng = np.random.default_rng(12)
        m = rng.uniform(-1, 1, size=(96, 96))
        cs = P.encode(m, 16, P.ChecksumScheme.FULL)
        for _ in range(20):
            left = rng.uniform(-1, 1, size=(96, 8))
            right = rng.uniform(-1, 1, size=(8, 96))
            P.maintain_gemm(cs, left, right)
            m -= left @ right
        assert report_json(P.verify_correct(m, cs)) == want
        return
    seed, scheme, kw, faults = spec[case]
    m = _rm(64, seed)
    orig = m.copy()
    cs = P.encode(m, 16, scheme, **kw)
    P.inject_faults(m, faults)
    rep = P.verify_correct(m, cs)
    assert report_json(rep) == want
    if case in ("single_corrects_0d", "full_corrects_1d_col", "full_corrects_1d_row",
                "multi_0d_distinct_blocks", "region_offsets"):
        assert np.allclose(m, orig, atol=1e-12)


def test_region_outside_fault_invisible():
    m = _rm(64, 9)
    cs = P.encode(m, 16, P.ChecksumScheme.FULL, r0=16, c0=32, shape=(48, 32))
    P.inject_faults(m, [P.InjectedFault(P.ErrorKind.D0, 0, 0, 0.9)])
    assert P.verify_correct(m, cs).clean


@pytest.mark.parametrize("seed", range(50))
def test_single_repairs_any_isolated_element(seed):
    """test_abft.py:109-119 (hypothesis-style sweep, seeded)."""
    rng = np.random.default_rng(1000 + seed)
    row, col = int(rng.integers(64)), int(rng.integers(64))
    mag = float(10 ** rng.uniform(-3, 3)) * (1 if rng.random() < 0.5 else -1)
    m = _rm(64, 10)
    cs = P.encode(m, 16, P.ChecksumScheme.SINGLE)
    orig = m.copy()
    P.inject_faults(m, [P.InjectedFault(P.ErrorKind.D0, row, col, mag)])
    P.verify_correct(m, cs)
    assert np.allclose(m, orig, atol=1e-9)


def test_inject_out_of_range_raises():
    m = _rm(8, 1)
    with pytest.raises(IndexError):
        P.inject_faults(m, [P.InjectedFault(P.ErrorKind.D0, 8, 0, 1.0)])


def _np_lu_nopiv(a, shift):
    """Unpivoted LU of a (mode 0) or of a - diag(s), s_c = -sign(pivot) (mode 2)."""
    a = a.copy()
    w = a.shape[0]
    s = np.zeros(w)
    for c in range(w):
        if shift:
            s[c] = 1.0 if a[c, c] < 0 else -1.0
            a[c, c] -= s[c]
        a[c + 1:, c] /= a[c, c]
        a[c + 1:, c + 1:] -= np.outer(a[c + 1:, c], a[c, c + 1:])
    return a, s


@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("mode", [0, 1, 2])
@pytest.mark.parametrize("w", [256, 200, 128, 64, 33, 1])
@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_diag_factor_variants(variant, mode, w, prec):
    """The diagonal-block factorization (one-CTA diag_factor and the cluster
    kernel): factors and triangular inverses against numpy in fp64
    (linalg.py:219-238; mode 2 = the sign-shifted LU of qr_panel.cu)."""
    torch = _torch()
    lib = _lib.load()
    rng = np.random.default_rng(w * 10 + mode)
    a = rng.uniform(-1, 1, (w, w))
    if mode == 0:
        a += np.diag(np.abs(a).sum(axis=1) + 1.0)
    elif mode == 1:
        a = a @ a.T + w * np.eye(w)
    else:
        a = np.linalg.qr(rng.standard_normal((w, w)))[0]  # the reconstruction's input: orthogonal
    dt = torch.float64 if prec == "f64" else torch.float32
    ld = w + 3
    buf = torch.zeros((w, ld), dtype=dt, device="cuda")
    buf[:, :w] = torch.from_numpy(a.T.copy()).to(dt)  # column-major: column j = row j of buf
    D = buf
    Li = torch.zeros((w, ld), dtype=dt, device="cuda")
    Ui = torch.zeros((w, ld), dtype=dt, device="cuda")
    sg = torch.zeros(w, dtype=dt, device="cuda")
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    fn = lib.abft_dev_diag_factor if prec == "f64" else lib.abft_dev_sdiag_factor
    rc = fn(None, variant, mode, w, D.data_ptr(), ld, Li.data_ptr(), ld,
            Ui.data_ptr() if mode != 1 else None, ld, info.data_ptr(), sg.data_ptr())
    assert rc == 0, _lib.last_error()
    torch.cuda.synchronize()
    assert int(info.item()) == 0
    got = D[:, :w].double().cpu().numpy().T
    linv = Li[:, :w].double().cpu().numpy().T
    tol = 1e-11 if prec == "f64" else 5e-4
    if mode == 1:
        ref = np.linalg.cholesky(a)
        np.testing.assert_allclose(got, ref, atol=tol * np.abs(ref).max(), rtol=0)
        np.testing.assert_allclose(linv, np.linalg.inv(ref), atol=tol * 10, rtol=0)
    else:
        ref, s = _np_lu_nopiv(a, mode == 2)
        np.testing.assert_allclose(got, ref, atol=tol * np.abs(ref).max(), rtol=0)
        L = np.tril(ref, -1) + np.eye(w)
        U = np.triu(ref)
        np.testing.assert_allclose(linv, np.linalg.inv(L), atol=tol * 10 * max(1, np.abs(np.linalg.inv(L)).max()), rtol=0)
        uinv = Ui[:, :w].double().cpu().numpy().T
        np.testing.assert_allclose(uinv, np.linalg.inv(U), atol=tol * 10 * max(1, np.abs(np.linalg.inv(U)).max()), rtol=0)
        if mode == 2:
            np.testing.assert_array_equal(sg.double().cpu().numpy(), s)


@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("mode,col", [(1, 77), (0, 150)])
def test_diag_factor_breakdown_column(variant, mode, col):
    """Breakdown reports the reference's column (Cholesky pivot <= 0, LU zero
    pivot: linalg.py:223-224, :234-235) from both kernels."""
    torch = _torch()
    lib = _lib.load()
    w = 256
    a = np.eye(w) * 4.0
    a[col, col] = -1.0 if mode == 1 else 0.0
    D = torch.from_numpy(a.T.copy()).cuda()
    Li = torch.zeros_like(D)
    Ui = torch.zeros_like(D)
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    rc = lib.abft_dev_diag_factor(None, variant, mode, w, D.data_ptr(), w, Li.data_ptr(), w,
                                  Ui.data_ptr() if mode == 0 else None, w, info.data_ptr(), None)
    assert rc == 0
    torch.cuda.synchronize()
    assert int(info.item()) == col + 1


def test_full_zero_bad_rows_two_bad_columns_raises_index_error():
    """Quirk Q5: FULL verification of a block whose row sums
    agree but two column sums disagree -- +d and -d in one row -- classifies
    it as 1-D and reads bad_rows[0] of an empty array (abft.py:267): the
    reference raises IndexError (checked against the reference itself in
    tests/test_oracle_golden.py), so does the drop-in."""
    n, b = 64, 16
    m = _rm(n, 21)
    cs = P.encode(m, b, P.ChecksumScheme.FULL)
    d = 0.5
    m[5, 2] += d
    m[5, 9] -= d
    with pytest.raises(IndexError):
        P.verify_correct(m, cs)
