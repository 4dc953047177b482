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
