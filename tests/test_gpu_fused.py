"""GPU: the fused-checksum GEMM epilogue (b = 128 / 256, LU and QR) gives the
same detection / correction as the CPU oracle and as the unfused path."""
import os

import numpy as np
import pytest

import oracle as O
import paper_2301_03166_b200 as P
from conftest import report_json

pytestmark = pytest.mark.gpu

COUNTS = {"0d": 2, "1d": 1, "2d": 1}


def run_gpu(kind, n, b, seed, scheme, fault_iters, no_fuse=False):
    old = os.environ.get("ABFT_NO_FUSE")
    os.environ["ABFT_NO_FUSE"] = "1" if no_fuse else "0"
    try:
        a = P.generate_test_matrix(kind, n, seed)
        f = P.Factorization(kind, a, b)
    finally:
        if old is None:
            os.environ.pop("ABFT_NO_FUSE")
        else:
            os.environ["ABFT_NO_FUSE"] = old
    rng = np.random.default_rng(seed)
    reps = [report_json(P.run_numeric_iteration(f, k, scheme,
                                                COUNTS if k in fault_iters else None, rng))
            for k in range(f.layout.n_blocks)]
    return reps, P.residual(a, f), f


def run_oracle(kind, n, b, seed, scheme, fault_iters):
    a = O.generate_test_matrix(kind, n, seed)
    f = O.OracleFactorization(kind, a, b)
    rng = np.random.default_rng(seed)
    reps = [O.protected_iteration(f, k, scheme, COUNTS if k in fault_iters else None, rng).to_json()
            for k in range(f.nb)]
    return reps, O.residual(a, f)


@pytest.mark.parametrize("kind", ["lu", "qr"])
@pytest.mark.parametrize("n,b", [(1024, 128), (1000, 128), (1536, 256), (1300, 256)])
@pytest.mark.parametrize("scheme", ["single", "full"])
def test_fused_matches_oracle(kind, n, b, scheme):
    fault_iters = {1, (-(-n // b)) - 2}
    got, res, _ = run_gpu(kind, n, b, 11, scheme, fault_iters)
    want, res_o = run_oracle(kind, n, b, 11, scheme, fault_iters)
    assert got == want
    if res_o <= 1e-8:
        assert res <= res_o + 16 * n * 2.220446049250313e-16
    else:
        assert res == pytest.approx(res_o, rel=1e-3)


@pytest.mark.parametrize("kind", ["lu", "qr"])
def test_fused_equals_unfused(kind):
    n, b = 1792, 256
    r1, res1, f1 = run_gpu(kind, n, b, 5, "full", {2})
    r2, res2, f2 = run_gpu(kind, n, b, 5, "full", {2}, no_fuse=True)
    assert r1 == r2
    np.testing.assert_allclose(f1.m, f2.m, rtol=0, atol=1e-12)


@pytest.mark.parametrize("kind", ["lu", "qr", "cholesky"])
def test_clean_large_run_has_no_false_positives(kind):
    """N = 4096, b = 256, no faults: no detections (SURVEY probe #5)."""
    n, b = 4096, 256
    a = P.generate_test_matrix("lu" if kind == "cholesky" else kind, n, 3)
    if kind == "cholesky":
        a = a @ a.T + n * np.eye(n)
    f = P.Factorization(kind, np.asfortranarray(a), b)
    reps = P.run_protected(f, "full", {}, np.random.default_rng(0))
    assert all(r.clean for r in reps)
    assert P.residual(a, f) < 64 * n * 2.220446049250313e-16


@pytest.mark.parametrize("kind", ["lu", "qr"])
@pytest.mark.parametrize("n,b", [(2048, 256), (1408, 128), (1300, 256)])
def test_lookahead_fast_path_equals_per_iteration(kind, n, b):
    """abft_factorize's look-ahead (LU: next diagonal block, QR: next
    Householder panel, factored on a side stream while the rest of the
    trailing matrix updates) gives the same reports as run_numeric_iteration,
    faults at two iterations (those run serialised)."""
    nb = -(-n // b)
    sched = {1: {P.ErrorKind.D0: 2, P.ErrorKind.D1: 1}, nb - 2: {P.ErrorKind.D0: 1}}
    a = P.generate_test_matrix(kind, n, 9)
    f1 = P.Factorization(kind, a, b)
    rng = np.random.default_rng(9)
    per = [report_json(P.run_numeric_iteration(f1, k, "full", sched.get(k), rng)) for k in range(nb)]
    f2 = P.Factorization(kind, a, b)
    fast = [report_json(r) for r in P.run_protected(f2, "full", sched, np.random.default_rng(9))]
    assert per == fast
    np.testing.assert_allclose(f2.m, f1.m, rtol=0, atol=1e-12)
    r1, r2 = P.residual(a, f1), P.residual(a, f2)
    assert r2 == pytest.approx(r1, rel=1e-6, abs=1e-15)
    if not any(r["uncorrectable"] for r in per):
        assert r2 < 1e-14


@pytest.mark.parametrize("n,b", [(2048, 256), (1408, 128), (1300, 256)])
@pytest.mark.parametrize("scheme", ["full", "single", "none"])
def test_lu_lookahead_depth2_equals_depth1(monkeypatch, n, b, scheme):
    """ABFT_LU_LA2=1 (off by default, measured slower): the look-ahead also
    forms L21(k+1) and -- after block row k+1 of the update is verified --
    PU(k+1) on the side stream, the rest of the update split into that block
    row and the rows below (events with a block-row offset). Same reports,
    bit-identical factor."""
    nb = -(-n // b)
    sched = {2: {P.ErrorKind.D0: 1}, nb - 3: {P.ErrorKind.D0: 1, P.ErrorKind.D1: 1}}
    a = P.generate_test_matrix("lu", n, 11)
    out = []
    for la2 in ("0", "1"):
        monkeypatch.setenv("ABFT_LU_LA2", la2)
        f = P.Factorization("lu", a, b)
        reps = [report_json(r) for r in P.run_protected(f, scheme, sched, np.random.default_rng(11))]
        out.append((reps, f.m))
    assert out[0][0] == out[1][0]
    assert np.array_equal(out[0][1], out[1][1])
    if scheme != "none":
        assert sum(len(r["locations"]) for r in out[1][0]) >= 2


@pytest.mark.parametrize("kind", ["cholesky", "lu", "qr"])
@pytest.mark.parametrize("n,b", [(2048, 256), (1300, 256), (1408, 128)])
def test_streamed_input_equals_set_matrix(kind, n, b):
    """abft_set_matrix_streamed: the input arrives block column by block
    column inside abft_factorize (Cholesky: only the lower block triangle,
    each iteration waiting for its block; its FULL row checksums start at
    zero and take each block's row sums on arrival). Same reports and the
    same factor as abft_set_matrix, with faults at two iterations; the device
    matrix is overwritten with junk first so nothing stale can pass."""
    import ctypes
    nb = -(-n // b)
    sched = {1: {P.ErrorKind.D0: 2, P.ErrorKind.D1: 1}, nb - 2: {P.ErrorKind.D0: 1}}
    a = P.generate_test_matrix(kind, n, 5)
    f1 = P.Factorization(kind, a, b)
    ref = [report_json(r) for r in P.run_protected(f1, "full", sched, np.random.default_rng(5))]
    f2 = P.Factorization(kind, a, b)
    lib = f2._lib
    junk = np.asfortranarray(np.random.default_rng(1).standard_normal((n, n)) * 1e3)
    assert lib.abft_set_matrix(f2._ctx, junk.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), n) == 0
    af = np.asfortranarray(a, dtype=np.float64)
    assert lib.abft_set_matrix_streamed(f2._ctx, af.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                        n) == 0
    got = [report_json(r) for r in P.run_protected(f2, "full", sched, np.random.default_rng(5))]
    assert got == ref
    m1, m2 = f1.m, f2.m
    if kind == "cholesky":  # the factorization zeroes what it does not copy in
        m1, m2 = np.tril(m1), np.tril(m2)
        assert not np.any(np.triu(f2.m, 1))
    np.testing.assert_allclose(m2, m1, rtol=0, atol=1e-12 * max(1.0, np.abs(m1).max()))


@pytest.mark.parametrize("n,b,chunk,split", [(2048, 128, 3, 8), (2048, 128, 2, -1), (1300, 256, 1, 3),
                                             (1408, 128, 4, 10), (2048, 256, 8, -1),
                                             (4096, 128, -1, -1), (2048, 128, 0, -1)])
@pytest.mark.parametrize("schemes", ["full", "single", "mixed"])
@pytest.mark.parametrize("kind", ["lu", "qr"])
def test_streamed_chunked_equals_set_matrix(monkeypatch, kind, n, b, chunk, split, schemes):
    """Streamed LU / QR input: block columns [0, split b) are factored chunk by
    chunk (left-looking over chunks) while the input arrives, the rest after
    a catch-up. Every block sees the same update / checksum sequence as the
    iteration-ordered schedule, so the factor is bit-identical and the
    reports equal; the seeded faults sit after `split` (a fault planned
    earlier makes the call wait for the whole input, tested above). Mixed
    schemes put unprotected iterations inside the chunked part (their
    successors re-encode)."""
    import ctypes
    monkeypatch.setenv("ABFT_STREAM_CHUNK", str(chunk))
    monkeypatch.setenv("ABFT_STREAM_SPLIT", str(split))
    nb = -(-n // b)
    sp = 3 * nb // 8 if split < 0 else min(split, nb - 1)
    sched = {sp: {P.ErrorKind.D0: 1}, nb - 2: {P.ErrorKind.D0: 1, P.ErrorKind.D1: 1}}
    cyc = ["full", "none", "single", "full", "none", "none", "single"]
    sch_list = ([cyc[k % len(cyc)] for k in range(nb)] if schemes == "mixed" else None)
    scheme = "full" if schemes == "mixed" else schemes
    a = P.generate_test_matrix(kind, n, 7)
    f1 = P.Factorization(kind, a, b)
    ref = [report_json(r) for r in P.run_protected(f1, scheme, sched, np.random.default_rng(7),
                                                   schemes=sch_list)]
    f2 = P.Factorization(kind, a, b)
    lib = f2._lib
    junk = np.asfortranarray(np.random.default_rng(1).standard_normal((n, n)) * 1e3)
    assert lib.abft_set_matrix(f2._ctx, junk.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), n) == 0
    af = np.asfortranarray(a, dtype=np.float64)
    assert lib.abft_set_matrix_streamed(f2._ctx, af.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                        n) == 0
    out = np.empty((n, n), order="F")
    got = [report_json(r) for r in P.run_protected(f2, scheme, sched, np.random.default_rng(7),
                                                   schemes=sch_list, out=out)]
    assert got == ref
    if schemes != "mixed":
        assert sum(len(r["locations"]) for r in got) >= 1
    assert np.array_equal(f2.m, f1.m)
    assert np.array_equal(out, f1.m)
    if kind == "qr":  # the compact-WY panels too
        assert len(f2.qr_t) == len(f1.qr_t) == nb
        for k in range(nb):
            assert np.array_equal(f2.qr_t[k], f1.qr_t[k])
            assert np.array_equal(f2._qr_vs[k], f1._qr_vs[k])


@pytest.mark.parametrize("kind", ["lu", "qr", "cholesky"])
def test_stream_input_python_api(kind):
    """Factorization.stream_input + run_protected(out=...): the public-API
    form of the streamed input (built-in chunking) gives the reports and the
    factor of the ordinary input path; fp32 likewise (SFactorization)."""
    n, b = 2048, 128
    nb = n // b
    sched = {nb // 2 + 1: {P.ErrorKind.D0: 1}}
    a = P.generate_test_matrix(kind, n, 13)
    f1 = P.Factorization(kind, a, b)
    ref = [report_json(r) for r in P.run_protected(f1, "full", sched, np.random.default_rng(13))]
    f2 = P.Factorization(kind, np.zeros((n, n)), b)
    f2.stream_input(np.asfortranarray(a))
    out = np.full((n, n), np.nan, order="F")  # every entry must arrive
    got = [report_json(r) for r in P.run_protected(f2, "full", sched, np.random.default_rng(13),
                                                   out=out)]
    assert got == ref and sum(len(r["locations"]) for r in got) == 1
    assert not np.isnan(out).any()
    assert np.array_equal(out, f2.m)
    if kind == "cholesky":  # the row blocks right of the diagonal arrive zeroed
        for k in range(nb - 1):
            assert not np.any(out[k * b:(k + 1) * b, (k + 1) * b:])
    m1 = f1.m if kind != "cholesky" else np.tril(f1.m)
    m2 = out if kind != "cholesky" else np.tril(out)
    np.testing.assert_allclose(m2, m1, rtol=0, atol=1e-12 * max(1.0, np.abs(m1).max()))
    if kind != "cholesky":
        assert np.array_equal(out, f1.m)
    s1 = P.SFactorization(kind, a, b)
    r1 = s1.run_protected("full", sched, np.random.default_rng(13))
    s2 = P.SFactorization(kind, np.zeros((n, n), dtype=np.float32), b)
    s2.stream_input(np.asfortranarray(a, dtype=np.float32))
    r2 = s2.run_protected("full", sched, np.random.default_rng(13))
    assert [r.locations for r in r1] == [r.locations for r in r2]
    if kind != "cholesky":
        assert np.array_equal(s2.m, s1.m)
