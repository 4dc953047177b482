"""GPU: the blocked factorizations and the protected iteration against the
reference's goldens (tests/golden, produced by running the reference)."""
import numpy as np
import pytest

import oracle as O
import paper_2301_03166_b200 as P
from conftest import GOLDEN, golden, report_json, sparse_reports

pytestmark = pytest.mark.gpu

EPS = 2.220446049250313e-16
KINDS = ["cholesky", "lu", "qr"]


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("n,b", [(64, 16), (96, 32), (100, 32), (128, 128), (256, 64), (512, 64)])
def test_blocked_matches_reference(kind, n, b):
    """test_linalg.py:37-50 + golden residual: residual within 16*n*eps of
    the reference's (the stated factor), and < 1e-12 as the reference test."""
    case = next(c for c in golden("linalg.json")
                if c["kind"] == kind and c["n"] == n and c["b"] == b and c["seed"] == 1)
    a = P.generate_test_matrix(kind, n, 1)
    f = P.Factorization(kind, a, b).run_all()
    res = P.residual(a, f)
    assert res < 1e-12
    assert res <= case["residual"] + 16 * n * EPS
    m = f.m
    if kind == "cholesky":
        assert np.allclose(np.tril(m), np.linalg.cholesky(a), atol=1e-9)
    elif kind == "qr":
        _, r_ref = np.linalg.qr(a)
        assert np.allclose(np.abs(np.diag(m)), np.abs(np.diag(r_ref)), rtol=1e-8)
    arrays = np.load(GOLDEN / "linalg.npz")
    key = f"{kind}_{n}_{b}"
    if key in arrays:
        assert np.allclose(m, arrays[key], rtol=1e-10, atol=1e-10)
    np.testing.assert_allclose(np.diag(m), case["diag"], rtol=1e-10, atol=1e-12)


def test_criterion1_residuals():
    worst = 0.0
    for kind in KINDS:
        for n in (128, 256, 512):
            a = P.generate_test_matrix(kind, n, 7)
            f = P.Factorization(kind, a, 64).run_all()
            worst = max(worst, P.residual(a, f))
    assert worst <= 1e-10


def test_cholesky_breakdown_raises():
    a = P.generate_test_matrix("cholesky", 32, 0)
    a[0, 0] = -1.0
    with pytest.raises(P.NumericBreakdownError):
        P.Factorization("cholesky", a, 8).run_all()


def test_lu_zero_pivot_raises():
    a = P.generate_test_matrix("lu", 32, 0)
    a[0, 0] = 0.0
    with pytest.raises(P.NumericBreakdownError):
        P.Factorization("lu", a, 8).run_all()


def test_iteration_order_enforced():
    a = P.generate_test_matrix("lu", 32, 0)
    f = P.Factorization("lu", a, 8)
    with pytest.raises(P.InvalidDimensionError):
        f.run_iteration(1)


def test_reconstruct_requires_completion():
    a = P.generate_test_matrix("qr", 64, 0)
    f = P.Factorization("qr", a, 16)
    with pytest.raises(P.NumericBreakdownError):
        f.reconstruct()


def test_qr_side_data_matches_oracle():
    a = P.generate_test_matrix("qr", 100, 3)
    f = P.Factorization("qr", a, 32).run_all()
    o = O.OracleFactorization("qr", a, 32).run_all()
    assert len(f.qr_t) == len(o.qr_t) == 4
    for k in range(4):
        np.testing.assert_allclose(f.qr_t[k], o.qr_t[k], rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose(f._qr_vs[k], o.qr_vs[k], rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("n,b", [(1024, 256), (700, 128), (256, 256), (300, 64)])
def test_qr_tensor_core_panel_matches_oracle(n, b):
    """The CholeskyQR2 + Householder-reconstruction panel (qr_panel.cu) gives
    the reference's V, T and R (linalg.py:260-300) to rounding, including the
    square last panel (the reference reflects its last column too: tau = 2)."""
    a = P.generate_test_matrix("qr", n, 5)
    f = P.Factorization("qr", a, b).run_all()
    o = O.OracleFactorization("qr", a, b).run_all()
    for k in range(len(o.qr_t)):
        np.testing.assert_allclose(f.qr_t[k], o.qr_t[k], rtol=0, atol=1e-12)
        np.testing.assert_allclose(f._qr_vs[k], o.qr_vs[k], rtol=0, atol=1e-12)
    np.testing.assert_allclose(f.m, o.m, rtol=0, atol=1e-10 * np.abs(o.m).max())
    assert P.residual(a, f) <= O.residual(a, o) + 16 * n * 2.220446049250313e-16


@pytest.mark.parametrize("case", ["zero_col", "rank_deficient", "ill_conditioned"])
def test_qr_degenerate_panel_takes_exact_fallback(case):
    """Panels whose Gram matrix is not safely positive definite (zero or
    dependent columns: the reference's normx == 0 branches, linalg.py:273-276)
    or too ill-conditioned for CholeskyQR2 run the per-column panel instead,
    and still match the reference's V / T / R."""
    n, b = 384, 64
    a = P.generate_test_matrix("qr", n, 11).copy()
    if case == "zero_col":
        a[:, 5] = 0.0
    elif case == "rank_deficient":
        a[:, 70] = 2.0 * a[:, 66] - a[:, 67]
    else:
        a[:, 130] = a[:, 129] + 1e-9 * a[:, 131]
    a = np.asfortranarray(a)
    f = P.Factorization("qr", a, b).run_all()
    o = O.OracleFactorization("qr", a, b).run_all()
    # from the dependent column on, the reflectors of a rank-deficient panel
    # are rounding noise (not comparable); an exactly zero column is exact
    k_cmp = {"zero_col": 1, "rank_deficient": 1, "ill_conditioned": 2}[case]
    for k in range(k_cmp):
        np.testing.assert_allclose(f.qr_t[k], o.qr_t[k], rtol=0, atol=1e-9)
        np.testing.assert_allclose(f._qr_vs[k], o.qr_vs[k], rtol=0, atol=1e-9)
    assert np.all(np.isfinite(f.m))
    assert P.residual(a, f) < 1e-12


def _protocol(kind, n, b, seed, scheme, counts, stop_after_fault=False):
    rng = np.random.default_rng(seed)
    nb = -(-n // b)
    k_fault = int(rng.integers(0, nb - 1))
    a = P.generate_test_matrix(kind, n, seed)
    f = P.Factorization(kind, a, b)
    reps = []
    for k in range(k_fault + 1 if stop_after_fault else nb):
        counts_k = counts if k == k_fault else None
        reps.append(report_json(P.run_numeric_iteration(f, k, scheme, counts_k, rng)))
    res = P.residual(a, f) if f.complete else None
    return k_fault, reps, res


@pytest.mark.parametrize("chunk", range(10))
def test_criterion5_all_seeds(chunk):
    """Criterion 5 (test_acceptance.py:217-256), seeds 0..999: detected /
    corrected locations bit-exact with the reference; 0D/SINGLE and 1D/FULL
    repaired (residual <= 1e-8), 1D/SINGLE flagged."""
    g = golden("crit5.json")
    E = P.ErrorKind
    for row in g["seeds"][chunk * 100:(chunk + 1) * 100]:
        seed = row["seed"]
        rng = np.random.default_rng(seed)
        k_fault = int(rng.integers(0, 7))
        a = P.generate_test_matrix("lu", 256, seed)
        for run in row["runs"]:
            f = P.Factorization("lu", a, 32)
            reps = []
            for k in range(run["iterations"]):
                counts = {E(run["kind"]): 1} if k == k_fault else None
                reps.append(report_json(P.run_numeric_iteration(f, k, run["scheme"], counts, rng)))
            assert sparse_reports(reps) == run["reports"], (seed, run["scheme"], run["kind"])
            if run["full_run"]:
                res = P.residual(a, f)
                assert res <= 1e-8
                assert res <= run["residual"] + 16 * 256 * EPS
            else:
                assert reps[-1]["uncorrectable"]


def test_multi_fault_runs_match_reference():
    for run in golden("multi.json")["runs"]:
        kf, reps, res = _protocol(run["kind"], run["n"], run["b"], run["seed"], run["scheme"],
                                  run["counts"])
        assert kf == run["k_fault"]
        assert sparse_reports(reps) == run["reports"], (run["kind"], run["scheme"], run["seed"])
        if run["residual"] <= 1e-8:
            assert res <= run["residual"] + 16 * run["n"] * EPS
        else:  # uncorrected faults: the same corrupted result (to fp noise)
            assert res == pytest.approx(run["residual"], rel=1e-3)


def test_c1_cholesky_2048_seeded_fault():
    """BASELINE config C1: Cholesky N=2048 b=256 FULL/SINGLE, seeded 0-D fault."""
    for run in golden("c1.json")["runs"]:
        kf, reps, res = _protocol("cholesky", 2048, 256, run["seed"], run["scheme"], {"0d": 1})
        assert kf == run["k_fault"]
        assert sparse_reports(reps) == run["reports"]
        assert res <= run["residual"] + 16 * 2048 * EPS


@pytest.mark.parametrize("kind", KINDS)
def test_run_protected_equals_per_iteration(kind):
    """The one-call fast path gives the same reports as run_numeric_iteration."""
    n, b, seed = 512, 64, 4
    sched = {2: {P.ErrorKind.D0: 2, P.ErrorKind.D1: 1}, 5: {P.ErrorKind.D0: 1}}
    a = P.generate_test_matrix(kind, n, seed)
    f1 = P.Factorization(kind, a, b)
    rng = np.random.default_rng(seed)
    per = [report_json(P.run_numeric_iteration(f1, k, "full", sched.get(k), rng)) for k in range(8)]
    f2 = P.Factorization(kind, a, b)
    fast = [report_json(r) for r in P.run_protected(f2, "full", sched, np.random.default_rng(seed))]
    assert per == fast
    assert abs(P.residual(a, f1) - P.residual(a, f2)) <= 1e-15


def test_snapshot_restore_roundtrip():
    a = P.generate_test_matrix("qr", 256, 2)
    f = P.Factorization("qr", a, 64)
    f.run_iteration(0)
    f.snapshot(0)
    m0 = f.m.copy()
    f.run_iteration(1)
    f.restore(0)
    assert f.k_done == 1
    f._set_qr_count(1)
    np.testing.assert_array_equal(f.m, m0)
    f.run_all()
    assert P.residual(a, f) < 1e-12


@pytest.mark.parametrize("kind", KINDS)
def test_streamed_result_equals_device_factor(kind):
    """run_protected(out=...) copies each finished column block to the host
    during the factorization: the streamed array is the final factor."""
    n, b, seed = 640, 128, 2
    a = P.generate_test_matrix(kind, n, seed)
    f = P.Factorization(kind, a, b)
    out = np.full((n, n), np.nan, order="F")
    reps = P.run_protected(f, "full", {2: {P.ErrorKind.D0: 1}}, np.random.default_rng(seed), out=out)
    np.testing.assert_array_equal(out, f.m)
    assert any(r.locations for r in reps)
