"""GPU: LU with partial pivoting (option; the reference factors unpivoted,
linalg.py:230-238). Parity with LAPACK dgetrf (scipy.linalg.lu_factor: the
same pivots, factors to rounding) on general matrices, and the ABFT protocol
on the pivoted path (seeded faults located at their planned positions and
corrected, clean runs report nothing)."""
import numpy as np
import pytest
import scipy.linalg as sl

import paper_2301_03166_b200 as P

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,b", [(512, 128), (640, 256), (300, 64), (256, 256)])
def test_pivoted_lu_matches_lapack(n, b):
    a = np.asfortranarray(np.random.default_rng(n + b).uniform(-1.0, 1.0, (n, n)))
    f = P.Factorization("lu", a, b, pivoting=True).run_all()
    lu, piv = sl.lu_factor(a)
    np.testing.assert_array_equal(f.piv, piv)
    np.testing.assert_allclose(f.m, lu, rtol=0, atol=1e-11 * np.abs(lu).max())
    assert P.residual(a, f) < 64 * n * 2.220446049250313e-16


def test_pivoting_is_a_no_op_on_reference_inputs():
    """The reference's LU inputs are row-diagonally dominant (linalg.py:63-78):
    partial pivoting keeps every diagonal pivot, the factor equals the
    unpivoted one."""
    n, b = 512, 128
    a = P.generate_test_matrix("lu", n, 4)
    f1 = P.Factorization("lu", a, b, pivoting=True).run_all()
    f0 = P.Factorization("lu", a, b).run_all()
    np.testing.assert_array_equal(f1.piv, np.arange(n))
    np.testing.assert_allclose(f1.m, f0.m, rtol=0, atol=1e-14 * np.abs(f0.m).max())  # rounding only


@pytest.mark.parametrize("scheme", ["full", "single"])
def test_pivoted_lu_abft_locates_and_corrects(scheme):
    n, b = 768, 128
    a = np.asfortranarray(np.random.default_rng(7).uniform(-1.0, 1.0, (n, n)))
    nb = n // b
    for seed in range(6):
        rng = np.random.default_rng(seed)
        k_fault = int(rng.integers(0, nb - 1))
        f = P.Factorization("lu", a, b, pivoting=True)
        reps = P.run_protected(f, scheme, {k_fault: {P.ErrorKind.D0: 1}}, rng)
        locs = [loc for r in reps for loc in r.locations]
        assert len(locs) == 1 and locs[0][3], (seed, locs)
        r0, c0 = (k_fault + 1) * b, (k_fault + 1) * b
        assert r0 <= locs[0][0] < n and c0 <= locs[0][1] < n
        assert P.residual(a, f) < 64 * n * 2.220446049250313e-16
    f = P.Factorization("lu", a, b, pivoting=True)
    assert all(r.clean for r in P.run_protected(f, "full", {}, np.random.default_rng(0)))


def test_pivoted_singular_raises():
    n, b = 256, 64
    a = np.asfortranarray(np.random.default_rng(3).uniform(-1.0, 1.0, (n, n)))
    a[:, 100] = 0.0
    with pytest.raises(P.NumericBreakdownError):
        P.Factorization("lu", a, b, pivoting=True).run_all()
