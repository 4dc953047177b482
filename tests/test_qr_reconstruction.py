"""CPU: the algebra of the tensor-core QR panel (csrc/qr_panel.cu) restated in
numpy -- CholeskyQR2 + Householder reconstruction with the sign-shifted LU --
against the reference's per-column Householder panel (the oracle's restatement
of linalg.py:260-300). Pins the sign rule, the T formula and the square last
panel (tau = 2) independently of the GPU."""
import numpy as np
import pytest

import oracle as O


def _lu_sign(x):
    x = x.copy()
    w = x.shape[0]
    s = np.zeros(w)
    for c in range(w):
        s[c] = 1.0 if x[c, c] < 0 else -1.0
        x[c, c] -= s[c]
        x[c + 1:, c] /= x[c, c]
        x[c + 1:, c + 1:] -= np.outer(x[c + 1:, c], x[c, c + 1:])
    return x, s


def _tensor_core_panel(a):
    """qr_panel_factor's sequence of GEMMs and small factorizations."""
    m, w = a.shape
    g1 = a.T @ a
    l1 = np.linalg.cholesky(g1)
    l1i = np.linalg.inv(l1)
    q1 = a @ l1i.T
    g2 = q1.T @ q1
    assert w * np.abs(g2 - np.eye(w)).max() < 0.5  # the device's orthogonality gate
    l2 = np.linalg.cholesky(g2)
    l2i = np.linalg.inv(l2)
    r = l2.T @ l1.T
    x, s = _lu_sign(q1[:w] @ l2i.T)
    y = np.tril(x, -1) + np.eye(w)
    u = np.triu(x)
    v = np.zeros((m, w))
    v[:w] = y
    v[w:] = q1[w:] @ (l2i.T @ np.linalg.inv(u))
    t = u @ (-(s[:, None]) * np.linalg.inv(y).T)
    p = np.zeros((m, w))
    p[:w] = np.triu(s[:, None] * r)
    return p, v, t


@pytest.mark.parametrize("m,w", [(300, 64), (64, 64), (1000, 50), (513, 128), (256, 256)])
def test_reconstruction_equals_reference_panel(m, w):
    rng = np.random.default_rng(m + w)
    a = np.asfortranarray(rng.uniform(-1.0, 1.0, (m, w)))
    # the oracle's panel on exactly this block (k = 0 of an m x m matrix whose
    # first w columns are a)
    full = np.zeros((m, m))
    full[:, :w] = a
    f = O.OracleFactorization("qr", np.asfortranarray(full), w)
    f.pd(0)
    p, v, t = _tensor_core_panel(a)
    np.testing.assert_allclose(p, f.m[:, :w], rtol=0, atol=1e-13 * max(1.0, np.abs(p).max()))
    np.testing.assert_allclose(v, f.qr_vs[0], rtol=0, atol=1e-12)
    np.testing.assert_allclose(t, f.qr_t[0], rtol=0, atol=1e-12)
