"""GPU: the BASELINE configurations the smaller parity tests do not reach.

* C2 (LU N=8192, SINGLE and FULL) and C3 (QR N=8192 SINGLE), b=256, the
  criterion-5 fault protocol, seed 0: reports bit-exact with the goldens
  frozen by running the reference itself (tests/golden/c2c3.json,
  tests/golden/make_golden.py c2c3), residual <= reference + 16 n eps.
  Both the per-iteration path (run_numeric_iteration, the reference's call)
  and the one-call fast path (run_protected) are checked.
* C4 (N=32768, b=256) for all three kinds: size-independent properties,
  since the reference takes hours there. A clean FULL run reports nothing
  (no false positives over ~128^2/2 block checks per iteration), and the
  criterion-5 fault lands exactly where the oracle's draws (the reference's
  sample_fault_plan order) put it and is corrected; the factor reconstructs
  A to ~n eps.
"""
import copy
import ctypes

import numpy as np
import pytest

import paper_2301_03166_b200 as P
from conftest import golden, report_json, sparse_reports
from paper_2301_03166_b200.abft import draw_plan
from paper_2301_03166_b200.simulator import _tmu_region

pytestmark = pytest.mark.gpu
EPS = 2.220446049250313e-16


@pytest.mark.parametrize("idx", range(3))
@pytest.mark.parametrize("path", ["per_iteration", "one_call"])
def test_c2_c3_match_reference_goldens(idx, path):
    run = golden("c2c3.json")["runs"][idx]
    n, b, seed = run["n"], run["b"], run["seed"]
    rng = np.random.default_rng(seed)
    nb = -(-n // b)
    k_fault = int(rng.integers(0, nb - 1))
    assert k_fault == run["k_fault"]
    a = P.generate_test_matrix(run["kind"], n, seed)
    f = P.Factorization(run["kind"], a, b)
    if path == "per_iteration":
        reps = [report_json(P.run_numeric_iteration(
            f, k, run["scheme"], {"0d": 1} if k == k_fault else None, rng)) for k in range(nb)]
    else:
        reps = [report_json(r) for r in
                P.run_protected(f, run["scheme"], {k_fault: {"0d": 1}}, rng)]
    assert sparse_reports(reps) == run["reports"], (run["kind"], run["scheme"])
    res = P.residual(a, f)
    assert res <= run["residual"] + 16 * n * EPS, (res, run["residual"])


def _c4_factorization(kind, n, b, seed):
    if kind == "cholesky":
        # host PCG64 draws (bit-identical), SPD product a a^T + n I on the GPU
        # (the host product alone takes ~6 minutes at this size)
        host = np.asfortranarray(np.random.default_rng(seed).uniform(-1.0, 1.0, size=(n, n)))
        f = P.Factorization(kind, host, b, keep_input=True)
        P.linalg.check(f._lib.abft_make_spd(f._ctx))
        f._dirty()
    else:
        f = P.Factorization(kind, P.generate_test_matrix(kind, n, seed), b, keep_input=True)
    return f


@pytest.mark.parametrize("kind", ["lu", "cholesky", "qr"])
def test_c4_n32768_clean_and_seeded_fault(kind):
    n, b, seed = 32768, 256, 0
    f = _c4_factorization(kind, n, b, seed)
    reps = P.run_protected(f, "full")
    assert all(not r.locations and not r.uncorrectable for r in reps)
    # criterion-5 fault: where the reference's draws put it
    rng = np.random.default_rng(seed)
    k_fault = int(rng.integers(0, -(-n // b) - 1))
    r0, c0, rows, cols = _tmu_region(kind, n, b, k_fault)
    want = draw_plan(copy.deepcopy(rng), {"0d": 1}, r0, c0, rows, cols, b)[0]
    P.linalg.check(f._lib.abft_reset(f._ctx))
    f._dirty()
    reps = P.run_protected(f, "full", {k_fault: {"0d": 1}}, rng)
    locs = [(r, c, k.value, fl) for rep in reps for r, c, k, fl in rep.locations]
    assert locs == [(want["row"], want["col"], "0d", True)], (k_fault, locs)
    out = ctypes.c_double(0.0)
    P.linalg.check(f._lib.abft_residual(f._ctx, None, n, ctypes.byref(out)))
    assert out.value <= 64 * n * EPS, out.value
