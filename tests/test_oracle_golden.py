"""The CPU oracle (oracle/) reproduces the REFERENCE's own outputs, frozen in
tests/golden/ by tests/golden/make_golden.py (run against /root/reference).
CPU only: this pins the checker before it is used against the B200 path."""
import hashlib

import numpy as np
import pytest

import oracle as O
from conftest import GOLDEN, golden, report_json, sparse_reports


def run_protocol(kind, n, b, seed, scheme, counts, stop_after_fault=False):
    rng = np.random.default_rng(seed)
    nb = -(-n // b)
    k_fault = int(rng.integers(0, nb - 1))
    a = O.generate_test_matrix(kind, n, seed)
    f = O.OracleFactorization(kind, a, b)
    reps = []
    for k in range(k_fault + 1 if stop_after_fault else nb):
        reps.append(report_json(O.protected_iteration(
            f, k, scheme, counts if k == k_fault else None, rng)))
    res = O.residual(a, f) if f.k_done == nb else None
    return k_fault, reps, res


def test_inputs_bit_exact():
    for case in golden("inputs.json"):
        a = O.generate_test_matrix(case["kind"], case["n"], case["seed"])
        assert a.flags.f_contiguous == case["fortran"]
        assert hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest() == case["sha256"]


def test_fault_plan_draws_match_reference():
    g = golden("plans.json")
    rng = np.random.default_rng(11)
    for want in g["small"]:
        got = O.draw_fault_plan(rng, {"0d": 1, "1d": 1, "2d": 1}, 8, 8, 24, 24, 8)
        assert [[d["kind"], d["row"], d["col"], O.magnitude(d["u"], d["negate"], 1.0),
                 d["extent"], d["orientation"]] for d in got] == want
    rng = np.random.default_rng(5)
    for scale, want in zip((0.3, 3.7, 1234.5), g["big"]):
        got = O.draw_fault_plan(rng, {"0d": 3, "1d": 2, "2d": 2}, 256, 512, 7936, 7680, 256)
        assert [[d["kind"], d["row"], d["col"], O.magnitude(d["u"], d["negate"], scale),
                 d["extent"], d["orientation"]] for d in got] == want


@pytest.mark.parametrize("case", list(golden("abft.json")))
def test_abft_fixture_reports(case):
    """pkg/tests/test_abft.py fixtures + SURVEY §8a quirks Q1-Q3."""
    rm = lambda n, s: np.random.default_rng(s).uniform(-1.0, 1.0, size=(n, n))  # noqa: E731
    want = golden("abft.json")[case]
    F = lambda kind, r, c, mag, **kw: dict(kind=kind, row=r, col=c, magnitude=mag, **kw)  # noqa
    spec = {
        "single_corrects_0d": (3, "single", {}, [F("0d", 10, 37, 0.5)]),
        "single_flags_1d": (4, "single", {}, [F("1d", 16, 5, 0.3, extent=4)]),
        "full_corrects_1d_col": (5, "full", {}, [F("1d", 16, 5, 0.3, extent=4)]),
        "full_corrects_1d_row": (6, "full", {}, [F("1d", 20, 16, 0.4, orientation="row", extent=4)]),
        "full_flags_2d": (7, "full", {}, [F("2d", 17, 18, 0.4, extent=3)]),
        "multi_0d_distinct_blocks": (8, "single", {}, [F("0d", 16 * i + 3, 16 * i + 7, 0.2 + i) for i in range(4)]),
        "region_offsets": (9, "full", dict(r0=16, c0=32, shape=(48, 32)), [F("0d", 40, 50, 0.9)]),
    }
    for sch in ("single", "full"):
        spec[f"q1_two_0d_one_block_{sch}"] = (21, sch, {}, [F("0d", 3, 5, 0.5), F("0d", 9, 11, -0.7)])
        spec[f"q2_two_0d_one_column_{sch}"] = (22, sch, {}, [F("0d", 3, 5, 0.5), F("0d", 9, 5, -0.7)])
        spec[f"q3_2d_corner_straddle_{sch}"] = (23, sch, {}, [F("2d", 14, 14, 0.5, extent=4)])
    if case == "no_false_positive_20_updates":
        rng = np.random.default_rng(12)
        m = rng.uniform(-1, 1, size=(96, 96))
        cs = O.encode(m, 16, "full")
        for _ in range(20):
            left = rng.uniform(-1, 1, size=(96, 8))
            right = rng.uniform(-1, 1, size=(8, 96))
            O.maintain(cs, left, right)
            m -= left @ right
        assert O.verify(m, cs).to_json() == want
        return
    seed, scheme, kw, faults = spec[case]
    m = rm(64, seed)
    orig = m.copy()
    cs = O.encode(m, 16, scheme, **kw)
    O.inject(m, faults)
    rep = O.verify(m, cs)
    assert rep.to_json() == want
    if not rep.uncorrectable and rep.corrected["0d"] + rep.corrected["1d"] == rep.detected["0d"] + rep.detected["1d"]:
        assert np.allclose(m, orig, atol=1e-12)


CRIT5 = golden("crit5.json")


@pytest.mark.parametrize("chunk", range(4))
def test_criterion5_locations(chunk):
    """First 200 criterion-5 seeds: every location and count equals the
    reference's (pkg/tests/test_acceptance.py:217-256)."""
    for row in CRIT5["seeds"][chunk * 50:(chunk + 1) * 50]:
        seed = row["seed"]
        rng = np.random.default_rng(seed)
        k_fault = int(rng.integers(0, 7))
        assert k_fault == row["k_fault"]
        a = O.generate_test_matrix("lu", 256, seed)
        for run in row["runs"]:
            f = O.OracleFactorization("lu", a, 32)
            reps = []
            for k in range(run["iterations"]):
                counts = {run["kind"]: 1} if k == k_fault else None
                reps.append(report_json(O.protected_iteration(f, k, run["scheme"], counts, rng)))
            assert sparse_reports(reps) == run["reports"], (seed, run["scheme"], run["kind"])
            if run["full_run"]:
                res = O.residual(a, f)
                assert res <= 1e-8
                assert abs(res - run["residual"]) <= 1e-14


def test_multi_fault_runs():
    for run in golden("multi.json")["runs"]:
        counts = run["counts"]
        kf, reps, res = run_protocol(run["kind"], run["n"], run["b"], run["seed"], run["scheme"], counts)
        assert kf == run["k_fault"]
        assert sparse_reports(reps) == run["reports"], (run["kind"], run["scheme"], run["seed"])
        assert res == pytest.approx(run["residual"], rel=1e-6, abs=1e-14)


def test_c1_cholesky_2048_full():
    """BASELINE config C1 (Cholesky N=2048 b=256, seeded single fault)."""
    g = golden("c1.json")
    for run in g["runs"][:6] + g["runs"][10:14]:
        kf, reps, res = run_protocol("cholesky", 2048, 256, run["seed"], run["scheme"], {"0d": 1})
        assert kf == run["k_fault"]
        assert sparse_reports(reps) == run["reports"]
        assert res == pytest.approx(run["residual"], rel=1e-3, abs=1e-15)


def test_small_factorizations():
    arrays = np.load(GOLDEN / "linalg.npz")
    for case in golden("linalg.json"):
        a = O.generate_test_matrix(case["kind"], case["n"], case["seed"])
        f = O.OracleFactorization(case["kind"], a, case["b"]).run_all()
        res = O.residual(a, f)
        assert res < 1e-12
        assert res == pytest.approx(case["residual"], rel=1e-6, abs=1e-16)
        key = f"{case['kind']}_{case['n']}_{case['b']}"
        if key in arrays and case["seed"] == 1:
            assert np.allclose(f.m, arrays[key], rtol=1e-12, atol=1e-12)


def test_oracle_q5_full_two_bad_columns_no_bad_row_raises():
    """Quirk Q5: FULL verification with row sums intact and two bad column
    sums raises IndexError in the reference (abft.py:267; reproduced by
    running slackwise.abft on this input when the reference is importable)."""
    n, b = 64, 16
    m = np.random.default_rng(21).uniform(-1.0, 1.0, (n, n))
    cs = O.encode(m, b, "full")
    m[5, 2] += 0.5
    m[5, 9] -= 0.5
    with pytest.raises(IndexError):
        O.verify(m, cs)
