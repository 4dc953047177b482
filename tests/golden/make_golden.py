"""Freeze golden vectors by running the REFERENCE itself (this container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

The reference (`slackwise`, pure Python) is imported from /root/reference,
which does not exist on the GPU box; the vectors are committed so the oracle
and the B200 path are pinned against the reference's own outputs everywhere.
Every case mirrors a reference test or an SURVEY.md §8c golden:
  * crit5.json   — criterion 5 protocol (pkg/tests/test_acceptance.py:217-256),
                   seeds 0..999: locations, counts, residuals
  * c1.json      — BASELINE config C1: Cholesky N=2048 b=256 FULL/SINGLE,
                   seeded single 0-D fault, seeds 0..9
  * multi.json   — multi-fault protected runs, every kind x scheme
  * abft.json    — pkg/tests/test_abft.py fixtures (reports, plans)
  * plans.json   — sample_fault_plan draws (abft.py:310-333)
  * linalg.json / linalg.npz — small factorizations (test_linalg.py:37-50)
  * inputs.json  — sha256 of generate_test_matrix outputs (linalg.py:63-78)
  * simrun.json  — simulate_run(engine="numeric") summaries (the mode-flag
                   path: modeled timing, Poisson fault streams, recovery;
                   simulator.py:314-335, :408-418) under campaign-scale
                   throughput, every kind x forced scheme, seeds 0..5
                   (`make_golden.py simrun` regenerates only this file)
  * c2c3.json    — BASELINE configs C2 (LU N=8192, SINGLE and FULL) and C3
                   (QR N=8192 SINGLE), b=256, criterion-5 fault, seed 0
                   (`make_golden.py c2c3` regenerates only this file)
"""
from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import slackwise as S  # noqa: E402

OUT = Path(__file__).resolve().parent
K = S.DecompositionKind
E = S.ErrorKind
SCH = S.ChecksumScheme


def sparse(reps: list) -> list:
    """Keep only iterations whose report is not clean: [[k, report], ...]."""
    return [[k, r] for k, r in enumerate(reps)
            if r["locations"] or r["uncorrectable"] or any(r["detected"].values())]


def rep_json(r) -> dict:
    return {"detected": {k.value: int(v) for k, v in r.detected.items()},
            "corrected": {k.value: int(v) for k, v in r.corrected.items()},
            "uncorrectable": bool(r.uncorrectable),
            "locations": [[int(a), int(b), c.value, bool(d)] for a, b, c, d in r.locations]}


def protected_run(kind, n, b, seed, scheme, counts_at, stop_after=None):
    """Criterion-5 style run: rng = default_rng(seed); k_fault drawn first."""
    rng = np.random.default_rng(seed)
    nb = -(-n // b)
    k_fault = int(rng.integers(0, nb - 1))
    a = S.generate_test_matrix(kind, n, seed)
    f = S.Factorization(kind, a, b)
    reps = []
    last = nb if stop_after is None else k_fault + 1
    for k in range(last):
        counts = counts_at if k == k_fault else None
        reps.append(rep_json(S.run_numeric_iteration(f, k, scheme, counts, rng)))
    res = float(S.residual(a, f)) if f.complete else None
    return {"seed": seed, "k_fault": k_fault, "iterations": len(reps), "reports": sparse(reps),
            "residual": res}


def crit5(nseeds=1000):
    out = []
    for seed in range(nseeds):
        row = {"seed": seed}
        r1 = protected_run(K.LU, 256, 32, seed, SCH.SINGLE, {E.D0: 1})
        # crit 5 reuses the same rng across its three sub-runs; mirror it
        rng = np.random.default_rng(seed)
        nb = 8
        k_fault = int(rng.integers(0, nb - 1))
        a = S.generate_test_matrix(K.LU, 256, seed)
        subs = []
        for scheme, ek, full_run in ((SCH.SINGLE, E.D0, True), (SCH.FULL, E.D1, True),
                                     (SCH.SINGLE, E.D1, False)):
            f = S.Factorization(K.LU, a, 32)
            reps = []
            for k in range(nb if full_run else k_fault + 1):
                counts = {ek: 1} if k == k_fault else None
                reps.append(rep_json(S.run_numeric_iteration(f, k, scheme, counts, rng)))
            subs.append({"scheme": scheme.value, "kind": ek.value, "full_run": full_run,
                         "iterations": len(reps), "reports": sparse(reps),
                         "residual": float(S.residual(a, f)) if full_run else None})
        row["k_fault"] = k_fault
        row["runs"] = subs
        assert r1["k_fault"] == k_fault
        out.append(row)
    return {"n": 256, "b": 32, "kind": "lu", "protocol": "pkg/tests/test_acceptance.py:217-256",
            "seeds": out}


def c1(seeds=range(10)):
    out = []
    for scheme in (SCH.FULL, SCH.SINGLE):
        for seed in seeds:
            r = protected_run(K.CHOLESKY, 2048, 256, seed, scheme, {E.D0: 1})
            r["scheme"] = scheme.value
            out.append(r)
    return {"n": 2048, "b": 256, "kind": "cholesky", "runs": out}


def multi():
    out = []
    counts = {E.D0: 2, E.D1: 1, E.D2: 1}
    for kind in (K.CHOLESKY, K.LU, K.QR):
        for scheme in (SCH.SINGLE, SCH.FULL, SCH.NONE):
            for seed in range(8):
                for n, b in ((256, 32), (200, 64)):
                    r = protected_run(kind, n, b, seed, scheme, counts)
                    r.update({"kind": kind.value, "scheme": scheme.value, "n": n, "b": b,
                              "counts": {"0d": 2, "1d": 1, "2d": 1}})
                    out.append(r)
    return {"runs": out}


def abft_fixtures():
    def rm(n, seed):
        return np.random.default_rng(seed).uniform(-1.0, 1.0, size=(n, n))
    cases = {}
    m = rm(64, 3)
    cs = S.encode(m, 16, SCH.SINGLE)
    S.inject_faults(m, [S.InjectedFault(E.D0, 10, 37, 0.5)])
    cases["single_corrects_0d"] = rep_json(S.verify_correct(m, cs))
    m = rm(64, 4)
    cs = S.encode(m, 16, SCH.SINGLE)
    S.inject_faults(m, [S.InjectedFault(E.D1, 16, 5, 0.3, extent=4)])
    cases["single_flags_1d"] = rep_json(S.verify_correct(m, cs))
    m = rm(64, 5)
    cs = S.encode(m, 16, SCH.FULL)
    S.inject_faults(m, [S.InjectedFault(E.D1, 16, 5, 0.3, extent=4)])
    cases["full_corrects_1d_col"] = rep_json(S.verify_correct(m, cs))
    m = rm(64, 6)
    cs = S.encode(m, 16, SCH.FULL)
    S.inject_faults(m, [S.InjectedFault(E.D1, 20, 16, 0.4, orientation="row", extent=4)])
    cases["full_corrects_1d_row"] = rep_json(S.verify_correct(m, cs))
    m = rm(64, 7)
    cs = S.encode(m, 16, SCH.FULL)
    S.inject_faults(m, [S.InjectedFault(E.D2, 17, 18, 0.4, extent=3)])
    cases["full_flags_2d"] = rep_json(S.verify_correct(m, cs))
    m = rm(64, 8)
    cs = S.encode(m, 16, SCH.SINGLE)
    S.inject_faults(m, [S.InjectedFault(E.D0, 16 * i + 3, 16 * i + 7, 0.2 + i) for i in range(4)])
    cases["multi_0d_distinct_blocks"] = rep_json(S.verify_correct(m, cs))
    m = rm(64, 9)
    cs = S.encode(m, 16, SCH.FULL, r0=16, c0=32, shape=(48, 32))
    S.inject_faults(m, [S.InjectedFault(E.D0, 40, 50, 0.9)])
    cases["region_offsets"] = rep_json(S.verify_correct(m, cs))
    # SURVEY §8a quirks Q1-Q3
    for scheme in (SCH.SINGLE, SCH.FULL):
        m = rm(64, 21)
        cs = S.encode(m, 16, scheme)
        S.inject_faults(m, [S.InjectedFault(E.D0, 3, 5, 0.5), S.InjectedFault(E.D0, 9, 11, -0.7)])
        cases[f"q1_two_0d_one_block_{scheme.value}"] = rep_json(S.verify_correct(m, cs))
        m = rm(64, 22)
        cs = S.encode(m, 16, scheme)
        S.inject_faults(m, [S.InjectedFault(E.D0, 3, 5, 0.5), S.InjectedFault(E.D0, 9, 5, -0.7)])
        cases[f"q2_two_0d_one_column_{scheme.value}"] = rep_json(S.verify_correct(m, cs))
        m = rm(64, 23)
        cs = S.encode(m, 16, scheme)
        S.inject_faults(m, [S.InjectedFault(E.D2, 14, 14, 0.5, extent=4)])
        cases[f"q3_2d_corner_straddle_{scheme.value}"] = rep_json(S.verify_correct(m, cs))
    # maintained updates stay clean (test_abft.py:137-146)
    rng = np.random.default_rng(12)
    m = rng.uniform(-1, 1, size=(96, 96))
    cs = S.encode(m, 16, SCH.FULL)
    for _ in range(20):
        left = rng.uniform(-1, 1, size=(96, 8))
        right = rng.uniform(-1, 1, size=(8, 96))
        S.maintain_gemm(cs, left, right)
        m -= left @ right
    cases["no_false_positive_20_updates"] = rep_json(S.verify_correct(m, cs))
    return cases


def plans():
    out = []
    rng = np.random.default_rng(11)
    for _ in range(50):
        plan = S.sample_fault_plan(rng, {E.D0: 1, E.D1: 1, E.D2: 1}, r0=8, c0=8, rows=24,
                                   cols=24, b=8, scale=1.0, iteration=0)
        out.append([[f.kind.value, f.row, f.col, f.magnitude, f.extent, f.orientation]
                    for f in plan])
    rng = np.random.default_rng(5)
    big = []
    for scale in (0.3, 3.7, 1234.5):
        plan = S.sample_fault_plan(rng, {E.D0: 3, E.D1: 2, E.D2: 2}, r0=256, c0=512, rows=7936,
                                   cols=7680, b=256, scale=scale, iteration=1)
        big.append([[f.kind.value, f.row, f.col, f.magnitude, f.extent, f.orientation]
                    for f in plan])
    return {"small": out, "big": big}


def linalg_cases():
    js, arrays = [], {}
    for kind in (K.CHOLESKY, K.LU, K.QR):
        for n, b in ((64, 16), (96, 32), (100, 32), (128, 128), (256, 64), (512, 64)):
            a = S.generate_test_matrix(kind, n, 1)
            f = S.Factorization(kind, a, b).run_all()
            res = float(S.residual(a, f))
            js.append({"kind": kind.value, "n": n, "b": b, "seed": 1, "residual": res,
                       "diag": np.diag(f.m).tolist()})
            if n <= 100:
                arrays[f"{kind.value}_{n}_{b}"] = f.m
    for kind in (K.CHOLESKY, K.LU, K.QR):
        for n in (128, 256, 512):
            a = S.generate_test_matrix(kind, n, 7)
            f = S.Factorization(kind, a, 64).run_all()
            js.append({"kind": kind.value, "n": n, "b": 64, "seed": 7,
                       "residual": float(S.residual(a, f)), "diag": np.diag(f.m).tolist()})
    return js, arrays


def inputs():
    out = []
    for kind in (K.CHOLESKY, K.LU, K.QR):
        for n in (1, 7, 64, 256):
            for seed in (0, 1, 7):
                a = S.generate_test_matrix(kind, n, seed)
                out.append({"kind": kind.value, "n": n, "seed": seed,
                            "sha256": hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest(),
                            "fortran": bool(a.flags.f_contiguous)})
    return out


def c2c3():
    """"C2 and C3 seed 0" (b = 256 as the bench; ~2-5 min each)."""
    out = []
    for kind, scheme in ((K.LU, SCH.SINGLE), (K.LU, SCH.FULL), (K.QR, SCH.SINGLE)):
        t0 = time.time()
        r = protected_run(kind, 8192, 256, 0, scheme, {E.D0: 1})
        r.update({"kind": kind.value, "scheme": scheme.value, "n": 8192, "b": 256,
                  "counts": {"0d": 1}, "ref_seconds": round(time.time() - t0, 1)})
        print(kind.value, scheme.value, r["reports"], r["residual"], flush=True)
        out.append(r)
    return {"runs": out}


def simrun():
    import dataclasses

    from slackwise.config import SimConfig
    from slackwise.power import default_cpu_model, default_gpu_model
    from slackwise.simulator import simulate_run
    cpu = dataclasses.replace(default_cpu_model(), base_flops_per_second=5e7)
    gpu = dataclasses.replace(default_gpu_model(), base_flops_per_second=2e7, f_max_mhz=2100.0)
    out = []
    for kind in (K.CHOLESKY, K.LU, K.QR):
        for mode, r in (("bsr", 1.0), ("bsr", 0.5), ("sr", 0.0), ("original", 0.0)):
            for forced in (None, SCH.NONE, SCH.SINGLE, SCH.FULL):
                if mode != "bsr" and forced is not None:
                    continue
                for seed in range(6):
                    c = SimConfig(kind=kind, n=256, b=32, seed=seed, cpu=cpu, gpu=gpu, mode=mode,
                                  r=r, engine="numeric", recovery="recompute")
                    sm, recs = simulate_run(c, forced_scheme=forced)
                    out.append({
                        "kind": kind.value, "mode": mode, "r": r, "seed": seed,
                        "forced": None if forced is None else forced.value,
                        "total_time_s": sm.total_time_s, "total_energy_j": sm.total_energy_j,
                        "correct": sm.correct, "residual": sm.residual,
                        "unrecoverable": sm.unrecoverable, "breakdown": sm.breakdown,
                        "faults_injected": {k.value if hasattr(k, "value") else k: int(v)
                                            for k, v in sm.faults_injected.items()},
                        "faults_detected": sm.faults_detected,
                        "faults_corrected": sm.faults_corrected,
                        "iterations_completed": sm.iterations_completed,
                        "abft_modes": [getattr(rc, "abft_mode", None) for rc in recs]})
    return {"runs": out}


def main():
    if sys.argv[1:] == ["simrun"]:
        (OUT / "simrun.json").write_text(json.dumps(simrun()))
        return
    if sys.argv[1:] == ["c2c3"]:
        (OUT / "c2c3.json").write_text(json.dumps(c2c3()))
        return
    t0 = time.time()
    (OUT / "inputs.json").write_text(json.dumps(inputs()))
    (OUT / "plans.json").write_text(json.dumps(plans()))
    (OUT / "abft.json").write_text(json.dumps(abft_fixtures(), indent=0))
    js, arrays = linalg_cases()
    (OUT / "linalg.json").write_text(json.dumps(js))
    np.savez_compressed(OUT / "linalg.npz", **arrays)
    print("small goldens", time.time() - t0)
    (OUT / "multi.json").write_text(json.dumps(multi()))
    print("multi", time.time() - t0)
    (OUT / "c1.json").write_text(json.dumps(c1()))
    print("c1", time.time() - t0)
    (OUT / "crit5.json").write_text(json.dumps(crit5()))
    print("crit5", time.time() - t0)
    (OUT / "c2c3.json").write_text(json.dumps(c2c3()))
    print("c2c3", time.time() - t0)


if __name__ == "__main__":
    main()
