"""GPU: the reference's own test suite (pkg/tests, all 137 tests) passes with
the B200 backend installed into the reference package (SURVEY.md §7 step 2,
§8b drop-in boundary). Needs the reference installed into baseline/_ref (see
tools/reference_suite.py); skipped where it was not installed."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not (REF / "_tests").is_dir(), reason="reference not installed in baseline/_ref")
def test_reference_suite_passes_with_b200_backend_installed():
    out = subprocess.run([sys.executable, str(ROOT / "tools" / "reference_suite.py")],
                         capture_output=True, text=True, timeout=1800, cwd=str(ROOT))
    last = out.stdout.strip().splitlines()[-1]
    info = json.loads(last)
    assert info["exit_code"] == 0, out.stdout[-4000:] + out.stderr[-2000:]
    # the hot path really ran on the GPU
    assert info["b200_kernel_launches"] > 1000, info


@pytest.mark.skipif(not (REF / "slackwise").is_dir(), reason="reference not installed in baseline/_ref")
def test_simulate_run_numeric_parity_mode():
    """The modeled-timing parity mode of the mode-flag path: the reference's
    own simulate_run(engine="numeric") (modeled t_tmu, Poisson fault draws,
    recovery policy; simulator.py:314-335, :408-481) driving the B200 hot path
    through install() reproduces the reference's fault streams and outcomes
    bit for bit (tests/golden/simrun.json, frozen from the reference run on
    the CPU): injected / detected / corrected counts, correctness, per-
    iteration schemes, modeled time and energy; residual to 16 n eps."""
    import sys as _sys
    _sys.path.insert(0, str(REF))
    import paper_2301_03166_b200 as P
    from conftest import golden
    import slackwise
    from slackwise.abft import ChecksumScheme
    from slackwise.config import SimConfig
    from slackwise.linalg import DecompositionKind
    from slackwise.power import default_cpu_model, default_gpu_model
    import dataclasses
    assert P.install("slackwise")
    try:
        from slackwise.simulator import simulate_run
        assert slackwise.simulator.run_numeric_iteration is P.run_numeric_iteration
        cpu = dataclasses.replace(default_cpu_model(), base_flops_per_second=5e7)
        gpu = dataclasses.replace(default_gpu_model(), base_flops_per_second=2e7,
                                  f_max_mhz=2100.0)
        for g in golden("simrun.json")["runs"]:
            c = SimConfig(kind=DecompositionKind(g["kind"]), n=256, b=32, seed=g["seed"],
                          cpu=cpu, gpu=gpu, mode=g["mode"], r=g["r"], engine="numeric",
                          recovery="recompute")
            forced = None if g["forced"] is None else ChecksumScheme(g["forced"])
            sm, recs = simulate_run(c, forced_scheme=forced)
            key = (g["kind"], g["mode"], g["r"], g["forced"], g["seed"])
            got_inj = {getattr(k, "value", k): int(v) for k, v in sm.faults_injected.items()}
            assert got_inj == g["faults_injected"], key
            assert (sm.faults_detected, sm.faults_corrected) == (g["faults_detected"],
                                                                 g["faults_corrected"]), key
            assert (sm.correct, sm.unrecoverable, sm.breakdown) == (g["correct"],
                                                                    g["unrecoverable"],
                                                                    g["breakdown"]), key
            assert sm.iterations_completed == g["iterations_completed"], key
            assert [rc.abft_mode for rc in recs] == g["abft_modes"], key
            assert sm.total_time_s == g["total_time_s"], key
            assert sm.total_energy_j == g["total_energy_j"], key
            if g["correct"]:
                assert sm.residual <= g["residual"] + 16 * 256 * 2.220446049250313e-16, key
            else:
                assert sm.residual == pytest.approx(g["residual"], rel=1e-3), key
    finally:
        P.uninstall()
