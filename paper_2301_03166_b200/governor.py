"""Run modes, adaptive ABFT and bi-directional slack reclamation on the B200
(SURVEY.md §8f rows 1-3).

The reference drives the protected iteration from a *modeled* run engine
(/root/reference/pkg/src/slackwise/simulator.py:203-589): per iteration it
predicts the CPU-side (PD + PU + transfer) and GPU-side (TMU) times, picks
clocks and a checksum scheme (scheduler.py:44-146, coverage.py:207-230),
draws Poisson fault counts for the chosen GPU clock (simulator.py:408-418),
runs the numeric iteration and books time and energy.

Here the same loop runs over the B200 path with MEASURED task times:

* the two "devices" of the paper are the panel stream (PD + PU, the
  reference's CPU side) and the trailing-update stream (TMU + its ABFT
  work, the GPU side); their per-iteration device times come from CUDA
  events inside libabft_b200.so (abft_profile_read);
* the history predictor (predictor.py:40-137), decide_sr / decide_bsr
  (scheduler.py:64-146) and the adaptive governor adaptive_abft
  (coverage.py:137-230) are restated below and fed with those times;
* clocks are a *virtual* DVFS domain: B200 application clocks are
  root-gated and must not be changed on these hosts, so the chosen
  frequencies drive the synthetic fault process (the reference's
  ErrorRateTable, coverage.py:24-86) and are recorded, not applied;
* energy is the NVML TotalEnergyConsumption delta of the GPU (J), not the
  modeled ledger (power.py:196-227).

The mode flags are the reference's (config.py:30-39): ``original`` and
``r2h`` run unprotected at base clocks, ``sr`` reclaims slack downward only,
``bsr`` overclocks the critical side under adaptive SINGLE/FULL checksums.

Two engines. ``engine="iteration"`` (default) is the reference's loop one
iteration at a time (snapshots + recompute recovery, a host synchronisation
per iteration, no look-ahead). ``engine="stream"`` (run_mode_streamed) runs
the modes on the one-call look-ahead path with a PHYSICAL lever: the panel
work of iteration k+1 runs on a side stream beside the update of k, and the
decision's reclaimed slack becomes the number of SMs left to that side stream
(abft_set_side_sms) -- the stream with slack gets fewer SMs, the critical one
more -- so the modes change measured time and NVML energy. Its decisions use
the history predictor over the per-iteration times of a calibration pass;
fault counts are drawn up front from the predicted update times; an
uncorrectable event falls back to the iteration engine (recompute recovery).
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np

from .abft import ChecksumScheme, ErrorKind
from .linalg import DecompositionKind, Factorization, _value, check, compute_flops, residual
from .simulator import run_numeric_iteration

MODES = ("original", "r2h", "sr", "bsr")                     # config.py:21
MODE_FLAGS = {                                               # config.py:30-39
    "original": {"reclaim_slack": False, "overclock": False,
                 "autoboost": False, "col_ft": False, "row_ft": False},
    "r2h":      {"reclaim_slack": False, "overclock": False,
                 "autoboost": True, "col_ft": False, "row_ft": False},
    "sr":       {"reclaim_slack": True, "overclock": False,
                 "autoboost": False, "col_ft": False, "row_ft": False},
    "bsr":      {"reclaim_slack": True, "overclock": True,
                 "autoboost": False, "col_ft": True, "row_ft": True},
}
RECOVERY_POLICIES = ("recompute", "abort", "continue")       # config.py:23
MAX_RECOVERY_RETRIES = 5                                     # simulator.py:34
FREQUENCY_GRID_MHZ = 100.0                                   # coverage.py:21
HISTORY_WEIGHTS = (0.5, 0.25, 0.125, 0.125)                  # predictor.py:18-19


def mode_from_flags(reclaim_slack: bool, overclock: bool, autoboost: bool) -> str:
    """config.py:50-57."""
    for mode, flags in MODE_FLAGS.items():
        if (flags["reclaim_slack"] == reclaim_slack and flags["overclock"] == overclock
                and flags["autoboost"] == autoboost):
            return mode
    raise ValueError("flag combination matches no run mode")


# ---------------------------------------------------------------------------
# error-rate model and coverage (coverage.py:24-230)
# ---------------------------------------------------------------------------
@dataclass
class ErrorRateTable:
    """Piecewise-linear errors/s vs MHz per ErrorKind (coverage.py:24-76)."""
    breakpoints: dict = field(default_factory=dict)

    def __post_init__(self):
        clean = {}
        for kind in ErrorKind:
            pts = sorted((float(f), float(r))
                         for f, r in self.breakpoints.get(kind, self.breakpoints.get(kind.value, [])))
            if any(r < 0 for _, r in pts):
                raise ValueError("negative error rate")
            if any(pts[i + 1][1] < pts[i][1] for i in range(len(pts) - 1)):
                raise ValueError("error rate must be non-decreasing in frequency")
            clean[kind] = pts
        self.breakpoints = clean

    def rate(self, f: float, kind: ErrorKind) -> float:
        pts = self.breakpoints.get(kind, [])
        if not pts:
            return 0.0
        xs = [p[0] for p in pts]
        ys = [p[1] for p in pts]
        if f <= xs[0]:
            return 0.0 if ys[0] == 0.0 or f < xs[0] else ys[0]
        return float(np.interp(f, xs, ys))

    def rates(self, f: float) -> tuple:
        return tuple(self.rate(f, k) for k in ErrorKind)

    def fault_free(self, f: float) -> bool:
        return all(r == 0.0 for r in self.rates(f))


def default_gpu_rate_table() -> ErrorRateTable:
    """coverage.py:79-86 (synthetic overclocking SDC curves)."""
    return ErrorRateTable({ErrorKind.D0: [(1900.0, 0.0), (2200.0, 2.0)],
                           ErrorKind.D1: [(1900.0, 0.0), (2200.0, 0.5)],
                           ErrorKind.D2: [(2100.0, 0.0), (2200.0, 0.05)]})


def scaled_rate_table(factor: float, table: ErrorRateTable | None = None) -> ErrorRateTable:
    """The table with every rate multiplied by `factor`: the default rates
    are per second of the reference's modeled (slow) devices; B200 update
    intervals are ~1e4x shorter, so campaigns that want faults to actually
    occur scale the rates up."""
    t = table or default_gpu_rate_table()
    return ErrorRateTable({k: [(f, r * factor) for f, r in pts] for k, pts in t.breakpoints.items()})


@dataclass(frozen=True)
class CoverageParams:
    """coverage.py:93-108."""
    s_slots: int
    fc_desired: float = 0.999999

    @staticmethod
    def for_matrix(n: int, b: int, fc_desired: float = 0.999999) -> "CoverageParams":
        nb = math.ceil(n / b)
        return CoverageParams(s_slots=nb * nb, fc_desired=fc_desired)


def _pmf(mean: float, k_max: int) -> np.ndarray:
    out = np.empty(k_max + 1)
    out[0] = math.exp(-mean)
    for k in range(1, k_max + 1):
        out[k] = out[k - 1] * mean / k
    return out


def _slot_products(s: int) -> np.ndarray:
    probs = np.empty(s + 1)
    probs[0] = 1.0
    for m in range(1, s + 1):
        probs[m] = probs[m - 1] * (s - (m - 1)) / s
    return probs


def fc_single(table: ErrorRateTable, params: CoverageParams, f: float, t: float) -> float:
    """coverage.py:137-147."""
    if t <= 0:
        raise ValueError("interval must be positive")
    l0, l1, l2 = table.rates(f)
    s = params.s_slots
    fc = float(_pmf(l0 * t, s) @ _slot_products(s)) * math.exp(-l1 * t) * math.exp(-l2 * t)
    return min(1.0, fc)


def fc_full(table: ErrorRateTable, params: CoverageParams, f: float, t: float) -> float:
    """coverage.py:150-162."""
    if t <= 0:
        raise ValueError("interval must be positive")
    l0, l1, l2 = table.rates(f)
    s = params.s_slots
    combined = np.convolve(_pmf(l0 * t, s), _pmf(l1 * t, s))[:s + 1]
    return min(1.0, float(combined @ _slot_products(s)) * math.exp(-l2 * t))


@dataclass(frozen=True)
class AdaptiveDecision:
    frequency: float
    single_check: bool
    full_check: bool


def adaptive_abft(params: CoverageParams, table: ErrorRateTable, f_desired: float,
                  f_base: float, t_predicted: float, f_floor: float = 0.0) -> AdaptiveDecision:
    """Cheapest scheme certifying fc_desired, stepping the clock down
    (coverage.py:207-230, the paper's Algorithm 1)."""
    f = f_desired
    while not table.fault_free(f):
        t_proj = t_predicted * f_base / f
        if fc_single(table, params, f, t_proj) >= params.fc_desired:
            return AdaptiveDecision(f, True, False)
        if fc_full(table, params, f, t_proj) >= params.fc_desired:
            return AdaptiveDecision(f, False, True)
        if f - FREQUENCY_GRID_MHZ < f_floor:
            return AdaptiveDecision(f, False, True)
        f -= FREQUENCY_GRID_MHZ
    return AdaptiveDecision(f, False, False)


# ---------------------------------------------------------------------------
# clock domains and decisions (power.py:20-64, scheduler.py:25-146)
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class ClockDomain:
    """A (virtual) DVFS domain: the reference ProcessorModel's frequency
    handling (power.py:52-60). ``alpha_default`` is the guardband factor."""
    name: str
    f_base_mhz: float
    f_min_mhz: float
    f_max_mhz: float
    alpha_default: float = 1.0
    f_step_mhz: float = 100.0

    def clamp(self, f: float) -> float:
        return min(self.f_max_mhz, max(self.f_min_mhz, f))

    def round_up_to_grid(self, f: float) -> float:
        return self.clamp(math.ceil(f / self.f_step_mhz - 1e-9) * self.f_step_mhz)


def panel_domain() -> ClockDomain:
    """The paper's CPU side (power.py:230-234 frequencies)."""
    return ClockDomain("panel", 3500.0, 800.0, 4500.0, 0.92)


def update_domain() -> ClockDomain:
    """The paper's GPU side (power.py:237-241 frequencies), against which the
    default rate table is defined."""
    return ClockDomain("update", 1300.0, 300.0, 2200.0, 0.90)


@dataclass(frozen=True)
class ScheduleDecision:
    f_cpu_mhz: float
    f_gpu_mhz: float
    alpha_cpu: float
    alpha_gpu: float
    single_check: bool
    full_check: bool
    skipped: bool
    idle_at_min: bool


def decide_sr(cpu: ClockDomain, gpu: ClockDomain, t_cpu: float, t_gpu: float,
              t_tr: float) -> ScheduleDecision:
    """scheduler.py:64-81 (no DVFS latency: the domains are virtual)."""
    slack = t_gpu - t_cpu - t_tr
    f_cpu, f_gpu = cpu.f_base_mhz, gpu.f_base_mhz
    if slack > 0.0:
        f_cpu = max(cpu.f_min_mhz, cpu.round_up_to_grid(cpu.f_base_mhz * t_cpu / (t_cpu + slack)))
    elif slack < 0.0 and t_gpu > 0.0:
        f_gpu = max(gpu.f_min_mhz, gpu.round_up_to_grid(gpu.f_base_mhz * t_gpu / (t_gpu - slack)))
    return ScheduleDecision(f_cpu, f_gpu, 1.0, 1.0, False, False, False, True)


def decide_bsr(cpu: ClockDomain, gpu: ClockDomain, t_cpu: float, t_gpu: float, t_tr: float,
               r: float, coverage: CoverageParams | None, table: ErrorRateTable | None,
               previous: ScheduleDecision | None = None) -> ScheduleDecision:
    """scheduler.py:84-146 (Algorithm 2 with the adaptive governor)."""
    if not 0.0 <= r <= 1.0:
        raise ValueError("reclamation ratio must be in [0, 1]")
    slack = t_gpu - t_cpu - t_tr
    if slack > 0.0:
        t_gpu_des = t_gpu - slack * r
        t_cpu_des = t_gpu_des - t_tr
    else:
        t_cpu_des = t_cpu - abs(slack) * r
        t_gpu_des = t_cpu_des + t_tr
    if t_gpu <= 0.0:
        f_gpu = gpu.f_base_mhz
    elif t_gpu_des > 0.0:
        f_gpu = gpu.round_up_to_grid(gpu.f_base_mhz * t_gpu / t_gpu_des)
    else:
        f_gpu = gpu.f_max_mhz
    if t_cpu <= 0.0:
        f_cpu = cpu.f_base_mhz
    elif t_cpu_des > 0.0:
        f_cpu = cpu.round_up_to_grid(cpu.f_base_mhz * t_cpu / t_cpu_des)
    else:
        f_cpu = cpu.f_max_mhz
    t_limit = max(t_gpu, t_cpu + t_tr)
    skip_gpu = t_gpu * gpu.f_base_mhz / f_gpu > t_limit
    skip_cpu = t_cpu * cpu.f_base_mhz / f_cpu > t_limit
    if skip_gpu:
        f_gpu = previous.f_gpu_mhz if previous else gpu.f_base_mhz
    if skip_cpu:
        f_cpu = previous.f_cpu_mhz if previous else cpu.f_base_mhz
    single = full = False
    if coverage is not None and table is not None:
        choice = adaptive_abft(coverage, table, f_gpu, gpu.f_base_mhz, t_gpu, gpu.f_min_mhz)
        f_gpu = gpu.clamp(choice.frequency)
        single, full = choice.single_check, choice.full_check
    return ScheduleDecision(f_cpu, f_gpu, cpu.alpha_default, gpu.alpha_default, single, full,
                            skip_cpu or skip_gpu, True)


def scheme_of(decision: ScheduleDecision) -> ChecksumScheme:
    """simulator.py:170-175."""
    if decision.full_check:
        return ChecksumScheme.FULL
    if decision.single_check:
        return ChecksumScheme.SINGLE
    return ChecksumScheme.NONE


# ---------------------------------------------------------------------------
# measured-time predictor (predictor.py:40-80 over CUDA-event times)
# ---------------------------------------------------------------------------
class _History:
    def __init__(self, kind, task, n, b):
        self.kind, self.task, self.n, self.b = kind, task, n, b
        self.times, self.iters = [], []

    def _c(self, k):
        return compute_flops(self.kind, self.task, self.n, self.b, k)

    def observe(self, k, seconds, f_used, f_base):
        self.times.append(seconds * f_used / f_base)
        self.iters.append(k)

    def predict(self, k):
        if self._c(k) == 0.0 or not self.times:
            return 0.0
        depth = min(4, len(self.times))
        w = HISTORY_WEIGHTS[:depth]
        tot = 0.0
        for i in range(depth):
            cj = self._c(self.iters[-1 - i])
            ratio = self._c(k) / cj if cj else 0.0
            tot += (w[i] / sum(w)) * ratio * self.times[-1 - i]
        return tot


# ---------------------------------------------------------------------------
# the run loop
# ---------------------------------------------------------------------------
@dataclass
class IterationRecord:
    k: int
    f_cpu_mhz: float
    f_gpu_mhz: float
    abft_mode: str
    skipped: bool
    t_panel_ms: float = 0.0    # PD + PU (measured)
    t_update_ms: float = 0.0   # TMU GEMMs + ABFT (measured)
    t_abft_ms: float = 0.0
    slack_pred_s: float = 0.0
    slack_actual_s: float = 0.0
    faults: dict = field(default_factory=lambda: {k.value: 0 for k in ErrorKind})
    detected: int = 0
    corrected: int = 0
    retries: int = 0
    pred_time_s: dict = field(default_factory=dict)    # task -> predicted seconds
    actual_time_s: dict = field(default_factory=dict)  # task -> measured seconds
    side_sms: int = 0          # stream engine: SMs left to the panel (0 = built-in split)


@dataclass
class RunSummary:
    mode: str
    r: float
    kind: str
    n: int
    b: int
    device_ms: float
    abft_ms: float
    energy_j: float | None
    residual: float
    correct: bool
    faults_injected: dict
    faults_detected: int
    faults_corrected: int
    unrecoverable: bool
    retries: int
    schemes: dict


class _Energy:
    def __init__(self, device: int):
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv, self.h, self.ok = pynvml, pynvml.nvmlDeviceGetHandleByIndex(device), True
        except Exception:
            pass

    def mj(self):
        if not self.ok:
            return None
        try:
            return float(self.nv.nvmlDeviceGetTotalEnergyConsumption(self.h))
        except Exception:
            return None


def _is_single(f) -> bool:
    return f.__class__.__name__ == "SFactorization"


def _profile(f) -> list:
    ms = (ctypes.c_double * 4)()
    read = f._lib.abft_s_profile_read if _is_single(f) else f._lib.abft_profile_read
    check(read(f._ctx, ms))
    return [ms[i] for i in range(4)]


def _profile_enable(f, on: bool) -> None:
    fn = f._lib.abft_s_profile if _is_single(f) else f._lib.abft_profile
    check(fn(f._ctx, 1 if on else 0))


def run_mode(kind, a0: np.ndarray, b: int, mode: str = "bsr", r: float = 0.5, seed: int = 0,
             rates: ErrorRateTable | None = None, recovery: str = "recompute",
             fc_desired: float = 0.999999, forced_scheme=None, device: int | None = None,
             cpu: ClockDomain | None = None, gpu: ClockDomain | None = None,
             precision: str = "f64", engine: str = "iteration"):
    """One factorization under a run mode (simulate_run(engine="numeric"),
    simulator.py:440-492) with measured B200 task times. Returns
    (RunSummary, [IterationRecord]). engine="stream": run_mode_streamed."""
    if engine == "stream":
        if precision != "f64":
            raise ValueError("engine='stream' drives the fp64 context")
        return run_mode_streamed(kind, a0, b, mode, r, seed, rates=rates, recovery=recovery,
                                 fc_desired=fc_desired, forced_scheme=forced_scheme,
                                 device=device, cpu=cpu, gpu=gpu)
    if engine != "iteration":
        raise ValueError("engine must be 'iteration' or 'stream'")
    if mode not in MODES:
        raise ValueError(f"mode must be one of {MODES}")
    if recovery not in RECOVERY_POLICIES:
        raise ValueError(f"recovery must be one of {RECOVERY_POLICIES}")
    kind = DecompositionKind(_value(kind))
    flags = MODE_FLAGS[mode]
    cpu = cpu or panel_domain()
    gpu = gpu or update_domain()
    table = rates or default_gpu_rate_table()
    n = a0.shape[0]
    if precision == "f32":
        from .single import SFactorization
        f = SFactorization(kind, a0, b, device=device)
    else:
        f = Factorization(kind, a0, b, device=device)
    nb = f.layout.n_blocks
    coverage = CoverageParams.for_matrix(n, b, fc_desired)
    _, fault_seed = np.random.SeedSequence(seed).spawn(2)   # simulator.py:212-215
    rng_fault = np.random.default_rng(fault_seed)
    hist = {t: _History(kind, t, n, b) for t in ("pd", "pu", "tmu")}
    forced = ChecksumScheme(_value(forced_scheme)) if forced_scheme is not None else None
    energy = _Energy(f.device)
    records, prev = [], None
    injected = {k.value: 0 for k in ErrorKind}
    detected = corrected = total_retries = 0
    unrecoverable = False
    e0 = energy.mj()
    total_ms = abft_ms = 0.0
    _profile_enable(f, True)
    for k in range(nb):
        # -- decide (simulator.py:274-305) --
        if mode == "original":
            dec = ScheduleDecision(cpu.f_base_mhz, gpu.f_base_mhz, 1.0, 1.0, False, False, False, False)
        elif mode == "r2h" or k == 0:
            a_c = cpu.alpha_default if mode == "bsr" else 1.0
            a_g = gpu.alpha_default if mode == "bsr" else 1.0
            dec = ScheduleDecision(cpu.f_base_mhz, gpu.f_base_mhz, a_c, a_g, False, False, False, True)
        else:
            t_cpu = hist["pd"].predict(k) + hist["pu"].predict(k)
            t_gpu = hist["tmu"].predict(k)
            if mode == "sr":
                dec = decide_sr(cpu, gpu, t_cpu, t_gpu, 0.0)
            else:
                ft_on = flags["col_ft"] and forced is None
                dec = decide_bsr(cpu, gpu, t_cpu, t_gpu, 0.0, r, coverage if ft_on else None,
                                 table if ft_on else None, prev)
        scheme = forced if forced is not None else scheme_of(dec)
        prev = dec
        t_cpu_p = hist["pd"].predict(k) + hist["pu"].predict(k)
        t_gpu_p = hist["tmu"].predict(k)
        rec = IterationRecord(k, dec.f_cpu_mhz, dec.f_gpu_mhz, scheme.value, dec.skipped,
                              slack_pred_s=t_gpu_p - t_cpu_p)
        attempts = 0
        while True:
            attempts += 1
            if recovery == "recompute":
                f.snapshot(0)
            before = _profile(f)
            # fault process for the chosen (virtual) update clock over the
            # predicted update interval at that clock (simulator.py:408-418)
            t_tmu = (t_gpu_p if t_gpu_p > 0 else 0.0) * gpu.f_base_mhz / dec.f_gpu_mhz
            lam = table.rates(dec.f_gpu_mhz)
            counts = {kk: int(rng_fault.poisson(l * t_tmu)) for kk, l in zip(ErrorKind, lam)}
            rep = (f.run_numeric_iteration(k, scheme, counts, rng_fault) if _is_single(f)
                   else run_numeric_iteration(f, k, scheme, counts, rng_fault))
            after = _profile(f)
            d = [x - y for x, y in zip(after, before)]
            total_ms += sum(d)
            abft_ms += d[3]
            for kk in ErrorKind:
                injected[kk.value] += counts[kk]
                rec.faults[kk.value] += counts[kk]
            rec.detected += rep.total_detected
            rec.corrected += rep.total_corrected
            detected += rep.total_detected
            corrected += rep.total_corrected
            if not rep.uncorrectable or recovery == "continue":
                break
            if recovery == "abort" or attempts > MAX_RECOVERY_RETRIES:
                unrecoverable = True
                break
            f.restore(0)
            rec.retries += 1
            total_retries += 1
        rec.pred_time_s = {"pd": hist["pd"].predict(k), "pu": hist["pu"].predict(k),
                           "tmu": t_gpu_p, "transfer": 0.0}
        rec.actual_time_s = {"pd": d[0] * 1e-3, "pu": d[1] * 1e-3, "tmu": (d[2] + d[3]) * 1e-3,
                             "transfer": 0.0}
        rec.t_panel_ms = d[0] + d[1]
        rec.t_update_ms = d[2] + d[3]
        rec.t_abft_ms = d[3]
        rec.slack_actual_s = (rec.t_update_ms - rec.t_panel_ms) * 1e-3
        # observe measured times; the physical clock never changed (the
        # domains are virtual), so they ARE the base-clock times. The update
        # side includes its ABFT work, as the reference adds checksum cost
        # to t_gpu (simulator.py:257-272).
        hist["pd"].observe(k, d[0] * 1e-3, 1.0, 1.0)
        hist["pu"].observe(k, d[1] * 1e-3, 1.0, 1.0)
        hist["tmu"].observe(k, (d[2] + d[3]) * 1e-3, 1.0, 1.0)
        records.append(rec)
        if unrecoverable:
            break
    _profile_enable(f, False)
    e1 = energy.mj()
    if not f.complete:
        res = float("inf")
    else:
        res = f.residual(a0) if _is_single(f) else residual(a0, f)
    tol = 1e-4 if _is_single(f) else 1e-8  # simulator.py:33 (fp64); fp32 restated (typical 1e-7..2e-5)
    schemes = {}
    for rec in records:
        schemes[rec.abft_mode] = schemes.get(rec.abft_mode, 0) + 1
    summary = RunSummary(mode, r, kind.value, n, b, total_ms, abft_ms,
                         (e1 - e0) / 1e3 if e0 is not None and e1 is not None else None,
                         res, res <= tol and not unrecoverable, injected, detected, corrected,
                         unrecoverable, total_retries, schemes)
    return summary, records


SIDE_BASE = {DecompositionKind.QR: (16, 8, 48), DecompositionKind.LU: (2, 2, 8),
             DecompositionKind.CHOLESKY: (1, 1, 8)}
# panel-side latency that more SMs do not shorten (three multi-CTA diagonal
# factors + small GEMMs per QR panel, tools/prof/diag_probe.py)
SIDE_FIXED_S = {DecompositionKind.QR: 0.75e-3}


def _side_time(kind, t_panel, R, base):
    """Panel-side time on R SMs from its time at the fixed split `base`."""
    if kind == DecompositionKind.QR:
        fix = min(t_panel, SIDE_FIXED_S[kind])
        return fix + (t_panel - fix) * base / R
    # LU / Cholesky: one-CTA diagonal factor below ceil(b/32) SMs, the
    # multi-CTA kernel (~2.2x faster, tools/prof/diag_probe.py) from there on
    return t_panel if R < 4 else t_panel / 2.2


def _qr_side_model(n, b, k):
    """ctx.cu qr_panel_sms: the QR panel's split from flop counts at the
    measured per-SM DMMA rate (panel: four tall GEMM passes + its fixed
    latency; update: C -= V mid on the other SMs)."""
    rate = 30.0e12 / 148.0
    p = (k - 1) * b  # panel k is factored beside the update of k - 1
    m1, cols = n - p - b, n - p - 2 * b
    best, best_t = 16, None
    for R in range(8, 49, 4):
        tp = 8.0 * m1 * b * b / (R * rate) + 0.8e-3
        tu = 2.0 * (n - p) * cols * b / ((148 - R) * rate) if cols > 0 else 0.0
        t = max(tp, tu)
        if best_t is None or t < 0.995 * best_t:
            best, best_t = R, t
    return best


def _side_sms_choice(kind, t_panel, t_update, r, reclaim, n=0, b=0, k=0):
    """SMs left to iteration k's panel work beside the look-ahead update: the
    fixed split without slack reclamation; with it, the split at which the
    predicted panel and update times meet (the side with slack gets fewer
    SMs, the critical side more), reached by the reclamation ratio r
    (scheduler.py:84-146 restated on SMs instead of clocks). QR uses the
    library's flop model (its panel time is part latency, part SM-bound)."""
    kind = DecompositionKind(_value(kind))
    base, lo, hi = SIDE_BASE[kind]
    if not reclaim or t_update <= 0.0 or t_panel <= 0.0:
        return base
    if kind == DecompositionKind.QR and n > 0 and k >= 1:
        return int(round(base + r * (_qr_side_model(n, b, k) - base)))
    best, best_t = base, None
    for R in range(lo, hi + 1):
        tp = _side_time(kind, t_panel, R, base)
        tu = t_update * (148.0 - base) / (148.0 - R)
        t = max(tp, tu)
        if best_t is None or t < best_t * 0.995 or (abs(t - best_t) <= best_t * 0.005 and R < best):
            best, best_t = R, t
    return int(round(base + r * (best - base)))


def run_mode_streamed(kind, a0: np.ndarray, b: int, mode: str = "bsr", r: float = 0.5,
                      seed: int = 0, rates: ErrorRateTable | None = None,
                      recovery: str = "recompute", fc_desired: float = 0.999999,
                      forced_scheme=None, device: int | None = None,
                      cpu: ClockDomain | None = None, gpu: ClockDomain | None = None):
    """run_mode on the one-call look-ahead path (engine="stream", module doc).
    Returns (RunSummary, [IterationRecord])."""
    from .simulator import run_protected
    if mode not in MODES:
        raise ValueError(f"mode must be one of {MODES}")
    if recovery not in RECOVERY_POLICIES:
        raise ValueError(f"recovery must be one of {RECOVERY_POLICIES}")
    kind = DecompositionKind(_value(kind))
    flags = MODE_FLAGS[mode]
    cpu = cpu or panel_domain()
    gpu = gpu or update_domain()
    table = rates or default_gpu_rate_table()
    n = a0.shape[0]
    f = Factorization(kind, a0, b, device=device, keep_input=True)
    lib, ctx = f._lib, f._ctx
    nb = f.layout.n_blocks
    buf = (ctypes.c_double * (4 * nb))()
    # calibration pass at the fixed split: per-iteration device times
    base = SIDE_BASE[kind][0]
    check(lib.abft_set_side_sms(ctx, (ctypes.c_int32 * nb)(*([base] * nb)), nb))
    check(lib.abft_profile(ctx, 1))
    run_protected(f, "full", {}, None)
    check(lib.abft_profile_read_iters(ctx, buf, nb))
    check(lib.abft_profile(ctx, 0))
    cal = [[buf[4 * k + t] * 1e-3 for t in range(4)] for k in range(nb)]
    check(lib.abft_reset(ctx))
    f.k_done = 0
    # decisions from the history predictor over the calibration times
    coverage = CoverageParams.for_matrix(n, b, fc_desired)
    _, fault_seed = np.random.SeedSequence(seed).spawn(2)   # simulator.py:212-215
    rng_fault = np.random.default_rng(fault_seed)
    hist = {t: _History(kind, t, n, b) for t in ("pd", "pu", "tmu")}
    forced = ChecksumScheme(_value(forced_scheme)) if forced_scheme is not None else None
    decisions, schemes, schedule, side, preds = [], [], {}, [], []
    prev = None
    for k in range(nb):
        t_cpu = hist["pd"].predict(k) + hist["pu"].predict(k)
        t_gpu = hist["tmu"].predict(k)
        if mode == "original":
            dec = ScheduleDecision(cpu.f_base_mhz, gpu.f_base_mhz, 1.0, 1.0, False, False, False, False)
        elif mode == "r2h" or k == 0:
            a_c = cpu.alpha_default if mode == "bsr" else 1.0
            a_g = gpu.alpha_default if mode == "bsr" else 1.0
            dec = ScheduleDecision(cpu.f_base_mhz, gpu.f_base_mhz, a_c, a_g, False, False, False, True)
        elif mode == "sr":
            dec = decide_sr(cpu, gpu, t_cpu, t_gpu, 0.0)
        else:
            ft_on = flags["col_ft"] and forced is None
            dec = decide_bsr(cpu, gpu, t_cpu, t_gpu, 0.0, r, coverage if ft_on else None,
                             table if ft_on else None, prev)
        prev = dec
        sch = forced if forced is not None else scheme_of(dec)
        decisions.append(dec)
        schemes.append(sch.value)
        side.append(_side_sms_choice(kind, t_cpu, t_gpu, r if mode == "bsr" else 1.0,
                                     flags["reclaim_slack"], n, b, k))
        preds.append((t_cpu, t_gpu))
        t_tmu = (t_gpu if t_gpu > 0 else 0.0) * gpu.f_base_mhz / dec.f_gpu_mhz
        lam = table.rates(dec.f_gpu_mhz)
        counts = {kk: int(rng_fault.poisson(l * t_tmu)) for kk, l in zip(ErrorKind, lam)}
        if any(counts.values()):
            schedule[k] = counts
        pd_, pu_, tmu_, abft_ = cal[k]
        hist["pd"].observe(k, pd_, 1.0, 1.0)
        hist["pu"].observe(k, pu_, 1.0, 1.0)
        hist["tmu"].observe(k, tmu_ + abft_, 1.0, 1.0)
    # the run: per-iteration schemes, side-stream SM shares and fault plans
    sarr = (ctypes.c_int32 * nb)(*side)
    check(lib.abft_set_side_sms(ctx, sarr, nb))
    energy = _Energy(f.device)
    check(lib.abft_profile(ctx, 1))
    e0 = energy.mj()
    reps = run_protected(f, "none", schedule, rng_fault, schemes=schemes)
    e1 = energy.mj()
    check(lib.abft_profile_read_iters(ctx, buf, nb))
    check(lib.abft_profile(ctx, 0))
    check(lib.abft_set_side_sms(ctx, None, 0))
    total_ms = ctypes.c_double(0.0)
    check(lib.abft_last_elapsed_ms(ctx, ctypes.byref(total_ms)))
    if recovery == "recompute" and any(rep.uncorrectable for rep in reps):
        # exact reference semantics (snapshot + recompute) on the iteration engine
        return run_mode(kind, a0, b, mode, r, seed, rates=rates, recovery=recovery,
                        fc_desired=fc_desired, forced_scheme=forced_scheme, device=device,
                        cpu=cpu, gpu=gpu)
    records = []
    injected = {kk.value: 0 for kk in ErrorKind}
    detected = corrected = 0
    abft_ms = 0.0
    for k in range(nb):
        dec, rep = decisions[k], reps[k]
        t = [buf[4 * k + i] for i in range(4)]
        rec = IterationRecord(k, dec.f_cpu_mhz, dec.f_gpu_mhz, schemes[k], dec.skipped,
                              slack_pred_s=preds[k][1] - preds[k][0])
        for kk, v in schedule.get(k, {}).items():
            rec.faults[kk.value] += v
            injected[kk.value] += v
        rec.detected, rec.corrected = rep.total_detected, rep.total_corrected
        detected += rep.total_detected
        corrected += rep.total_corrected
        rec.pred_time_s = {"pd": preds[k][0], "pu": 0.0, "tmu": preds[k][1], "transfer": 0.0}
        rec.actual_time_s = {"pd": t[0] * 1e-3, "pu": t[1] * 1e-3, "tmu": (t[2] + t[3]) * 1e-3,
                             "transfer": 0.0}
        rec.t_panel_ms, rec.t_update_ms, rec.t_abft_ms = t[0] + t[1], t[2] + t[3], t[3]
        rec.slack_actual_s = (rec.t_update_ms - rec.t_panel_ms) * 1e-3
        rec.side_sms = side[k]
        abft_ms += t[3]
        records.append(rec)
    res = residual(a0, f)
    sch_count = {}
    for sname in schemes:
        sch_count[sname] = sch_count.get(sname, 0) + 1
    unrec = any(rep.uncorrectable for rep in reps)
    summary = RunSummary(mode, r, kind.value, n, b, float(total_ms.value), abft_ms,
                         (e1 - e0) / 1e3 if e0 is not None and e1 is not None else None,
                         res, res <= 1e-8 and not unrec, injected, detected, corrected, unrec, 0,
                         sch_count)
    return summary, records


def sweep_reclamation_ratio(kind, a0: np.ndarray, b: int, ratios=None, seed: int = 0, **kw):
    """simulator.py:629-647 on the B200: one bsr run per r."""
    ratios = [round(0.05 * i, 2) for i in range(21)] if ratios is None else list(ratios)
    return [run_mode(kind, a0, b, "bsr", r, seed, **kw)[0] for r in ratios]


def compare_modes(kind, a0: np.ndarray, b: int, r: float = 0.5, seed: int = 0, **kw) -> dict:
    """simulator.py:650-669 on the B200: every mode on the same input."""
    return {m: run_mode(kind, a0, b, m, r, seed, **kw)[0] for m in MODES}


# ---------------------------------------------------------------------------
# derived tables of the reference's sweep / compare / campaign commands
# (simulator.py:620-710, cli.py:233-277) over measured B200 runs: time =
# device time of the factorization, energy = NVML joules (None without NVML)
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class SweepPoint:
    r: float
    time_s: float
    energy_j: float | None
    ed2p: float | None
    pareto: bool


def _ed2p(energy_j, time_s):
    """power.py ed2p: energy x delay^2."""
    return None if energy_j is None else energy_j * time_s * time_s


def sweep_points(summaries: list) -> list:
    """simulator.py:636-647: flag the Pareto-efficient (time, energy) points
    (without energy readings, time alone orders them)."""
    pts = []
    for s in summaries:
        t, e = s.device_ms * 1e-3, s.energy_j
        dominated = False
        for o in summaries:
            to, eo = o.device_ms * 1e-3, o.energy_j
            if e is None or eo is None:
                dominated |= to < t
            else:
                dominated |= to <= t and eo <= e and (to < t or eo < e)
        pts.append(SweepPoint(float(s.r), t, e, _ed2p(e, t), not dominated))
    return pts


def mode_table(summaries: dict) -> dict:
    """simulator.py:650-669: savings / speedup relative to 'original'."""
    base = summaries["original"]
    bt, be = base.device_ms * 1e-3, base.energy_j
    out = {}
    for mode, s in summaries.items():
        t, e = s.device_ms * 1e-3, s.energy_j
        ok = e is not None and be
        out[mode] = {
            "summary": s,
            "energy_saving_pct": 100.0 * (1.0 - e / be) if ok else None,
            "ed2p_reduction_pct": 100.0 * (1.0 - _ed2p(e, t) / _ed2p(be, bt)) if ok else None,
            "speedup": bt / t,
            # the reference's floor is its modeled peak-efficiency energy
            # (power.py theoretical_min_energy); no measured counterpart
            "energy_gap_fraction": None,
        }
    return out


CAMPAIGN_SCHEMES = ("none", "single", "full", "adaptive")


@dataclass(frozen=True)
class CampaignRow:
    scheme: str
    trials: int
    correct_fraction: float
    overhead_fraction: float


def fault_campaign(kind, a0: np.ndarray, b: int, trials: int, seed: int = 0,
                   schemes=CAMPAIGN_SCHEMES, **kw) -> list:
    """simulator.py:683-710 on the B200: bsr mode, recovery 'continue', each
    forced scheme (and the adaptive governor) over seeds seed..seed+trials-1;
    correct_fraction = runs whose final residual passes, overhead_fraction =
    mean measured ABFT share of the device time."""
    if trials < 1:
        raise ValueError("need at least one trial")
    rows = []
    for scheme in schemes:
        forced = None if scheme == "adaptive" else scheme
        rest = {k: v for k, v in kw.items() if k != "r"}
        sums = [run_mode(kind, a0, b, "bsr", kw.get("r", 0.5), seed + t, recovery="continue",
                         forced_scheme=forced, **rest)[0]
                for t in range(trials)]
        rows.append(CampaignRow(scheme, trials, sum(1 for s in sums if s.correct) / trials,
                                float(np.mean([s.abft_ms / s.device_ms if s.device_ms else 0.0
                                               for s in sums]))))
    return rows


# ---------------------------------------------------------------------------
# output formats (cli.py:33-122): the reference's trace CSV and summary JSON
# ---------------------------------------------------------------------------
TRACE_HEADER = ("iter,task,pred_time_s,actual_time_s,slack_pred_s,"
                "slack_actual_s,f_cpu_mhz,f_gpu_mhz,abft_mode,faults_0d,"
                "faults_1d,faults_2d,detected,corrected,e_cpu_dyn_j,"
                "e_cpu_stat_j,e_cpu_idle_j,e_gpu_dyn_j,e_gpu_stat_j,"
                "e_gpu_idle_j,skipped")                 # cli.py:33-37
_TRACE_TASKS = ("pd", "pu", "tmu", "transfer", "idle")  # cli.py:39


def trace_rows(records: list) -> list:
    """cli.py:46-92 over B200 records: one row per task plus an idle row per
    iteration; slack on the pd row, fault counters on the tmu row. Times are
    measured device times; per-task energies are not metered separately on
    one GPU (the run's NVML total is in the summary), so those columns are 0."""
    rows = []
    fmt = lambda x: repr(float(x))  # noqa: E731  (cli.py:42-43)
    for rec in records:
        for task in _TRACE_TASKS:
            is_pd, is_tmu = task == "pd", task == "tmu"
            pred = 0.0 if task == "idle" else rec.pred_time_s.get(task, 0.0)
            act = 0.0 if task == "idle" else rec.actual_time_s.get(task, 0.0)
            cells = [str(rec.k), task, fmt(pred), fmt(act),
                     fmt(rec.slack_pred_s if is_pd else 0.0),
                     fmt(rec.slack_actual_s if is_pd else 0.0),
                     fmt(rec.f_cpu_mhz), fmt(rec.f_gpu_mhz), rec.abft_mode,
                     str(rec.faults["0d"] if is_tmu else 0),
                     str(rec.faults["1d"] if is_tmu else 0),
                     str(rec.faults["2d"] if is_tmu else 0),
                     str(rec.detected if is_tmu else 0),
                     str(rec.corrected if is_tmu else 0),
                     fmt(0.0), fmt(0.0), fmt(0.0), fmt(0.0), fmt(0.0), fmt(0.0),
                     "1" if rec.skipped else "0"]
            rows.append(",".join(cells))
    return rows


def _write_atomic(path: str, text: str) -> None:
    """cli.py:95-106."""
    import os
    import tempfile
    directory = os.path.dirname(os.path.abspath(path)) or "."
    os.makedirs(directory, exist_ok=True)
    fd, tmp = tempfile.mkstemp(dir=directory, prefix=".b200-")
    try:
        with os.fdopen(fd, "w", encoding="utf-8", newline="\n") as fh:
            fh.write(text)
        os.replace(tmp, path)
    except BaseException:
        if os.path.exists(tmp):
            os.unlink(tmp)
        raise


def write_trace(path: str, records: list) -> None:
    """cli.py:109-110."""
    _write_atomic(path, "\n".join([TRACE_HEADER] + trace_rows(records)) + "\n")


def write_summary(path: str, summary: RunSummary) -> None:
    """cli.py:113-122 (sorted keys, indent 2)."""
    import dataclasses
    import json
    _write_atomic(path, json.dumps(dataclasses.asdict(summary), sort_keys=True, indent=2) + "\n")


def _fmt_opt(x) -> str:
    return "" if x is None else repr(float(x))


def write_sweep(path: str, points: list) -> None:
    """cli.py:233-245: r,time_s,energy_j,ed2p,pareto."""
    lines = ["r,time_s,energy_j,ed2p,pareto"]
    for p in points:
        lines.append(",".join([repr(float(p.r)), repr(float(p.time_s)), _fmt_opt(p.energy_j),
                               _fmt_opt(p.ed2p), "1" if p.pareto else "0"]))
    _write_atomic(path, "\n".join(lines) + "\n")


def write_compare(path: str, table: dict) -> None:
    """cli.py:248-266 (sorted keys, indent 2)."""
    import json
    doc = {}
    for mode, row in table.items():
        s = row["summary"]
        t = s.device_ms * 1e-3
        doc[mode] = {"energy_saving_pct": row["energy_saving_pct"],
                     "ed2p_reduction_pct": row["ed2p_reduction_pct"],
                     "speedup": row["speedup"],
                     "energy_gap_fraction": row["energy_gap_fraction"],
                     "total_time_s": t, "total_energy_j": s.energy_j,
                     "ed2p": _ed2p(s.energy_j, t)}
    _write_atomic(path, json.dumps(doc, sort_keys=True, indent=2) + "\n")


def write_campaign(path: str, rows: list) -> None:
    """cli.py:269-277: scheme,correct_fraction,overhead_fraction."""
    lines = ["scheme,correct_fraction,overhead_fraction"]
    for row in rows:
        lines.append(",".join([row.scheme, repr(float(row.correct_fraction)),
                               repr(float(row.overhead_fraction))]))
    _write_atomic(path, "\n".join(lines) + "\n")
