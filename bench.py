#!/usr/bin/env python
"""Benchmark: ABFT-protected blocked factorization TFLOP/s on B200.

Headline (BASELINE.json metric "ABFT dpotrf/dgetrf/dgeqrf TFLOP/s at N=32768,
1/2/4/8 GPU; ABFT overhead %; J"): one step = one complete ABFT-protected
factorization of an N=32768 fp64 matrix (default: LU / dgetrf, b=256, FULL =
col_ft+row_ft checksums as under the `bsr` mode flags, one seeded 0-D fault
injected and corrected, criterion-5 protocol). TFLOP/s uses the LAPACK flop
convention (2n^3/3 LU, n^3/3 Cholesky, 4n^3/3 QR), ABFT work not counted.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
  python -m torch.distributed.run --nproc-per-node N bench.py --gpus N ...

N > 1: ONE global N=32768 matrix distributed 1-D block-cyclic by column
blocks over the ranks (strong scaling: total work fixed); time is the max
over ranks. --impl reference times the reference algorithm's CPU restatement
(oracle/, numpy + LAPACK) on a bounded sample: a complete protected
factorization at N=4096 (an N=32768 factorization takes hours on the host);
its line's config names the order it actually timed.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

FLOPS = {"cholesky": lambda n: n ** 3 / 3.0, "lu": lambda n: 2.0 * n ** 3 / 3.0,
         "qr": lambda n: 4.0 * n ** 3 / 3.0}
LAPACK = {"cholesky": "dpotrf", "lu": "dgetrf", "qr": "dgeqrf"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--kind", default="lu", choices=["lu", "cholesky", "qr"])
    ap.add_argument("--n", "--order", dest="n", type=int, default=32768)
    ap.add_argument("--b", type=int, default=256)
    ap.add_argument("--scheme", default="full", choices=["none", "single", "full"])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-overhead", action="store_true", help="skip the scheme=none run")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--extra-kinds", default="", help="comma list of kinds also measured")
    ap.add_argument("--profile-only", action="store_true", help="one step, for ncu")
    ap.add_argument("--precision", default="f64", choices=["f64", "f32"],
                    help="f32: the s* variants (sgetrf/spotrf) on the tcgen05 tf32 path")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="N>1 transport (gloo: several ranks sharing one GPU, for testing)")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# environment helpers
# ---------------------------------------------------------------------------

def all_max(x: float) -> float:
    """Max over ranks (identity for a single process)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(x)
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi-equivalent sampling through NVML during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.ok = True
        except Exception:
            return
        self.samples, self.reasons = [], set()
        self._stop = threading.Event()
        self.max_mhz = self.nv.nvmlDeviceGetMaxClockInfo(self.h, self.nv.NVML_CLOCK_SM)

    def energy_mj(self) -> float | None:
        if not self.ok:
            return None
        try:
            return float(self.nv.nvmlDeviceGetTotalEnergyConsumption(self.h))
        except Exception:
            return None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name not in ("gpu_idle",):
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.1)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def fault_plan(n: int, b: int, seed: int):
    """Criterion-5 protocol (pkg/tests/test_acceptance.py:221-224): rng =
    default_rng(seed); k_fault = rng.integers(0, nb-1); {0d: 1} at k_fault."""
    rng = np.random.default_rng(seed)
    nb = -(-n // b)
    k_fault = int(rng.integers(0, nb - 1))
    return k_fault, rng


# ---------------------------------------------------------------------------
# CPU reference arm (oracle restatement of the reference algorithm)
# ---------------------------------------------------------------------------

CPU_N = 4096  # order of the bounded CPU sample (full factorization, ~10-30 s on the host)


def cpu_sample(kind: str, n: int, b: int, scheme: str, seed: int):
    """The reference algorithm's CPU path (oracle/, numpy + LAPACK, the
    reference's own operations) timed on a complete protected factorization of
    order n with the same block size, scheme and fault protocol as the GPU
    workload. Returns (TFLOP/s, seconds)."""
    import oracle as O
    a = O.generate_test_matrix(kind, n, seed)
    k_fault, rng = fault_plan(n, b, seed)
    f = O.OracleFactorization(kind, a, b)
    t0 = time.perf_counter()
    for k in range(f.nb):
        O.protected_iteration(f, k, scheme, {"0d": 1} if k == k_fault else None, rng)
    dt = time.perf_counter() - t0
    return FLOPS[kind](n) / dt / 1e12, dt


def cpu_sample_desc(kind, n, b, scheme) -> str:
    return (f"oracle (numpy/LAPACK restatement of slackwise's algorithm) complete protected "
            f"{kind} factorization N={n} b={b} scheme={scheme}, criterion-5 fault protocol; "
            f"N=32768 itself takes ~2 min per iteration on the host")


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    n = min(args.n, CPU_N)
    for _ in range(args.warmup):  # first LAPACK calls in a process are slow
        cpu_sample(args.kind, 512, min(args.b, 512), args.scheme, args.seed)
    vals = [cpu_sample(args.kind, n, args.b, args.scheme, args.seed) for _ in range(args.steps)]
    value = statistics.median(v[0] for v in vals)
    ms = statistics.median(v[1] for v in vals) * 1e3
    cfg = config(args, n=n)
    cfg["sample_of"] = config(args)["workload"]
    line = {"impl": "reference", "metric": metric_name(args), "value": value, "unit": "TFLOP/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "config": cfg,
            "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": os.cpu_count(),
                             "kind": "port", "sample": cpu_sample_desc(args.kind, n, args.b,
                                                                       args.scheme),
                             "cpu": cpu_model()},
            "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def metric_name(args) -> str:
    name = LAPACK[args.kind] if args.precision == "f64" else "s" + LAPACK[args.kind][1:]
    return (f"ABFT {name} TFLOP/s ({'fp64' if args.precision == 'f64' else 'fp32'} N={args.n}, "
            f"{args.scheme.upper()} checksums, 1 seeded fault)")


def config(args, n: int | None = None) -> dict:
    """The workload; ``n`` overrides the order (the reference arm's sample)."""
    n = args.n if n is None else n
    prec = "fp64" if args.precision == "f64" else "fp32 (tcgen05 3xTF32)"
    return {"workload": f"{args.kind} {prec} N={n} b={args.b} scheme={args.scheme} "
                        f"(col_ft+row_ft as under mode=bsr), one 0-D fault at a seeded "
                        f"iteration (criterion-5 protocol)",
            "kind": args.kind, "n": n, "b": args.b, "scheme": args.scheme,
            "seed": args.seed,
            "l2": f"working set {n * n * (8 if args.precision == 'f64' else 4) / 1e9:.1f} GB "
                  + (">> 126 MB L2; no flush needed" if n * n * 4 > 4 * 126e6 else
                     "(CPU sample)"),
            "parallelism": (f"block-cyclic columns over {args.gpus} GPUs "
                            f"({'panel-update reduce' if args.kind == 'cholesky' and os.environ.get('ABFT_DIST_CHOL', '').startswith('l') else 'panel broadcast + cross-rank look-ahead'}"
                            f" over {args.dist_backend})") if args.gpus > 1 else "single"}


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------

class Arm:
    """One device-resident factorization context reused across steps."""

    def __init__(self, kind, n, b, seed, device):
        import paper_2301_03166_b200 as P
        from paper_2301_03166_b200 import _lib
        self.P, self.L = P, _lib
        self.lib = _lib.load()
        self.kind, self.n, self.b, self.seed = kind, n, b, seed
        t0 = time.perf_counter()
        if kind == "cholesky":
            # host PCG64 uniform (bit-identical draws); SPD product on the GPU
            host = np.asfortranarray(np.random.default_rng(seed).uniform(-1.0, 1.0, size=(n, n)))
        else:
            host = P.generate_test_matrix(kind, n, seed)
        self.gen_s = time.perf_counter() - t0
        self.f = P.Factorization(kind, host, b, device=device, keep_input=True)
        if kind == "cholesky":
            P.linalg.check(self.lib.abft_make_spd(self.f._ctx))
            self.f._dirty()
            host = self.f.m  # the SPD input, for the end-to-end leg
        self.host = host
        _GEN["s"] = self.gen_s
        import torch
        self.torch = torch
        self.stream = torch.cuda.ExternalStream(self.lib.abft_stream(self.f._ctx))

    def step(self, scheme):
        k_fault, rng = fault_plan(self.n, self.b, self.seed)
        self.P.linalg.check(self.lib.abft_reset(self.f._ctx))
        sched = {k_fault: {"0d": 1}}
        reps = self.P.run_protected(self.f, scheme, sched, rng)
        return k_fault, reps

    def timed(self, scheme, steps):
        torch = self.torch
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(self.stream)
        out = None
        for _ in range(steps):
            out = self.step(scheme)
        e1.record(self.stream)
        e1.synchronize()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1), out

    def profile(self, scheme):
        lib = self.lib
        lib.abft_profile(self.f._ctx, 1)
        self.step(scheme)
        ms = (ctypes.c_double * 4)()
        lib.abft_profile_read(self.f._ctx, ms)
        lib.abft_profile(self.f._ctx, 0)
        return {"pd": ms[0], "pu": ms[1], "tmu_gemm": ms[2], "abft": ms[3]}

    def residual(self):
        out = ctypes.c_double(0.0)
        self.P.linalg.check(self.lib.abft_residual(self.f._ctx, None, self.n, ctypes.byref(out)))
        return out.value


class DistArm:
    """Block-cyclic factorization over all ranks: rank 0 alone
    generates the global input and scatters every rank its column blocks
    (scatter_input); each rank keeps its local input on the device."""

    def __init__(self, kind, n, b, seed, device):
        import paper_2301_03166_b200 as P
        from paper_2301_03166_b200 import _lib
        from paper_2301_03166_b200.distributed import DistributedFactorization
        import torch.distributed as dist
        self.P, self.L = P, _lib
        self.lib = _lib.load()
        self.kind, self.n, self.b, self.seed = kind, n, b, seed
        t0 = time.perf_counter()
        host = None
        if dist.get_rank() == 0:
            if kind == "cholesky":
                # uniform draws on the host, SPD product on rank 0's GPU
                host = np.asfortranarray(np.random.default_rng(seed).uniform(-1.0, 1.0, size=(n, n)))
                tmp = P.Factorization(kind, host, b, device=device)
                P.linalg.check(self.lib.abft_make_spd(tmp._ctx))
                tmp._dirty()
                host = tmp.m
                del tmp
            else:
                host = P.generate_test_matrix(kind, n, seed)
        self.gen_s = time.perf_counter() - t0
        _GEN["s"] = self.gen_s
        self.host = host  # rank 0 only
        self.f = DistributedFactorization(kind, host, b, device=device, keep_input=True, root=0,
                                          n=n)
        import torch
        self.torch = torch
        self.stream = torch.cuda.ExternalStream(self.f.stream_ptr())

    def step(self, scheme):
        k_fault, rng = fault_plan(self.n, self.b, self.seed)
        self.f.reset()
        reps = self.f.run_protected(scheme, {k_fault: {"0d": 1}}, rng)
        return k_fault, reps

    timed = Arm.timed

    def profile(self, scheme):
        return {"pd": None, "pu": None, "tmu_gemm": None, "abft": None}

    def residual(self):
        return self.f.residual(self.host)


class SArm(Arm):
    """fp32 (s*) factorization context on the tcgen05 path, device-resident."""

    def __init__(self, kind, n, b, seed, device):
        import paper_2301_03166_b200 as P
        from paper_2301_03166_b200 import _lib
        self.P, self.L = P, _lib
        self.lib = _lib.load()
        self.kind, self.n, self.b, self.seed = kind, n, b, seed
        t0 = time.perf_counter()
        if kind == "cholesky":
            host = np.asfortranarray(np.random.default_rng(seed).uniform(-1.0, 1.0, size=(n, n)))
        else:
            host = P.generate_test_matrix(kind, n, seed)
        self.gen_s = time.perf_counter() - t0
        _GEN["s"] = self.gen_s
        self.f = P.SFactorization(kind, host, b, device=device, keep_input=True,
                                  spd_on_device=(kind == "cholesky"))
        self.host = self.f.m if kind == "cholesky" else np.asfortranarray(host, dtype=np.float32)
        import torch
        self.torch = torch
        self.stream = torch.cuda.ExternalStream(self.f.stream_ptr())

    def step(self, scheme):
        k_fault, rng = fault_plan(self.n, self.b, self.seed)
        self.f.reset()
        return k_fault, self.f.run_protected(scheme, {k_fault: {"0d": 1}}, rng)

    def profile(self, scheme):
        lib = self.lib
        lib.abft_s_profile(self.f._ctx, 1)
        self.step(scheme)
        ms = (ctypes.c_double * 4)()
        lib.abft_s_profile_read(self.f._ctx, ms)
        lib.abft_s_profile(self.f._ctx, 0)
        return {"pd": ms[0], "pu": ms[1], "tmu_gemm": ms[2], "abft": ms[3]}

    def residual(self):
        return self.f.residual(None)


def tf32x3_peak() -> tuple:
    """Effective 3xTF32 tensor peak: measured dense bf16 (MEASURED_PEAKS.json,
    burst) / 2 for TF32 operands / 3 MMAs per product; fallback 1.59 PF bf16."""
    try:
        d = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        return d["bf16_tflops"] / 6.0, "measured bf16 burst / 2 (tf32) / 3 (3xTF32 split), of measured"
    except Exception:
        return 1590.0 / 6.0, "fallback bf16 1.59 PF / 2 / 3 (B200_PROFILING.md), of fallback"


def hbm_peak() -> tuple:
    """Measured HBM copy bandwidth (MEASURED_PEAKS.json), else the fallback."""
    try:
        d = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        for key in ("hbm_gbs", "hbm_copy_gbs", "hbm_GBs"):
            if key in d:
                return float(d[key]), f"MEASURED_PEAKS.json {key}"
    except Exception:
        pass
    return 6533.5, "fallback (SURVEY §8d MEASURED_PEAKS hbm_gbs)"


def tmu_flops(kind, n, b) -> float:
    from paper_2301_03166_b200.linalg import compute_flops
    return sum(compute_flops(kind, "tmu", n, b, k) for k in range(-(-n // b)))


def verify_bytes(kind, n, b, scheme) -> float:
    """Algorithmic bytes of the checksum verification per factorization: one
    fp64 read of every protected region, plus the fresh encode
    pass Cholesky needs (its region is a new panel each iteration)."""
    if scheme == "none":
        return 0.0
    tot = 0.0
    nb = -(-n // b)
    for k in range(nb):
        p, pe = k * b, min(k * b + b, n)
        rows, cols = {"cholesky": (n - p, pe - p), "lu": (n - pe, n - pe)}.get(kind, (n - p, n - pe))
        if rows > 0 and cols > 0:
            tot += rows * cols * (2 if kind == "cholesky" else 1)
    return 8.0 * tot


def run_ours(args):
    import torch
    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        local = local % torch.cuda.device_count()  # gloo test mode: ranks may share a GPU
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    torch.cuda.set_device(local)
    P = __import__("paper_2301_03166_b200")
    lib = P._lib.load()
    peak = ctypes.c_double(0.0)
    P.linalg.check(lib.abft_probe_dmma_peak(20000, ctypes.byref(peak)))
    if args.precision == "f32":
        if world > 1:
            raise SystemExit("fp32 runs: single GPU")
        arm = SArm(args.kind, args.n, args.b, args.seed, local)
    else:
        arm = (DistArm if world > 1 else Arm)(args.kind, args.n, args.b, args.seed, local)
    if args.profile_only:
        arm.step(args.scheme)
        torch.cuda.synchronize()
        return
    for _ in range(args.warmup):
        arm.step(args.scheme)
    launches0 = lib.abft_launch_count()
    clk = ClockSampler(local)
    en0 = clk.energy_mj()
    if world > 1:
        torch.distributed.barrier()
    with clk:
        ms, (k_fault, reps) = arm.timed(args.scheme, args.steps)
    en1 = clk.energy_mj()
    launches = (lib.abft_launch_count() - launches0) // max(1, args.steps)
    res = arm.residual()
    # the single planned 0-D fault must be located at its planned (row, col)
    # and corrected; a run that misses it is not a protected factorization
    locs = [loc for r in reps for loc in r.locations]
    fixed = sum(r.corrected[P.ErrorKind.D0] for r in reps)
    want = planned_fault(args.kind, args.n, args.b, args.seed)
    fault_ok = (fixed == 1 and len(locs) == 1 and (int(locs[0][0]), int(locs[0][1])) == want
                and bool(locs[0][3])) if args.scheme != "none" else None
    ms_max = all_max(ms)
    ms_step = ms_max / args.steps
    flops = FLOPS[args.kind](args.n)
    # N > 1 factors ONE global matrix over all ranks (strong scaling)
    value = flops / (ms_step * 1e-3) / 1e12

    overhead = None
    if not args.no_overhead and args.scheme != "none":
        for _ in range(1):
            arm.step("none")
        ms_none, _ = arm.timed("none", args.steps)
        overhead = 100.0 * (ms - ms_none) / ms_none
    if overhead is not None and world > 1:
        ov = all_max(ms_none)
        overhead = 100.0 * (ms_max - ov) / ov
    prof = arm.profile(args.scheme)
    tflops_tmu = tmu_flops(args.kind, args.n, args.b)
    achieved = tflops_tmu / (prof["tmu_gemm"] * 1e-3) / 1e12 if prof["tmu_gemm"] else None
    if args.kind == "cholesky" and args.precision == "f32":
        # the fp32 look-ahead update is not bracketed on its side stream:
        # use the whole factorization
        achieved = value
    vbytes = verify_bytes(args.kind, args.n, args.b, args.scheme)

    if args.precision == "f64":
        roofline = {"bound": "tensor",
                    "kernel": "dgemm_tma_dmma (trailing-matrix update)" if args.kind != "cholesky"
                    else "dgemm_tma_dmma (panel updates: TMU(k) on the main stream + the "
                         "look-ahead's update of panel k+1 on the side stream)",
                    "achieved": achieved, "peak": peak.value, "unit": "TFLOP/s",
                    "frac": (achieved / peak.value) if achieved else None,
                    # dram read+write of one fused trailing-update launch (M=N~31.2k, K=256)
                    # from `ncu --set full` (profiles/ncu_full_gemm_lu32k_r01.txt); the
                    # algorithmic bytes of that launch are 15.7e9 (C in, D out, panels once);
                    # 26.63e9 before the grouped unit order
                    # QR: the fused C -= V (T^T W) launch of an early iteration
                    # (profiles/ncu_full_gemm_qr32k_r01.txt)
                    "traffic": {"lu": 16.16e9, "qr": 15.36e9}.get(args.kind),
                    "traffic_algorithmic": {"lu": 15.7e9, "qr": 15.4e9}.get(args.kind),
                    "peak_source": "measured DMMA issue rate on this GPU "
                                   "(abft_probe_dmma_peak; MEASURED_PEAKS.json has no fp64)"}
    else:
        p32, src32 = tf32x3_peak()
        roofline = {"bound": "tensor",
                    "kernel": "sgemm_tc05 (tcgen05 kind::tf32, 3xTF32)" if args.kind != "cholesky"
                    else "whole spotrf (panel updates split across streams by the look-ahead)",
                    "achieved": achieved, "peak": p32, "unit": "TFLOP/s",
                    "frac": (achieved / p32) if achieved else None, "traffic": None,
                    "peak_source": src32}
        if args.kind == "lu" and prof["tmu_gemm"]:
            # the K = b trailing update reads C and writes D once (8 B per element in
            # fp32): at b = 128 it is HBM-bound before it is tensor-bound
            elems = sum((args.n - min((k + 1) * args.b, args.n)) ** 2
                        for k in range(-(-args.n // args.b)))
            gbs = 8.0 * elems / (prof["tmu_gemm"] * 1e-3) / 1e9
            hbm = hbm_peak()
            roofline["hbm_view"] = {"achieved": gbs, "peak": hbm[0], "unit": "GB/s",
                                    "frac": gbs / hbm[0], "bytes_per_factorization": 8.0 * elems,
                                    "peak_source": hbm[1]}
    e2e = None
    if not args.no_e2e and args.precision == "f32":
        e2e = run_e2e_s(arm, args)
    elif not args.no_e2e:
        e2e = run_e2e(arm, args) if world == 1 else run_e2e_dist(arm, args)
    extra = {}
    for kind in [k for k in args.extra_kinds.split(",") if k and k != args.kind]:
        extra[kind] = measure_kind(kind, args, local)
    cpu = None
    if rank == 0 and not args.no_cpu:
        n_cpu = min(args.n, CPU_N)
        cpu_sample(args.kind, 512, min(args.b, 512), args.scheme, args.seed)  # warm LAPACK
        tf, dt = cpu_sample(args.kind, n_cpu, args.b, args.scheme, args.seed)
        cpu = {"value": tf, "unit": "TFLOP/s", "cores": os.cpu_count(), "kind": "port",
               "sample": cpu_sample_desc(args.kind, n_cpu, args.b, args.scheme) +
                         f" ({dt:.1f} s)", "cpu": cpu_model()}
    if rank != 0:
        return
    line = {
        "metric": metric_name(args), "value": value, "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": args.precision,
        "data": f"synthetic: generate_test_matrix({args.kind!r}, {args.n}, seed={args.seed}) "
                "(PCG64 draws bit-identical to the reference)",
        "config": config(args),
        "abft_overhead_pct": overhead,
        "energy_j_per_factorization": ((en1 - en0) / 1e3 / args.steps
                                       if en0 is not None and en1 is not None else None),
        "clocks": clk.summary(),
        "e2e": e2e,
        "gpu_launches": launches,
        "roofline": roofline,
        "abft_verify": {
            "region_bytes": vbytes,
            "note": ("verify-side block sums of LU/QR trailing updates are produced in the GEMM "
                     "epilogue (no separate read of the region); 'ms' is all remaining ABFT work "
                     "(encode of the first region, operand sums, maintenance GEMMs, verify "
                     "kernel, Cholesky panel passes)"),
            "ms": prof["abft"],
            "pct_of_step": 100.0 * prof["abft"] / ms_step if prof["abft"] is not None else None},
        "profile_ms": prof,
        "whole_step_frac_of_peak": value / world / peak.value,
        "residual": res, "residual_over_n_eps": res / (args.n * 2.220446049250313e-16),
        "fault": {"k_fault": k_fault, "planned": list(want),
                  "locations": [[int(a), int(b), c.value, bool(d)] for a, b, c, d in locs],
                  "corrected_0d": int(fixed), "located_and_corrected": fault_ok},
        "cpu_baseline": cpu,
        "input_generation_s": arm_gen_s(),
    }
    if extra:
        line["extra_kinds"] = extra
    if fault_ok is False:
        line["invalid"] = "the seeded 0-D fault was not located and corrected"
    print(json.dumps(line), flush=True)
    if fault_ok is False:
        raise SystemExit(1)


def planned_fault(kind, n, b, seed):
    """(row, col) of the criterion-5 fault: the draws run_protected makes at
    k_fault (sample_fault_plan order, abft.py:314-332)."""
    from paper_2301_03166_b200.abft import draw_plan
    from paper_2301_03166_b200.simulator import _tmu_region
    k_fault, rng = fault_plan(n, b, seed)
    r0, c0, rows, cols = _tmu_region(kind, n, b, k_fault)
    d = draw_plan(rng, {"0d": 1}, r0, c0, rows, cols, b)[0]
    return int(d["row"]), int(d["col"])


_GEN = {"s": None}


def arm_gen_s():
    return _GEN["s"]


def measure_kind(kind, args, local):
    import torch
    arm = Arm(kind, args.n, args.b, args.seed, local)
    arm.step(args.scheme)
    ms, _ = arm.timed(args.scheme, max(1, args.steps))
    ms_step = ms / max(1, args.steps)
    ms_none, _ = arm.timed("none", 1)
    prof = arm.profile(args.scheme)
    out = {"value": FLOPS[kind](args.n) / (ms_step * 1e-3) / 1e12, "unit": "TFLOP/s",
           "ms_per_step": ms_step, "abft_overhead_pct": 100.0 * (ms_step - ms_none) / ms_none,
           "profile_ms": prof, "residual": arm.residual()}
    del arm
    torch.cuda.empty_cache()
    return out


def run_e2e(arm, args):
    """Same metric through the public API with host buffers: pinned H2D of the
    input, protected factorization, D2H of the factors, every step."""
    import torch
    P, lib, f = arm.P, arm.lib, arm.f
    n = args.n
    pinned_in = torch.empty((n, n), dtype=torch.float64, pin_memory=True).numpy()
    pinned_in[...] = arm.host.T  # torch row-major storage holding the Fortran matrix
    src = pinned_in.T           # Fortran-ordered view of the pinned buffer
    pinned_out = torch.empty((n, n), dtype=torch.float64, pin_memory=True).numpy().T
    torch.cuda.synchronize()
    # Cholesky streams the input in by block columns inside the factorization
    # call (the lower block triangle it reads); LU / QR stream all of it and
    # factor the left 3/8 chunk by chunk as it arrives
    chol = args.kind == "cholesky"
    set_in = lib.abft_set_matrix_streamed
    h2d = 8 * n * n
    if chol:
        h2d = sum(8 * (n - j * args.b) * min(args.b, n - j * args.b) for j in range(-(-n // args.b)))
    times = []
    # the kept device copy of the input (residual / abft_reset) already holds
    # this matrix: the streamed set does not refresh it
    P.linalg.check(lib.abft_keep_input(f._ctx, 0))
    try:
        for i in range(1 + args.steps):
            t0 = time.perf_counter()
            P.linalg.check(set_in(f._ctx, P._lib.dptr(src), n))
            k_fault, rng = fault_plan(n, args.b, args.seed)
            # the factor streams to the pinned host buffer as column blocks finish
            P.run_protected(f, args.scheme, {k_fault: {"0d": 1}}, rng, out=pinned_out)
            dt = time.perf_counter() - t0
            if i:
                times.append(dt)
    finally:
        P.linalg.check(lib.abft_keep_input(f._ctx, 1))
    sec = statistics.median(times)
    return {"value": FLOPS[args.kind](n) / sec / 1e12, "unit": "TFLOP/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 8 * n * n,
            "ms_per_step": sec * 1e3,
            "api": ("abft_set_matrix_streamed (block columns H2D inside the call, lower block "
                    "triangle)" if chol else
                    "abft_set_matrix_streamed (block columns H2D inside the call; " +
                    ("the left 3/8 factored chunk by chunk as it arrives)" if args.kind == "lu" else
                     "panels 0-2 factored as their block columns arrive, the rest updated in "
                     "n/8-wide pieces as they arrive)")) +
                   " + run_protected(out=pinned host; finished column blocks stream D2H on a "
                   "copy stream during the factorization)"}


def run_e2e_s(arm, args):
    """fp32 e2e: pinned fp32 host input in, factorization, factor out."""
    import torch
    f, n = arm.f, args.n
    pinned_in = torch.empty((n, n), dtype=torch.float32, pin_memory=True).numpy()
    pinned_in[...] = arm.host.T
    src = pinned_in.T
    pinned_out = torch.empty((n, n), dtype=torch.float32, pin_memory=True).numpy().T
    chol = args.kind == "cholesky"  # streamed input, as run_e2e
    streamed = True
    set_in = arm.lib.abft_s_set_matrix_streamed
    h2d = 4 * n * n
    if chol:
        h2d = sum(4 * (n - j * args.b) * min(args.b, n - j * args.b) for j in range(-(-n // args.b)))
    times = []
    if streamed:
        arm.P.linalg.check(arm.lib.abft_s_keep_input(f._ctx, 0))
    try:
        for i in range(1 + args.steps):
            t0 = time.perf_counter()
            arm.P.linalg.check(set_in(f._ctx, arm.P._lib.fptr(src), n))
            k_fault, rng = fault_plan(n, args.b, args.seed)
            f.run_protected(args.scheme, {k_fault: {"0d": 1}}, rng, out=pinned_out)
            if i:
                times.append(time.perf_counter() - t0)
    finally:
        if streamed:
            arm.P.linalg.check(arm.lib.abft_s_keep_input(f._ctx, 1))
    sec = statistics.median(times)
    return {"value": FLOPS[args.kind](n) / sec / 1e12, "unit": "TFLOP/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 4 * n * n,
            "ms_per_step": sec * 1e3,
            "api": ("abft_s_set_matrix_streamed (block columns H2D inside the call, lower block "
                    "triangle)" if chol else
                    "abft_s_set_matrix_streamed (block columns H2D inside the call; " +
                    ("the left 1/4 factored chunk by chunk as it arrives)" if args.kind == "lu" else
                     "panels 0-2 factored as their block columns arrive, the rest updated in "
                     "n/8-wide pieces as they arrive)")) +
                   " + SFactorization.run_protected(out=pinned host; column blocks stream D2H "
                   "during the factorization)"}


def run_e2e_dist(arm, args):
    """e2e at N>1: every rank copies its column blocks (pinned host, n x
    local columns: 1/N of the matrix per rank) in, runs the distributed
    factorization and copies its columns out; time = max over ranks."""
    import torch
    f, n = arm.f, args.n
    local = f.local_input  # this rank's column blocks (scattered from rank 0)
    pinned_in = torch.empty((max(f.ncl, 1), n), dtype=torch.float64, pin_memory=True).numpy()
    pinned_in[:f.ncl] = local.T
    src = pinned_in.T
    pinned_out = torch.empty((max(f.ncl, 1), n), dtype=torch.float64, pin_memory=True).numpy().T
    times = []
    for i in range(1 + args.steps):
        torch.distributed.barrier()
        t0 = time.perf_counter()
        f._prefetched.clear()
        arm.P.linalg.check(arm.lib.abft_dist_set_local(f._ctx, arm.P._lib.dptr(src), n))
        k_fault, rng = fault_plan(n, args.b, args.seed)
        f.run_protected(args.scheme, {k_fault: {"0d": 1}}, rng)
        arm.P.linalg.check(arm.lib.abft_dist_get_matrix(f._ctx, arm.P._lib.dptr(pinned_out), n))
        dt = all_max(time.perf_counter() - t0)
        if i:
            times.append(dt)
    sec = statistics.median(times)
    return {"value": FLOPS[args.kind](n) / sec / 1e12, "unit": "TFLOP/s",
            "h2d_bytes_per_step": 8 * n * n, "d2h_bytes_per_step": 8 * n * n,
            "ms_per_step": sec * 1e3,
            "api": "DistributedFactorization.set_matrix + run_protected + abft_dist_get_matrix "
                   "(per rank, its column blocks; bytes summed over ranks)"}


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
