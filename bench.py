#!/usr/bin/env python
"""Benchmark of the B200 GRF generator (driver contract: one JSON line on rank 0).

Workload (default, BASELINE.json configs[1] = "c2"): 2D 512x512 periodic grid
on [0,1)^2, fp32, a batch of 1024 independent fields (seeds 0..1023 = Philox
field index), Matern spectral density nu=1.5, length 0.1; Algorithm 2 is the
headline ("value"), Algorithm 1 is timed too ("alg1"). One step = one batch.
Weak scaling: rank r generates fields [r*B, (r+1)*B). No input tensors exist
(fields are generated from (seed, field) keys); the 1 GiB output per step per
GPU is larger than the 126 MB L2, so no L2 flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c1..c5]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MEASURED_PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
TRAFFIC_JSON = os.path.join(ROOT, "profiles", "ncu_traffic.json")
HBM_FALLBACK_GBS = 6650.0

# name: counts, lengths, density (family, params), dtype, fields per GPU per step, algorithms
CONFIGS = {
    "c1": dict(counts=(512, 512), density=("gauss", 0.05), dtype="f64", fields=1, algs=(1,),
               desc="2D 512x512 fp64, Algorithm 2, single field, seed 0, Gaussian covariance ell=0.05"),
    "c2": dict(counts=(512, 512), density=("matern", 1.5, 0.1), dtype="f32", fields=1024, algs=(1, 0),
               desc="2D 512x512 fp32, batch 1024 fields, Matern nu=1.5 ell=0.1, Algorithms 2 and 1"),
    "c3": dict(counts=(4096, 4096), density=("matern", 0.5, 0.02), dtype="f32", fields=64, algs=(1,),
               desc="2D 4096x4096 fp32, batch 64 fields, Matern nu=0.5 ell=0.02, Algorithm 2"),
    "c4": dict(counts=(512, 512, 512), density=("gauss", 0.03), dtype="f32", fields=1, algs=(1,),
               desc="3D 512^3 fp32 single field, Gaussian covariance ell=0.03, Algorithm 2"),
    "c5": dict(counts=(1024, 1024), density=("matern", 2.5, 0.05), dtype="f32", fields=512, algs=(1,),
               desc="1024x1024 fp32 SPDE steps, Matern nu=2.5 ell=0.05, Algorithm 2, 512 steps/GPU/batch"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--slab", action="store_true", help="c4: force the slab (multi-GPU) leg, also at N=1")
    return ap.parse_args()


def hbm_peak():
    try:
        with open(MEASURED_PEAKS) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK_GBS, "fallback"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi sampled every 200 ms while the timed region runs."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.3)
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ reference arm
def density_oracle(po, cfg):
    d = len(cfg["counts"])
    fam = cfg["density"]
    if fam[0] == "gauss":
        return po.density("gauss", d, ell=fam[1])
    return po.density("matern", d, nu=fam[1], ell=fam[2])


def cpu_reference_rate(cfg, alg, nfields, threads):
    """The reference's own synthesize() (oracle/_ref: proj/core compiled
    unmodified; FFTW replaced by the API stand-in), one field per std::thread
    over `threads` host threads — the reference's batch pattern (stats.cpp:57-81)."""
    from oracle import pyoracle as po

    counts = cfg["counts"]
    lengths = (1.0,) * len(counts)
    if po.reference_available():
        lib, kind = po.Reference(), "reference"
        secs, _ = lib.bench_batch(counts, lengths, density_oracle(po, cfg), alg, 0, nfields, threads)
    else:  # the plain-C port (single thread per field, same batch pattern in Python threads is not used)
        import numpy as np

        lib, kind = po.Port(), "port"
        threads = 1
        draws = np.random.default_rng(0).standard_normal(lib.count_draws(counts, alg))
        t0 = time.perf_counter()
        for _ in range(nfields):
            lib.synthesize(counts, lengths, density_oracle(po, cfg), alg, draws)
        secs = time.perf_counter() - t0
    pts = float(nfields) * float(__import__("math").prod(counts))
    return pts / secs / 1e9, kind, threads, secs


def sized_sample(cfg, alg, threads, target_s):
    """Fields per sample so one sample takes ~target_s wall on `threads` threads
    (probe: one field per thread; 512^3 is a single field)."""
    import math

    if math.prod(cfg["counts"]) > 2 ** 26:
        return 1
    probe = max(1, threads)
    _, _, _, secs = cpu_reference_rate(cfg, alg, probe, threads)
    n = int(probe * target_s / max(secs, 1e-3))
    n = max(probe, (n // probe) * probe)
    return min(n, 2048 * probe)


def run_reference_arm(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    alg = cfg["algs"][0]
    # each step: a bounded sample of ~1 s wall on all host threads (the whole run stays within minutes)
    nfields = sized_sample(cfg, alg, threads, target_s=1.0)
    for _ in range(max(0, args.warmup)):
        cpu_reference_rate(cfg, alg, max(1, nfields // 4), threads)
    rates, secs_all = [], 0.0
    kind = "reference"
    for _ in range(args.steps):
        r, kind, used_threads, secs = cpu_reference_rate(cfg, alg, nfields, threads)
        rates.append(r)
        secs_all += secs
    value = statistics.median(rates)
    line = {
        "impl": "reference", "metric": "GRF grid points/sec (Gpts/s)", "value": value, "unit": "Gpts/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": secs_all / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["desc"], "counts": list(cfg["counts"]), "algorithm": alg},
        "cpu_baseline": {"value": value, "unit": "Gpts/s", "cores": used_threads, "kind": kind,
                         "sample": f"{nfields} fields per step through grf::synthesize (seed overload, "
                                   f"xoshiro substreams (0, j)), one field per std::thread"},
        "e2e": {"value": value, "unit": "Gpts/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)


# ------------------------------------------------------------------ our arm
# Algorithmic (compulsory) bytes per FIELD each kernel must move, as a function
# of (P points, |H| half cells, s = real bytes). See DESIGN.md §Roofline.
def kernel_alg_bytes(name, P, H, s):
    c = 2 * s
    table = {
        "c2r_last": H * c + P * s,          # read half spectrum, write field
        "fused_rows_c2r": P * s + P * s,    # read packed spectrum (P/2 complex), write field
        "fused_cols_gen": P * s,            # write packed column-transformed spectrum
        "fused2d_persistent": P * s,        # whole path in one kernel: compulsory field write only
        "fused2d_alg1_persistent": P * s,   # Algorithm 1, whole path in one kernel
        "fused3d_colgen": P * s,            # 3D pass A: generation + axis-0 FFT, writes W (P/2 complex)
        "fused3d_planes": P * s + P * s,    # 3D pass B: reads W, writes the field
        "gen_half": H * c,
        "line_c2c": 2 * H * c,
        "r2c_last_noise": H * c,
        "scale_half": 2 * H * c,
    }
    return table.get(name)


def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    from paper_1105_2737_b200 import grfc

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    counts = cfg["counts"]
    lengths = (1.0,) * len(counts)
    d = len(counts)
    fam = cfg["density"]
    dens = grfc.Density.gaussian_cov(d, fam[1]) if fam[0] == "gauss" else grfc.Density.matern(d, fam[1], fam[2])
    dtype = grfc.F64 if cfg["dtype"] == "f64" else grfc.F32
    B = cfg["fields"]
    P = 1
    for n in counts:
        P *= n
    s = 8 if dtype == grfc.F64 else 4
    H = grfc.half_cells(counts)
    stream = torch.cuda.current_stream()
    out = torch.empty((B,) + tuple(counts), dtype=torch.float64 if dtype == grfc.F64 else torch.float32,
                      device="cuda")
    first = rank * B

    def time_alg(alg, K, W, sampler=None):
        plan = grfc.Plan(counts, lengths, dens, alg, dtype, device=local)
        for _ in range(W):
            plan.generate(0, first, B, out.data_ptr(), P, stream.cuda_stream)
        launches = 0
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        torch.cuda.synchronize()
        start.record(stream)
        for _ in range(K):
            plan.generate(0, first, B, out.data_ptr(), P, stream.cuda_stream)
            launches += grfc.last_launch_count()
        end.record(stream)
        torch.cuda.synchronize()
        barrier()
        ms = max_over_ranks(start.elapsed_time(end) / K)
        return plan, ms, launches

    # ---- headline: Algorithm 2 (one-FFT overwrite), clocks sampled during warm-up + timed region
    main_alg = cfg["algs"][0]
    with ClockSampler(local) as clk:
        plan, ms, launches = time_alg(main_alg, args.steps, args.warmup)
    clocks = clk.summary()
    value = world * B * P / (ms / 1e3) / 1e9

    # ---- per-kernel timing pass (same calls, CUDA events around each launch on its stream)
    grfc.kernel_timing_enable(True)
    for _ in range(max(3, min(args.steps, 20))):
        plan.generate(0, first, B, out.data_ptr(), P, stream.cuda_stream)
    torch.cuda.synchronize()
    rows = grfc.kernel_timing_read()
    grfc.kernel_timing_enable(False)
    nsteps_timed = max(3, min(args.steps, 20))
    peak, peak_kind = hbm_peak()
    dom = max(rows.items(), key=lambda kv: kv[1][0])
    dname, (dms, dl) = dom
    fields_per_launch = B * nsteps_timed / dl
    per_field = kernel_alg_bytes(dname, P, H, s)
    traffic = None
    try:
        with open(TRAFFIC_JSON) as f:
            tj = json.load(f)
        key = f"{args.config}:{dname}"
        if key in tj:
            traffic = tj[key]["bytes_per_launch"]
    except Exception:
        pass
    roofline = None
    if per_field is not None:
        ach = per_field * fields_per_launch / (dms / dl / 1e3) / 1e9
        roofline = {"bound": "hbm", "kernel": dname, "achieved": ach, "peak": peak, "unit": "GB/s",
                    "frac": ach / peak, "traffic": traffic, "peak_kind": peak_kind,
                    "alg_bytes_per_launch": per_field * fields_per_launch,
                    "avg_launch_us": dms / dl * 1e3}
    # compute-side diagnostic: nominal FFT flops 2.5 P log2 P per field (benchFFT
    # convention, one C2R; Algorithm 1 would be 2x) against a measured FFMA2 peak, and which ceiling binds
    compute = None
    try:
        fp32_peak = grfc.measure_fp32_peak(local)
        flops = 2.5 * P * math.log2(P) * B
        t_meas = ms / 1e3
        t_hbm = B * P * s / (peak * 1e9)
        t_fp = flops / (fp32_peak * 1e12)
        compute = {"nominal_fft_tflops": flops / t_meas / 1e12, "fp32_peak_tflops": fp32_peak,
                   "frac": flops / t_meas / 1e12 / fp32_peak, "t_hbm_us": t_hbm * 1e6, "t_fp32_us": t_fp * 1e6,
                   "t_measured_us": t_meas * 1e6, "binding": "fp32" if t_fp > t_hbm else "hbm",
                   "t_roof_frac": max(t_hbm, t_fp) / t_meas,
                   "note": "peak = packed FFMA2 probe (grfc_measure_fp32_peak) on this GPU; the path also "
                           "spends issue slots on Philox, Box-Muller, density and exchanges"}
    except Exception as e:  # noqa: BLE001
        compute = {"error": str(e)}
    path_gbs = B * P * s / (ms / 1e3) / 1e9
    kernels = {k: {"ms_per_step": v[0] / nsteps_timed, "launches_per_step": v[1] / nsteps_timed}
               for k, v in rows.items()}

    # ---- Algorithm 1, same batch
    alg1 = None
    if len(cfg["algs"]) > 1:
        _, ms1, _ = time_alg(cfg["algs"][1], max(3, args.steps // 2), args.warmup)
        alg1 = {"value": world * B * P / (ms1 / 1e3) / 1e9, "unit": "Gpts/s", "ms_per_step": ms1,
                "algorithm": "two_fft"}

    # ---- end to end through the public host API: D2H of every field inside the timed region
    host = torch.empty(out.shape, dtype=out.dtype, pin_memory=True)
    Ke = max(2, min(args.steps, 10))
    for _ in range(1):
        plan.generate_host_ptr(0, first, B, host.data_ptr(), stream.cuda_stream)
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(Ke):
        plan.generate_host_ptr(0, first, B, host.data_ptr(), stream.cuda_stream)
    t1 = time.perf_counter()
    barrier()
    ems = max_over_ranks((t1 - t0) / Ke * 1e3)
    e2e = {"value": world * B * P / (ems / 1e3) / 1e9, "unit": "Gpts/s", "h2d_bytes_per_step": 0,
           "d2h_bytes_per_step": B * P * s, "ms_per_step": ems,
           "note": "inputs are (seed, field range) scalars; every field is copied to pinned host memory"}

    # ---- CPU baseline (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        try:
            nf = sized_sample(cfg, main_alg, threads, target_s=10.0)  # ~10 s of host work
            rate, kind, used, secs = cpu_reference_rate(cfg, main_alg, nf, threads)
            cpu = {"value": rate, "unit": "Gpts/s", "cores": used, "kind": kind,
                   "sample": f"{nf} fields of this workload (Algorithm {main_alg + 1 if main_alg else 1}, fp64) "
                             f"through the reference grf::synthesize, one field per std::thread; {secs:.2f} s wall",
                   "fft": "FFTW API stand-in (oracle/fft_core.c); FFTW absent from the image"}
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": "Gpts/s", "cores": 0, "kind": "unavailable", "sample": str(e)}
        if len(counts) == 2:  # FFTW-class check beside it: scipy.fft (pocketfft), transform only
            try:
                from oracle import fftw_class_proxy as fp

                pr, psecs = fp.rate(counts, (1.0, 1.0), cfg["density"], 64, threads)
                nfp = max(64, int(64 * 5.0 / max(psecs, 1e-3)) // 16 * 16)  # ~5 s sample
                pr, psecs = fp.rate(counts, (1.0, 1.0), cfg["density"], nfp, threads)
                cpu["fftw_class_fft_only"] = {
                    "value": pr, "unit": "Gpts/s", "cores": threads,
                    "sample": f"{nfp} inverse real 2D FFTs only (scipy.fft.irfft2 / pocketfft, workers={threads}, "
                              f"fp64, {psecs:.2f} s): a production CPU FFT library on the transform alone, to compare with "
                              f"the reference's whole path on the FFTW stand-in"}
            except Exception as e:  # noqa: BLE001
                cpu["fftw_class_fft_only"] = {"value": None, "error": str(e)}

    if rank == 0:
        line = {
            "metric": "GRF grid points/sec (Gpts/s)", "value": value, "unit": "Gpts/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": cfg["dtype"], "data": "synthetic",
            "config": {"workload": cfg["desc"], "config": args.config, "counts": list(counts),
                       "fields_per_gpu_per_step": B, "algorithm": "one_fft_overwrite" if main_alg == 1 else "two_fft",
                       "path": plan.path, "parallelism": f"batch-sharded x{world} (no collective)",
                       "l2": "no inputs; output per step per GPU (%d MiB) %s L2 (126 MB)" % (
                           B * P * s >> 20, ">" if B * P * s > 126e6 else "<=")},
            "hbm_gbs_path": path_gbs,
            "path_roofline": {"bound": "hbm", "achieved": path_gbs, "peak": peak, "unit": "GB/s",
                              "frac": path_gbs / peak,
                              "note": "compulsory P*s output bytes per field / whole-path time (SURVEY 8d)"},
            "roofline": roofline, "compute_roofline": compute, "kernels": kernels, "alg1": alg1, "e2e": e2e, "cpu_baseline": cpu,
            "gpu_launches": launches, "clocks": clocks,
        }
        emit(line)
    if world > 1:
        dist.destroy_process_group()


def run_slab(args, cfg):
    """c4 on N > 1 GPUs: ONE 512^3 field slab-decomposed over the ranks
    (strong scaling). Per step: pass A (generation + axis-0 FFT of the rank's
    spectrum slab) -> NCCL all_to_all_single of contiguous blocks over NVLink
    -> pass B (axis-1/2 FFTs of the rank's field planes). include/grfc.h
    grfc_slab_*."""
    import torch
    import torch.distributed as dist

    from paper_1105_2737_b200 import grfc

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29517")
    os.environ.setdefault("WORLD_SIZE", str(world))
    os.environ.setdefault("RANK", str(rank))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    counts = cfg["counts"]
    d = len(counts)
    dens = grfc.Density.gaussian_cov(d, cfg["density"][1])
    plan = grfc.Plan(counts, (1.0,) * d, dens, grfc.ONE_FFT_OVERWRITE, grfc.F32, device=local)
    buf, block, slab_pts = plan.slab_sizes(world)
    out = torch.empty(slab_pts, dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()
    # the library's own data plane: an NCCL communicator bootstrapped from rank 0's
    # unique id (broadcast over the torch process group), then per field
    # grfc_slab_generate = pass A -> grouped ncclSend/ncclRecv -> pass B
    uid = [grfc.comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = grfc.Comm(uid[0], world, rank, local)

    def step(field):
        plan.slab_generate(comm, 0, field, out.data_ptr(), stream.cuda_stream)

    for i in range(args.warmup):
        step(i)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        dist.barrier()
        torch.cuda.synchronize()
        start.record(stream)
        for i in range(args.steps):
            step(i)
        end.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
    t = torch.tensor([start.elapsed_time(end) / args.steps], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    P = 1
    for n in counts:
        P *= n
    value = P / (ms / 1e3) / 1e9
    # end to end: the rank's slab copied to pinned host memory every step
    host = torch.empty(slab_pts, dtype=torch.float32, pin_memory=True)
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(max(2, min(args.steps, 5))):
        step(i)
        host.copy_(out, non_blocking=False)
    e2e_ms = (time.perf_counter() - t0) / max(2, min(args.steps, 5)) * 1e3
    te = torch.tensor([e2e_ms], dtype=torch.float64, device="cuda")
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    peak, kind = hbm_peak()
    if rank == 0:
        nvl = 2 * buf * 4 * (world - 1) / world  # bytes each rank sends over NVLink per step
        line = {
            "metric": "GRF grid points/sec (Gpts/s)", "value": value, "unit": "Gpts/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": cfg["desc"], "config": args.config, "counts": list(counts),
                       "parallelism": f"slab x{world} (grfc_slab_generate: pass A, NCCL grouped send/recv, pass B)",
                       "path": plan.path, "l2": "output 512 MiB per step > L2"},
            "path_roofline": {"bound": "hbm", "achieved": P * 4 / (ms / 1e3) / 1e9 / world, "peak": peak,
                              "unit": "GB/s per GPU", "frac": P * 4 / (ms / 1e3) / 1e9 / world / peak},
            "nvlink_bytes_per_rank_per_step": nvl,
            "e2e": {"value": P / (float(te.item()) / 1e3) / 1e9, "unit": "Gpts/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": P * 4, "ms_per_step": float(te.item())},
            "gpu_launches": 2 * args.steps, "clocks": clk.summary(), "cpu_baseline": None,
        }
        emit(line)
    del comm
    dist.destroy_process_group()


_JSON_FD = None


def emit(line):
    """The one JSON line, on the process's original stdout (see main)."""
    data = (json.dumps(line) + "\n").encode()
    if _JSON_FD is None:
        sys.stdout.write(data.decode())
        sys.stdout.flush()
    else:
        os.write(_JSON_FD, data)


def main():
    global _JSON_FD
    # Library banners written to fd 1 from C code (e.g. NCCL's version line at
    # communicator creation) would precede the JSON line: route fd 1 to stderr for
    # the run and keep the original stdout for the result alone.
    sys.stdout.flush()
    _JSON_FD = os.dup(1)
    os.dup2(2, 1)
    args = parse()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference_arm(args, cfg)
    elif args.config == "c4" and (int(os.environ.get("WORLD_SIZE", "1")) > 1 or args.slab):
        run_slab(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
