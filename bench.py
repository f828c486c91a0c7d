#!/usr/bin/env python
"""Benchmark of the FlashFPS hot path on B200 (BASELINE.json metric:
"4-stage FPS clouds/sec & ms/cloud at N=200K; speedup vs exhaustive CUDA FPS").

Workload (BASELINE.json configs[4], "C5" in SURVEY.md §8d): per rank a batch of
64 synthetic clouds of N=200,000 fp32 points (uniform unit cube, cloud b drawn
from numpy default_rng(b), reference io.py:209-210), 4-stage budgets
50000/12500/3125/781 (1/4 downsampling).  One step = hierarchical_sample of
the whole batch with FPS-Prune p=0.75 + FPS-Cache (the FlashFPS pipeline:
K1 greedy over the 50,000-point candidate prefix for 12,500 iterations, K2
budget fill, layers 2-4 as prefix views) — plus, for N>1 ranks, the layer-1
index gather.  The comparison arm is the same build's exhaustive 4-stage
CUDA FPS (p=0, cache off: 200K->50K, then 50K->12.5K, 12.5K->3125,
3125->781 restricted runs).

Arms:
  python bench.py [--gpus N --steps K --warmup W]        ours (one JSON line)
  python bench.py --impl reference ...                   the reference's CPU
      algorithm (the oracle port, oracle/) on all host cores, same metric.
Multi-GPU: torchrun, one rank per GPU, weak scaling (64 clouds per rank),
timing = max over ranks of CUDA-event time.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

BUDGETS = {200_000: (50_000, 12_500, 3_125, 781), 300_000: (75_000, 18_750, 4_687, 1_171),
           100_000: (25_000, 6_250, 1_562, 390), 24_000: (6_000, 1_500, 375, 93)}
BYTES_PER_UNIT_F32 = 20   # 12 B xyz read + 4 B dist read + 4 B dist write
FLOPS_PER_UNIT = 9        # 3 sub + 3 mul + 2 add + 1 min
METRIC = "4-stage FPS clouds/sec at N=200K (FPS-Prune p=0.75 + FPS-Cache)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--batch", type=int, default=64, help="clouds per rank")
    ap.add_argument("--n", type=int, default=200_000)
    ap.add_argument("--p", type=float, default=0.75)
    ap.add_argument("--cloud", choices=["uniform", "lidar"], default="uniform")
    ap.add_argument("--exh-steps", type=int, default=None,
                    help="timed steps of the exhaustive arm (default: --steps)")
    ap.add_argument("--no-exhaustive", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-clouds", type=int, default=None,
                    help="clouds in the CPU sample (default: one per host core)")
    return ap.parse_args()


# --------------------------------------------------------------------- inputs
def lidar_cloud(n: int, seed: int) -> np.ndarray:
    """Deterministic LiDAR-like frame (no reference generator exists):
    64 beams from -25 to +3 degrees elevation, sensor 1.8 m above a ground
    plane, seeded box obstacles, range <= 80 m, 2 cm noise; ~1/r^2 density.
    Random draws come from numpy default_rng(seed); the ray/box slab tests run
    in torch (CUDA when available, else CPU) in float64."""
    import torch
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    rng = np.random.default_rng(seed)
    nb = 64
    elev = np.deg2rad(np.linspace(-25.0, 3.0, nb))
    boxes = np.column_stack([rng.uniform(-60, 60, 40), rng.uniform(-60, 60, 40),
                             rng.uniform(1.0, 6.0, 40), rng.uniform(1.0, 3.5, 40)])
    lo = torch.tensor(np.stack([boxes[:, 0] - boxes[:, 2], boxes[:, 1] - boxes[:, 2],
                                np.full(len(boxes), -1.8)], 1), device=dev)
    hi = torch.tensor(np.stack([boxes[:, 0] + boxes[:, 2], boxes[:, 1] + boxes[:, 2],
                                -1.8 + boxes[:, 3]], 1), device=dev)
    out = np.empty((0, 3))
    while out.shape[0] < n:
        m = 2 * n
        az = rng.uniform(-np.pi, np.pi, m)
        el = elev[rng.integers(0, nb, m)]
        d = np.stack([np.cos(el) * np.cos(az), np.cos(el) * np.sin(az), np.sin(el)], 1)
        r = np.full(m, 80.0)
        down = d[:, 2] < 0
        r[down] = np.minimum(80.0, 1.8 / -d[down, 2])
        dt = torch.tensor(d, device=dev)
        rt = torch.tensor(r, device=dev)
        for c0 in range(0, m, 1 << 16):   # slab test of every ray against every box
            iv = (1.0 / dt[c0:c0 + (1 << 16)])[:, None, :]
            t1, t2 = lo[None] * iv, hi[None] * iv
            tmin = torch.nan_to_num(torch.minimum(t1, t2), nan=-torch.inf).amax(2)
            tmax = torch.nan_to_num(torch.maximum(t1, t2), nan=torch.inf).amin(2)
            hit = (tmax >= tmin) & (tmin > 0)
            th = torch.where(hit, tmin, torch.full_like(tmin, torch.inf)).amin(1)
            rt[c0:c0 + (1 << 16)] = torch.minimum(rt[c0:c0 + (1 << 16)], th)
        r = rt.cpu().numpy()
        keep = r < 80.0
        p = d[keep] * r[keep, None] + rng.normal(0, 0.02, (int(keep.sum()), 3))
        out = np.vstack([out, p])
    return out[rng.permutation(out.shape[0])[:n]].astype(np.float32)


def make_clouds(kind: str, batch: int, n: int, first: int) -> np.ndarray:
    out = np.empty((batch, n, 3), dtype=np.float32)
    for b in range(batch):
        if kind == "uniform":
            out[b] = np.random.default_rng(first + b).random((n, 3))
        else:
            out[b] = lidar_cloud(n, first + b)
    return out


# ------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 50 ms while the
    timed region runs (B200_PROFILING.md clocks line); one query right after
    the region if it ended before the first sample."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "50", "-i", str(self.index)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [ln for ln in out.splitlines() if ln.strip()]
            if not self.lines:  # region shorter than the first sample: query once now
                try:
                    self.lines = [ln for ln in subprocess.run(
                        ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                         "-i", str(self.index)], capture_output=True, text=True,
                        timeout=10).stdout.splitlines() if ln.strip()]
                except (OSError, subprocess.TimeoutExpired):
                    self.lines = []
        return False

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in getattr(self, "lines", []):
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------- helpers
# Test-only switch: every rank on cuda:0 with gloo collectives, to exercise the
# multi-rank path (barriers, max-over-ranks timing, index gather) on a 1-GPU box.
# The ranks' kernels never wait on each other; the numbers it prints are not a
# scaling measurement.
SHARE_GPU = os.environ.get("FFPS_BENCH_SHARE_GPU") == "1"


def gpu_index(local_rank: int) -> int:
    return 0 if SHARE_GPU else local_rank

def peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return {"hbm_gbs": float(d["hbm_gbs"]), "src": "measured (MEASURED_PEAKS.json)",
                "sm_max_mhz": float(d.get("sm_max_mhz", 1965.0))}
    except (OSError, KeyError, ValueError):
        return {"hbm_gbs": 6650.0, "src": "fallback (B200_PROFILING.md)", "sm_max_mhz": 1965.0}


def stage_units(n: int, budgets, p: float, cache: bool) -> list[tuple[int, int]]:
    """(candidates, iterations) of every greedy launch of one cloud; units =
    candidates * (iterations - 1) = the reference's distance_evals."""
    from paper_2604_17720_b200 import PruneConfig
    cfg = PruneConfig(p=p)
    k = cfg.kernel_budget(budgets[0])
    c = min(cfg.candidate_count(n, budgets[0]), n)
    out = [(c, k)]
    if not cache:
        prev = budgets[0]
        for m in budgets[1:]:
            out.append((prev, m))
            prev = m
    return out


def cpu_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_pipeline_sample(n: int, budgets, p: float, clouds: int, kind: str, threads: int):
    """The reference algorithm on the host (oracle port, oracle/fps_oracle.c,
    restating fps_core.py:110-175 + fps_prune.py:68-111 + fps_cache.py:204-240),
    one cloud per thread: returns (seconds, clouds)."""
    from oracle import oracle
    xyz = make_clouds(kind, clouds, n, 10_000)
    k = max(1, math.floor((1.0 - p) * budgets[0]))
    c = min(max(k, math.floor((1.0 - p) * n)), n)
    t0 = time.perf_counter()
    order, sel = oracle.run_kernel_batch(xyz, k, np.zeros(clouds, np.int64), n=c,
                                         threads=threads)
    if budgets[0] > k:
        for b in range(clouds):
            oracle.fill_slice(order[b], n, budgets[0] - k)
    return time.perf_counter() - t0, clouds


def emit(obj):
    print(json.dumps(obj), flush=True)


# ----------------------------------------------------------- reference arm
def run_reference(args, rank: int, world: int):
    if rank != 0:
        return
    budgets = BUDGETS[args.n]
    cores = cpu_cores()
    clouds = args.cpu_clouds or cores
    for _ in range(min(args.warmup, 1)):
        cpu_pipeline_sample(args.n, budgets, args.p, min(clouds, cores), args.cloud, cores)
    times = []
    for _ in range(args.steps):
        dt, cnt = cpu_pipeline_sample(args.n, budgets, args.p, clouds, args.cloud, cores)
        times.append(dt)
    sec = float(np.mean(times))
    val = clouds / sec
    sample = (f"{clouds} clouds of N={args.n} {args.cloud} per step, FPS-Prune p={args.p} "
              f"+ FPS-Cache 4-stage {budgets}, one cloud per host thread")
    emit({"metric": METRIC, "impl": "reference", "value": val, "unit": "clouds/s",
          "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
          "ms_per_step": sec * 1e3, "ms_per_cloud": sec * 1e3 / clouds * cores,
          "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
          "dtype": "f32", "data": "synthetic",
          "config": {"workload": f"C5 FlashFPS 4-stage N={args.n}", "n": args.n,
                     "budgets": list(budgets), "p": args.p, "cache": True,
                     "cloud": args.cloud, "clouds_per_step": clouds},
          "cpu_baseline": {"value": val, "unit": "clouds/s", "cores": cores, "kind": "port",
                           "sample": sample},
          "e2e": {"value": val, "unit": "clouds/s", "h2d_bytes_per_step": 0,
                  "d2h_bytes_per_step": 0}})


# ------------------------------------------------------------------ our arm
def run_ours(args, rank: int, world: int, local_rank: int):
    import torch
    import torch.distributed as dist

    import paper_2604_17720_b200 as ffps
    from paper_2604_17720_b200 import _device, _native
    from paper_2604_17720_b200.sharded import gather_rows

    torch.cuda.set_device(gpu_index(local_rank))
    dev = torch.device("cuda", gpu_index(local_rank))
    _native.load()
    budgets = BUDGETS[args.n]
    B = args.batch
    global_batch = B * world
    cfg_flash = ffps.PruneConfig(p=args.p)
    cfg_exh = ffps.PruneConfig(p=0.0)

    host = make_clouds(args.cloud, B, args.n, rank * B)
    x = torch.from_numpy(host).to(dev)
    pinned = torch.from_numpy(host).pin_memory()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > L2

    def barrier():
        if world > 1:
            dist.barrier()

    def step(xin, cfg, cache):
        layers, total, _ = ffps.hierarchical_sample_batch(xin, budgets, cfg, 0, cache)
        if world > 1:
            gather_rows(layers[0].indices, global_batch)
        return layers, total

    def ramp(seconds=1.0):
        """Untimed load before the warm-up steps: a fresh box idles at low SM
        clocks and needs a moment under load to reach its boost clock.
        Time-bounded, so the ranks run different numbers of steps here: no
        collective (the gather) inside, or the ranks' collectives mismatch."""
        t0 = time.perf_counter()
        while time.perf_counter() - t0 < seconds:
            ffps.hierarchical_sample_batch(x, budgets, cfg_flash, 0, True)
            torch.cuda.synchronize()
        barrier()

    def timed(cfg, cache, steps, warmup, timer=False):
        for _ in range(warmup):
            step(x, cfg, cache)
        torch.cuda.synchronize()
        barrier()
        ms, kern = [], []
        l0 = _device.launches()
        for _ in range(steps):
            flush.zero_()
            s = torch.cuda.Event(enable_timing=True)
            e = torch.cuda.Event(enable_timing=True)
            if timer:
                with _device.kernel_timer() as kt:
                    s.record()
                    step(x, cfg, cache)
                    e.record()
            else:
                kt = None
                s.record()
                step(x, cfg, cache)
                e.record()
            torch.cuda.synchronize()
            ms.append(s.elapsed_time(e))
            if kt is not None:
                kern.extend(kt.kernel_ms())
        launches = _device.launches() - l0
        barrier()
        tot = torch.tensor([sum(ms)], dtype=torch.float64, device="cpu" if SHARE_GPU else dev)
        if world > 1:
            dist.all_reduce(tot, op=dist.ReduceOp.MAX)
        return float(tot.item()), ms, kern, launches

    vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
    phys = vis.split(",")[gpu_index(local_rank)] if vis and vis.split(",")[0].isdigit() \
        else str(gpu_index(local_rank))
    ramp()
    with ClockSampler(int(phys)) as clk:
        tot_ms, ms, kern, launches = timed(cfg_flash, True, args.steps, args.warmup, timer=True)
    clocks = clk.summary()
    ms_step = tot_ms / args.steps
    value = global_batch / (ms_step / 1e3)

    # end to end through the public host API: pinned host clouds in, host
    # indices + selection distances out, every step
    out_i = torch.empty((B, budgets[0]), dtype=torch.int64).pin_memory()
    out_s = torch.empty((B, budgets[0]), dtype=torch.float32).pin_memory()
    for _ in range(args.warmup):
        ffps.hierarchical_sample_host(pinned, budgets, cfg_flash, out=(out_i, out_s))
    barrier()
    e2e_ms = []
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        ffps.hierarchical_sample_host(pinned, budgets, cfg_flash, out=(out_i, out_s))
        e.record()
        torch.cuda.synchronize()
        e2e_ms.append(s.elapsed_time(e))
    e2e_tot = torch.tensor([sum(e2e_ms)], dtype=torch.float64,
                           device="cpu" if SHARE_GPU else dev)
    if world > 1:
        dist.all_reduce(e2e_tot, op=dist.ReduceOp.MAX)
    e2e_step = float(e2e_tot.item()) / args.steps
    e2e_val = global_batch / (e2e_step / 1e3)
    c1_, _ = stage_units(args.n, budgets, args.p, True)[0]
    h2d = B * c1_ * 3 * 4   # cache on: only the candidate prefix is read (fps_prune.py:92)
    d2h = B * budgets[0] * (8 + 4)

    # exhaustive 4-stage arm of the same build (the paper's "standard CUDA FPS")
    exh = None
    exh_std = None
    flash_std = None
    if not args.no_exhaustive:
        ks = args.exh_steps or args.steps
        ex_units = sum(c * (m - 1) for c, m in stage_units(args.n, budgets, 0.0, False)) * B

        def arm(cfg, cache, schedule, steps):
            prev = _device.set_schedule(schedule)
            try:
                tot, _, kk, _ = timed(cfg, cache, steps, min(args.warmup, 3), timer=True)
            finally:
                _device.set_schedule(prev)
            return tot / steps, kk

        # exhaustive 4-stage (p=0, cache off) with the headline's own schedule
        ex_step, ex_kern = arm(cfg_exh, False, "auto", ks)
        exh = {"value": global_batch / (ex_step / 1e3), "unit": "clouds/s",
               "ms_per_step": ex_step, "ms_per_cloud": ex_step / B, "steps": ks,
               "schedule": "auto (" + _native.auto_schedule(args.n, B) + ")",
               "stage1_kernel_ms": float(np.mean([k[3] for k in ex_kern if k[1] == args.n])),
               "units_per_step": ex_units,
               "speedup_flash_vs_exhaustive": ex_step / ms_step}
        # the paper's baseline: standard FPS (every point every iteration, K1)
        sd_step, sd_kern = arm(cfg_exh, False, "stream", max(2, ks // 3))
        exh_std = {"value": global_batch / (sd_step / 1e3), "unit": "clouds/s",
                   "ms_per_step": sd_step, "ms_per_cloud": sd_step / B,
                   "schedule": "stream (K1, standard exhaustive-update FPS)",
                   "stage1_kernel_ms": float(np.mean([k[3] for k in sd_kern if k[1] == args.n])),
                   "speedup_flash_vs_standard_exhaustive": sd_step / ms_step}
        fs_step, _ = arm(cfg_flash, True, "stream", max(2, ks // 3))
        flash_std = {"value": global_batch / (fs_step / 1e3), "unit": "clouds/s",
                     "ms_per_step": fs_step, "schedule": "stream (K1)",
                     "speedup_flash_stream_vs_standard_exhaustive": sd_step / fs_step}

    # matched sampling-quality metric (north star): covering radius of layer 1
    # (metrics.py:45-52) for FlashFPS vs the exhaustive run, every cloud
    quality = None
    if not args.no_exhaustive:
        fl_l, _, _ = ffps.hierarchical_sample_batch(x, budgets, cfg_flash, 0, True)
        ex_l, _, _ = ffps.hierarchical_sample_batch(x, budgets, cfg_exh, 0, False)
        torch.cuda.synchronize()
        qs, qe = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        qs.record()
        r_fl = ffps.coverage_radius_batch(x, fl_l[0].indices)
        qe.record()
        r_ex = ffps.coverage_radius_batch(x, ex_l[0].indices)
        torch.cuda.synchronize()
        ratio = (r_fl / r_ex).cpu().numpy()
        quality = {"metric": "coverage radius of layer 1 (k-center objective, metrics.py:45-52)",
                   "flash_mean": float(r_fl.mean()), "exhaustive_mean": float(r_ex.mean()),
                   "ratio_median": float(np.median(ratio)), "ratio_max": float(ratio.max()),
                   "coverage_kernel_ms_per_batch": qs.elapsed_time(qe), "clouds": B}

    # roofline of the dominant kernel (K1 on the flash stage)
    c1, k1 = stage_units(args.n, budgets, args.p, True)[0]
    units_launch = B * c1 * (k1 - 1)
    kms = float(np.mean([k[3] for k in kern])) if kern else float("nan")
    pk = peaks()
    achieved = units_launch * BYTES_PER_UNIT_F32 / (kms / 1e3) / 1e9
    sched_full = _native.auto_schedule(c1, B)   # e.g. "grid@2" = K1g, 2 CTAs per cloud
    sched = sched_full.split("@")[0]
    plan = {"schedule": sched, "schedule_auto": sched_full,
            **_native.bucket_plan(_native.F32, c1)} \
        if sched in ("bucket", "multi", "grid") else \
        {"schedule": "stream", **_native.plan(_native.F32, c1, B)}
    sm_mhz = clocks["sm_mhz"] or pk["sm_max_mhz"]
    issue_ceiling = 148 * 128 * sm_mhz * 1e6 / 9.0   # ~9 FP32-pipe instr / unit
    traffic = None
    try:  # per-launch DRAM bytes of the same kernel from one `ncu --set full` capture
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            tj = json.load(fh)
        kname = {"bucket": "fps_bucket_kernel", "multi": "fps_multi_kernel",
                 "grid": "fps_grid_kernel"}.get(plan["schedule"], "fps_greedy_kernel")
        hit = [v for k_, v in tj.items() if kname in k_]
        traffic = hit[0]["dram_bytes"] if hit else None
    except (OSError, ValueError, KeyError):
        traffic = None
    roof = {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
            "frac": achieved / pk["hbm_gbs"], "traffic": traffic,
            "kernel": {"bucket": "fps_bucket_kernel (K1b)", "multi": "fps_multi_kernel (K1m)",
                       "grid": "fps_grid_kernel (K1g)"}.get(plan["schedule"],
                                                           "fps_greedy_kernel (K1)"),
            "kernel_ms": kms,
            "units_per_launch": units_launch, "bytes_per_unit": BYTES_PER_UNIT_F32,
            "peak_src": pk["src"],
            "note": ("algorithmic bytes of the standard streaming FPS (20 B per point-"
                     "iteration = distance_evals) / time of one greedy call on the launching "
                     "stream (CUDA events around ffps_run_kernel: for K1b/K1m/K1g that is "
                     "the K0 bucket build plus the greedy kernel, so the greedy kernel alone "
                     "is faster than kernel_ms); >1 because the state stays on chip / in L2 "
                     "and the bucketed schedules skip provably unaffected buckets"),
            "issue_bound": {"achieved_units_per_s": units_launch / (kms / 1e3),
                            "ceiling_units_per_s": issue_ceiling,
                            "frac": units_launch / (kms / 1e3) / issue_ceiling,
                            "sm_mhz": sm_mhz},
            "latency": {"iterations": k1, "ns_per_iteration": kms * 1e6 / k1},
            "plan": plan}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = cpu_cores()
        clouds = args.cpu_clouds or cores
        dt, cnt = cpu_pipeline_sample(args.n, budgets, args.p, clouds, args.cloud, cores)
        cpu = {"value": cnt / dt, "unit": "clouds/s", "cores": cores, "kind": "port",
               "sample": f"{cnt} clouds of N={args.n} {args.cloud}, FPS-Prune p={args.p} + "
                         f"FPS-Cache, one cloud per host thread, {dt:.1f} s wall"}

    if rank == 0:
        emit({"metric": METRIC, "value": value, "unit": "clouds/s", "n_gpus": world,
              "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
              "ms_per_cloud": ms_step / B, "higher_is_better": True, "scaling": "weak",
              "vs_baseline": None, "dtype": "f32", "data": "synthetic",
              "config": {"workload": f"C5 FlashFPS 4-stage N={args.n} (BASELINE configs[4])",
                         "n": args.n, "budgets": list(budgets), "p": args.p, "cache": True,
                         "clouds_per_rank": B, "global_batch": global_batch,
                         "cloud": args.cloud, "parallelism": f"shard-by-cloud x{world}",
                         "l2": "256 MiB flush write between timed steps"},
              "e2e": {"value": e2e_val, "unit": "clouds/s", "ms_per_step": e2e_step,
                      "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
              "gpu_launches": launches, "roofline": roof, "exhaustive": exh,
              "exhaustive_standard": exh_std, "flash_standard_schedule": flash_std,
              "quality": quality,
              "cpu_baseline": cpu, "clocks": clocks,
              "step_ms": [round(v, 4) for v in ms]})


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(gpu_index(local_rank))
        if SHARE_GPU:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
