#!/usr/bin/env python
"""Benchmark of the FlashFPS hot path on B200 (BASELINE.json metric:
"4-stage FPS clouds/sec & ms/cloud at N=200K; speedup vs exhaustive CUDA FPS").

Workload (BASELINE.json configs[4], "C5" in SURVEY.md §8d): a global batch of
64 synthetic clouds of N=200,000 fp32 points (uniform unit cube, cloud b drawn
from numpy default_rng(b), reference io.py:209-210), 4-stage budgets
50000/12500/3125/781 (1/4 downsampling), computed in binary64 like the
reference (fps_core.py:74-83; the fp32 clouds upcast exactly, geometry.py:52-54;
the kernels keep the coordinates as float and do every rounded operation in
binary64: FFPS_F32_F64).  One step = hierarchical_sample of the batch with
FPS-Prune p=0.75 + FPS-Cache (the FlashFPS pipeline: K0 bucket build + K1g
greedy over the 50,000-point candidate prefix for 12,500 iterations, K2 budget
fill, layers 2-4 as prefix views) — plus, for N>1 ranks, the layer-1 index
gather.  The comparison arm is the same build's exhaustive 4-stage CUDA FPS
(p=0, cache off: 200K->50K, then 50K->12.5K, 12.5K->3125, 3125->781
restricted runs), also binary64.

Arms:
  python bench.py [--gpus N --steps K --warmup W]        ours (one JSON line)
  python bench.py --impl reference ...                   the reference's CPU
      algorithm in binary64 (the oracle port, oracle/) on all host cores.
Multi-GPU: one rank per GPU (torchrun; `--gpus N` without torchrun re-launches
itself under torch.distributed.run).  Strong scaling by default: the global
batch of 64 clouds is split by cloud (sharded.shard_range); `--batch B` gives
weak scaling (B clouds per rank).  Timing = max over ranks of CUDA-event time.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import socket
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

BUDGETS = {200_000: (50_000, 12_500, 3_125, 781), 300_000: (75_000, 18_750, 4_687, 1_171),
           100_000: (25_000, 6_250, 1_562, 390), 24_000: (6_000, 1_500, 375, 93)}
BYTES_PER_UNIT = {"f32": 20, "f64": 40}  # xyz read + dist read + dist write
METRIC = "4-stage FPS clouds/sec at N=200K (FPS-Prune p=0.75 + FPS-Cache)"
PREC_CODE = {"f32": 0, "f64": 2}   # ABI dtype of the fp32 clouds: binary32 / FFPS_F32_F64


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--global-batch", type=int, default=64,
                    help="clouds per step over all ranks (strong scaling; BASELINE configs[4])")
    ap.add_argument("--batch", type=int, default=None,
                    help="clouds per rank (weak scaling; overrides --global-batch)")
    ap.add_argument("--n", type=int, default=200_000)
    ap.add_argument("--p", type=float, default=0.75)
    ap.add_argument("--dtype", choices=["f64", "f32"], default="f64",
                    help="arithmetic: f64 = the reference's binary64 (headline)")
    ap.add_argument("--cloud", choices=["uniform", "lidar"], default="uniform")
    ap.add_argument("--exh-steps", type=int, default=None,
                    help="timed steps of the exhaustive arm (default: --steps)")
    ap.add_argument("--no-exhaustive", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the secondary measurements (f32 arm, divergence, quality)")
    ap.add_argument("--cpu-clouds", type=int, default=None,
                    help="clouds in the CPU sample (default: one per host core)")
    return ap.parse_args(argv)


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


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_pipeline_sample(n: int, budgets, p: float, clouds: int, kind: str, threads: int,
                        dtype: str):
    """The reference algorithm on the host (oracle port, oracle/fps_oracle.c,
    restating fps_core.py:110-175 + fps_prune.py:68-111 + fps_cache.py:204-240),
    one cloud per thread, binary64 on the upcast fp32 clouds (or binary32):
    returns (seconds, clouds)."""
    from oracle import oracle
    xyz = make_clouds(kind, clouds, n, 10_000)
    if dtype == "f64":
        xyz = xyz.astype(np.float64)
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


def shard(args, world: int, rank: int) -> tuple[int, int, int, str]:
    """(first cloud, clouds on this rank, global batch, scaling)."""
    from paper_2604_17720_b200.sharded import shard_range
    if args.batch is not None:
        return rank * args.batch, args.batch, args.batch * world, "weak"
    lo, hi = shard_range(args.global_batch, world, rank)
    return lo, hi - lo, args.global_batch, "strong"


# ----------------------------------------------------------- reference arm
def run_reference(args, rank: int, world: int):
    if rank != 0:
        return
    budgets = BUDGETS[args.n]
    cores = cpu_cores()
    clouds = args.cpu_clouds or 2 * cores   # each step ~2.5 s of host work
    for _ in range(min(args.warmup, 1)):
        cpu_pipeline_sample(args.n, budgets, args.p, min(clouds, cores), args.cloud, cores,
                            args.dtype)
    times = []
    for _ in range(args.steps):
        dt, cnt = cpu_pipeline_sample(args.n, budgets, args.p, clouds, args.cloud, cores,
                                      args.dtype)
        times.append(dt)
    sec = float(np.mean(times))
    val = clouds / sec
    sample = (f"{clouds} clouds of N={args.n} {args.cloud} per step, FPS-Prune p={args.p} "
              f"+ FPS-Cache 4-stage {budgets}, binary{64 if args.dtype == 'f64' else 32}, "
              f"one cloud per host thread on {cores} threads ({cpu_model()})")
    _, _, gb, scaling = shard(args, world, 0)
    emit({"metric": METRIC, "impl": "reference", "value": val, "unit": "clouds/s",
          "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
          "ms_per_step": sec * 1e3, "ms_per_cloud": sec * 1e3 / clouds * cores,
          "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
          "dtype": args.dtype, "data": "synthetic",
          "config": {"workload": f"C5 FlashFPS 4-stage N={args.n} (BASELINE configs[4])",
                     "n": args.n, "budgets": list(budgets), "p": args.p, "cache": True,
                     "cloud": args.cloud, "global_batch": gb, "clouds_per_step": clouds},
          "cpu_baseline": {"value": val, "unit": "clouds/s", "cores": cores, "kind": "port",
                           "cpu": cpu_model(), "sample": sample},
          "e2e": {"value": val, "unit": "clouds/s", "h2d_bytes_per_step": 0,
                  "d2h_bytes_per_step": 0}})


# ------------------------------------------------------------------ our arm
def divergence(a: "torch.Tensor", b: "torch.Tensor", n: int) -> dict:
    """Per-cloud comparison of two (B, k) index orders of the same clouds:
    first differing position (-1: identical), positions that differ, and the
    overlap of the two selected sets (|A & B| / k)."""
    import torch
    B, k = a.shape
    diff = a != b
    anyd = diff.any(1)
    first = torch.where(anyd, diff.int().argmax(1), torch.full_like(anyd, -1, dtype=torch.int64))
    mask = torch.zeros((B, n), dtype=torch.int8, device=a.device)
    mask.scatter_(1, a, 1)
    inter = mask.gather(1, b).sum(1)
    return {"clouds": B, "k": k,
            "identical_clouds": int((~anyd).sum()),
            "first_divergence": [int(v) for v in first.cpu()],
            "mismatched_positions": [int(v) for v in diff.sum(1).cpu()],
            "set_overlap": [round(float(v) / k, 6) for v in inter.cpu()]}


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
    first, B, global_batch, scaling = shard(args, world, rank)
    prec = args.dtype                       # arithmetic of the headline
    cfg_flash = ffps.PruneConfig(p=args.p)
    cfg_exh = ffps.PruneConfig(p=0.0)

    host = make_clouds(args.cloud, B, args.n, first)
    x = torch.from_numpy(host).to(dev)     # fp32 clouds resident in HBM
    pinned = torch.from_numpy(host).pin_memory()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > L2

    def barrier():
        if world > 1:
            dist.barrier()

    def step(cfg, cache, precision=prec):
        layers, total, _ = ffps.hierarchical_sample_batch(x, budgets, cfg, 0, cache,
                                                          precision=precision)
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
            ffps.hierarchical_sample_batch(x, budgets, cfg_flash, 0, True, precision=prec)
            torch.cuda.synchronize()
        barrier()

    def timed(cfg, cache, steps, warmup, timer=False, precision=prec):
        for _ in range(warmup):
            step(cfg, cache, precision)
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
                    step(cfg, cache, precision)
                    e.record()
            else:
                kt = None
                s.record()
                step(cfg, cache, precision)
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

    # end to end through the public host API: pinned fp32 host clouds in, host
    # indices + binary64 selection distances out, every step
    out_i = torch.empty((B, budgets[0]), dtype=torch.int64).pin_memory()
    out_s = torch.empty((B, budgets[0]),
                        dtype=torch.float64 if prec == "f64" else torch.float32).pin_memory()
    for _ in range(args.warmup):
        ffps.hierarchical_sample_host(pinned, budgets, cfg_flash, out=(out_i, out_s),
                                      precision=prec)
    barrier()
    e2e_ms = []
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        ffps.hierarchical_sample_host(pinned, budgets, cfg_flash, out=(out_i, out_s),
                                      precision=prec)
        e.record()
        torch.cuda.synchronize()
        e2e_ms.append(s.elapsed_time(e))
    e2e_tot = torch.tensor([sum(e2e_ms)], dtype=torch.float64,
                           device="cpu" if SHARE_GPU else dev)
    if world > 1:
        dist.all_reduce(e2e_tot, op=dist.ReduceOp.MAX)
    e2e_step = float(e2e_tot.item()) / args.steps
    e2e_val = global_batch / (e2e_step / 1e3)
    c1_, k1_ = stage_units(args.n, budgets, args.p, True)[0]
    h2d = B * c1_ * 3 * 4   # cache on: only the fp32 candidate prefix is read (fps_prune.py:92)
    # int64 indices of layer 1 + the greedy part of its selection distances (the
    # fill's are 0 by definition and are written on the host, fps_prune.py:104-105)
    d2h = B * budgets[0] * 8 + B * k1_ * out_s.element_size()

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
               "dtype": prec,
               "schedule": "auto (" + _native.auto_schedule(args.n, B, PREC_CODE[prec]) + ")",
               "stage1_kernel_ms": float(np.mean([k[3] for k in ex_kern if k[1] == args.n])),
               "units_per_step": ex_units,
               "speedup_flash_vs_exhaustive": ex_step / ms_step}
        # the paper's baseline: standard FPS (every point every iteration, K1);
        # ~6.5 s per binary64 step (HBM-streamed), so 1 warm-up + 2 timed steps
        def arm_std(cfg, cache, steps):
            prev = _device.set_schedule("stream")
            try:
                tot, _, kk, _ = timed(cfg, cache, steps, 1, timer=True)
            finally:
                _device.set_schedule(prev)
            return tot / steps, kk

        sd_step, sd_kern = arm_std(cfg_exh, False, 2)
        exh_std = {"value": global_batch / (sd_step / 1e3), "unit": "clouds/s",
                   "ms_per_step": sd_step, "ms_per_cloud": sd_step / B, "dtype": prec,
                   "schedule": "stream (K1, standard exhaustive-update FPS)",
                   "stage1_kernel_ms": float(np.mean([k[3] for k in sd_kern if k[1] == args.n])),
                   "speedup_flash_vs_standard_exhaustive": sd_step / ms_step}
        fs_step, _ = arm_std(cfg_flash, True, 2)
        flash_std = {"value": global_batch / (fs_step / 1e3), "unit": "clouds/s",
                     "ms_per_step": fs_step, "schedule": "stream (K1)", "dtype": prec,
                     "speedup_flash_stream_vs_standard_exhaustive": sd_step / fs_step}

    extras = {}
    if not args.no_extras:
        # the same pipeline in binary32 (secondary: not the reference's arithmetic)
        f32_ms, _, _, _ = timed(cfg_flash, True, max(3, args.steps // 2), 1, precision="f32")
        f32_step = f32_ms / max(3, args.steps // 2)
        extras["f32"] = {"value": global_batch / (f32_step / 1e3), "unit": "clouds/s",
                         "ms_per_step": f32_step,
                         "note": "binary32 arithmetic: indices may differ from the reference "
                                 "(see divergence)"}
        # every divergence of binary32 from the reference's binary64, per cloud
        fl64, _, _ = ffps.hierarchical_sample_batch(x, budgets, cfg_flash, 0, True,
                                                    precision="f64")
        fl32, _, _ = ffps.hierarchical_sample_batch(x, budgets, cfg_flash, 0, True,
                                                    precision="f32")
        div = {"flash_layer1_greedy": divergence(fl64[0].indices[:, :k1_],
                                                 fl32[0].indices[:, :k1_], c1_)}
        if not args.no_exhaustive:
            ex64, _, _ = ffps.hierarchical_sample_batch(x, budgets, cfg_exh, 0, False,
                                                        precision="f64")
            ex32, _, _ = ffps.hierarchical_sample_batch(x, budgets, cfg_exh, 0, False,
                                                        precision="f32")
            div["exhaustive_layer1"] = divergence(ex64[0].indices, ex32[0].indices, args.n)
        div["note"] = ("binary32 run vs the binary64 run (= the reference, bit for bit) on the "
                       "same clouds; the headline is binary64, so its indices have no divergence")
        extras["divergence_f32_vs_f64"] = div
        # matched sampling-quality metric (north star): covering radius of layer 1
        # (metrics.py:45-52) for FlashFPS vs the exhaustive run, every cloud
        if not args.no_exhaustive:
            torch.cuda.synchronize()
            qs, qe = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            qs.record()
            r_fl = ffps.coverage_radius_batch(x, fl64[0].indices, precision="f64")
            qe.record()
            r_ex = ffps.coverage_radius_batch(x, ex64[0].indices, precision="f64")
            torch.cuda.synchronize()
            ratio = (r_fl / r_ex).cpu().numpy()
            extras["quality"] = {
                "metric": "coverage radius of layer 1 (k-center objective, metrics.py:45-52)",
                "flash_mean": float(r_fl.mean()), "exhaustive_mean": float(r_ex.mean()),
                "ratio_median": float(np.median(ratio)), "ratio_max": float(ratio.max()),
                "coverage_kernel_ms_per_batch": qs.elapsed_time(qe), "clouds": B}

    roof = latency_roofline(args, x, budgets, cfg_flash, prec, kern, clocks, B)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = cpu_cores()
        clouds = args.cpu_clouds or 8 * cores   # ~10 s of host work
        dt, cnt = cpu_pipeline_sample(args.n, budgets, args.p, clouds, args.cloud, cores, prec)
        cpu = {"value": cnt / dt, "unit": "clouds/s", "cores": cores, "kind": "port",
               "cpu": cpu_model(),
               "sample": f"{cnt} clouds of N={args.n} {args.cloud}, FPS-Prune p={args.p} + "
                         f"FPS-Cache, binary{64 if prec == 'f64' else 32}, one cloud per host "
                         f"thread, {dt:.1f} s wall"}

    if rank == 0:
        emit({"metric": METRIC, "value": value, "unit": "clouds/s", "n_gpus": world,
              "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
              "ms_per_cloud": ms_step / B, "higher_is_better": True, "scaling": scaling,
              "vs_baseline": None, "dtype": prec, "data": "synthetic",
              "config": {"workload": f"C5 FlashFPS 4-stage N={args.n} (BASELINE configs[4])",
                         "n": args.n, "budgets": list(budgets), "p": args.p, "cache": True,
                         "global_batch": global_batch, "clouds_per_rank": B,
                         "cloud": args.cloud, "input": "fp32 xyz",
                         "arithmetic": "binary64 (FFPS_F32_F64)" if prec == "f64"
                         else "binary32",
                         "parallelism": f"shard-by-cloud x{world}",
                         "l2": "256 MiB flush write between timed steps"},
              "e2e": {"value": e2e_val, "unit": "clouds/s", "ms_per_step": e2e_step,
                      "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
              "gpu_launches": launches, "roofline": roof, "exhaustive": exh,
              "exhaustive_standard": exh_std, "flash_standard_schedule": flash_std,
              **extras,
              "cpu_baseline": cpu, "clocks": clocks,
              "step_ms": [round(v, 4) for v in ms]})


def latency_roofline(args, x, budgets, cfg_flash, prec, kern, clocks, B) -> dict:
    """Roofline of the dominant kernel (K1g, the greedy stage of the step).

    K1g never streams its state from HBM (the bucket table sits in shared
    memory, the bucket SoA in L2), so bytes do not bound it: each greedy
    round is a dependent chain (flag -> re-evaluate -> rank -> DSMEM exchange
    -> chain test).  The bound is the latency of that chain.  Its floor is
    measured live with the same kernel instance on the smallest table that
    keeps the standard ranking path (16 bucket groups per CTA, the same
    clusters per SM): peak = 1 / floor round time.  achieved = the rounds of
    one C5 launch (kernel counters, ffps_run_kernel_stats) / the greedy
    call's CUDA-event time (K0 bucket build included, so frac is
    conservative).  Workloads whose greedy stage AUTO runs on another
    schedule get the HBM-streaming comparison only."""
    import torch
    import paper_2604_17720_b200 as ffps
    from paper_2604_17720_b200 import _device, _native
    c1, k1 = stage_units(args.n, budgets, args.p, True)[0]
    sched = _native.auto_schedule(c1, B, PREC_CODE[prec])
    kms = float(np.mean([k[3] for k in kern if k[1] == c1])) if kern else float("nan")
    units = B * c1 * (k1 - 1)
    if not sched.startswith("grid"):
        gbs = units * BYTES_PER_UNIT[prec] / (kms / 1e3) / 1e9
        pk = peaks()
        return {"bound": "hbm", "achieved": gbs, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": gbs / pk["hbm_gbs"], "traffic": None, "kernel": sched,
                "kernel_ms": kms, "peak_src": pk["src"],
                "note": "greedy stage not on the multi-winner schedule: the standard "
                        "streaming FPS's algorithmic bytes over the greedy call's time"}
    with _device.grid_stats() as gs:
        ffps.hierarchical_sample_batch(x, budgets, cfg_flash, 0, True, precision=prec)
    torch.cuda.synchronize()
    st = [r for r in gs.records if r[1] == c1][0][3].double()
    rounds = float(st[:, 0].mean())
    cycles = float(st[:, 1].mean())
    flagged = float(st[:, 2].mean())
    general = float(st[:, 3].mean()) / max(1, int(sched.split("@")[1]) if "@" in sched else 1)
    # floor: the same kernel instance (KM = 16, CL, bucket size) on the
    # smallest table that keeps the standard ranking path: KM bucket groups
    # of 32 buckets per CTA (fewer groups than KM make every round take the
    # general path), a quarter of the points as iterations (the C5 ratio)
    gp = _native.grid_plan(PREC_CODE[prec], c1, B, sched)
    cl, ppl = gp["cl"], gp["ppl"]
    nf = min(32 * ppl * 32 * 16 * cl, x.shape[1])
    floor_x = x[:, :nf].contiguous()
    prev = _device.set_schedule(sched)
    prev_ppl = os.environ.get("FFPS_GRID_PPL")
    os.environ["FFPS_GRID_PPL"] = str(ppl)  # the headline's bucket size class
    try:
        with _device.grid_stats() as gf:
            ffps.fps_batch(floor_x, nf // 4, precision=prec)
            torch.cuda.synchronize()
    finally:
        _device.set_schedule(prev)
        if prev_ppl is None:
            os.environ.pop("FFPS_GRID_PPL", None)
        else:
            os.environ["FFPS_GRID_PPL"] = prev_ppl
    sf = gf.records[0][3].double()
    f_rounds = float(sf[:, 0].mean())
    f_cycles = float(sf[:, 1].mean())
    f_general = float(sf[:, 3].mean()) / cl
    floor_cpr = f_cycles / max(f_rounds, 1.0)
    cpr = cycles / max(rounds, 1.0)
    sm_mhz = clocks.get("sm_mhz") or peaks()["sm_max_mhz"]
    peak = sm_mhz * 1e6 / floor_cpr                  # rounds/s per cloud at the floor
    achieved = rounds / (kms / 1e3)                  # rounds/s per cloud, event-timed
    return {"bound": "latency", "achieved": achieved, "peak": peak,
            "unit": "greedy rounds/s per cloud", "frac": achieved / peak,
            "traffic": dram_traffic("fps_grid_kernel", prec, f"512, {ppl}, 16, {cl}>"),
            "kernel": "fps_grid_kernel (K1g) " + sched, "kernel_ms": kms,
            "rounds_per_cloud": rounds, "winners_per_round": (k1 - 1) / max(rounds, 1.0),
            "cycles_per_round": cpr, "floor_cycles_per_round": floor_cpr,
            "frac_cycles": floor_cpr / cpr,
            "floor": f"same kernel ({32 * ppl}-point buckets), {nf}-point clouds (16 bucket "
                     f"groups per CTA), "
                     f"{nf // 4} iterations, {B} clouds: {f_rounds:.0f} rounds, "
                     f"{f_general:.0f} through the general ranking path",
            "general_path_rounds_per_cloud": general,
            "buckets_reevaluated_per_round": flagged / max(rounds, 1.0),
            "sm_mhz": sm_mhz,
            "streaming_equivalent": {
                "note": "NOT a roofline: the standard streaming FPS's algorithmic bytes "
                        "(distance_evals x bytes/unit) over the greedy call's time",
                "units_per_launch": units, "bytes_per_unit": BYTES_PER_UNIT[prec],
                "gbs": units * BYTES_PER_UNIT[prec] / (kms / 1e3) / 1e9}}


def dram_traffic(kname: str, prec: str = "f64", inst: str = ""):
    """Per-launch DRAM bytes of a kernel from one `ncu --set full` capture
    (profiles/traffic.json), or None: the exact template instance when given
    (e.g. "512, 2, 16, 2>"), else the instance of the headline's arithmetic
    (float coordinates + binary64 = <double, float, ...>)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            tj = json.load(fh)
        tag = "<double, float," if prec == "f64" else "<float,"
        hit = [v for k_, v in tj.items() if kname in k_ and tag in k_ and inst in k_]
        if not inst:
            hit = hit or [v for k_, v in tj.items() if kname in k_]
        return hit[0]["dram_bytes"] if hit else None
    except (OSError, ValueError, KeyError):
        return None


def free_port() -> int:
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # --gpus is authoritative: one rank per GPU under torch.distributed.run
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
               f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    if world != args.gpus and not SHARE_GPU:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch one rank per GPU")
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
