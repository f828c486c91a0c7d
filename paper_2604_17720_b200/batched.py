"""Batched device API: the whole hot path for B clouds per call.

Every function takes a batch of clouds ``xyz`` of shape (B, N, 3) — a CUDA
tensor (float32 or float64), or a host array/tensor that is copied to the
current device — and keeps all intermediate results on the device:

* ``fps_batch``               fps            (fps_core.py:185-196)
* ``fps_prune_batch``         fps_prune      (fps_prune.py:68-111)
* ``run_restricted_batch``    run_restricted (fps_cache.py:189-201)
* ``hierarchical_sample_batch`` hierarchical_sample_detailed (fps_cache.py:204-240)
* ``hierarchical_sample_host``  the same from/to host buffers (the end-to-end
  call the benchmark times: H2D copy, kernels, D2H copy)

Validation raises the reference's exceptions before any device work; the
stats are the reference's analytic counters for ONE cloud (every cloud of a
batch has the same shape, so the same counters).  The single-cloud API in
fps_core / fps_prune / fps_cache is this module with B = 1.

``precision``: the arithmetic of the run.  None follows the coordinates
(float32 -> binary32, float64 -> binary64).  "f64" on float32 coordinates
runs the reference's binary64 arithmetic on them (PointCloud upcasts a float32
cloud exactly, geometry.py:52-54) while the coordinates stay float32 in HBM,
L2 and shared memory; selection distances come back as float64 and every
result equals the float64 run on the upcast cloud, bit for bit.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import _device
from .errors import (BudgetExceedsCloud, BudgetOutOfRange, SeedNotInCandidates,
                     SeedOutOfRange)
from .fps_core import OrderedSample, SamplerStats
from .fps_prune import FillMode, PruneConfig

__all__ = ["BatchSample", "as_device_batch", "fps_batch", "fps_prune_batch",
           "run_restricted_batch", "hierarchical_sample_batch", "hierarchical_sample_fused",
           "hierarchical_sample_host", "cache_footprint_bytes"]

BYTES_PER_ENTRY = 36  # fps_cache.py:28 (uint32 index + 3 x f64 + f64 dist2)


@dataclass
class BatchSample:
    """Ordered samples of B clouds: ``indices`` (B, M) int64 original
    indices and ``selection_dist2`` (B, M) in the input dtype, on the device.
    Cache-on deeper layers are views (prefix slices) of layer 1."""

    indices: torch.Tensor
    selection_dist2: torch.Tensor
    fill_boundary: int

    def __len__(self) -> int:
        return int(self.indices.shape[1])

    def to_ordered(self, b: int) -> OrderedSample:
        return OrderedSample(self.indices[b].cpu().numpy(),
                             self.selection_dist2[b].to(torch.float64).cpu().numpy(),
                             fill_boundary=self.fill_boundary)


def cache_footprint_bytes(m1: int) -> int:
    if m1 < 1:
        raise BudgetOutOfRange(f"cache size must be >= 1; got {m1}")
    return int(m1) * BYTES_PER_ENTRY


def as_device_batch(xyz, device=None) -> torch.Tensor:
    """(B, N, 3) contiguous CUDA float32/float64 tensor (a (N, 3) input is a
    batch of one).  Host inputs are copied; float64 stays float64."""
    dev = _device.require_cuda(device)
    if isinstance(xyz, torch.Tensor):
        t = xyz
    else:
        a = np.asarray(xyz)
        if a.dtype not in (np.float32, np.float64):
            a = a.astype(np.float64)
        t = torch.from_numpy(a if a.flags.writeable and a.flags.c_contiguous
                             else np.array(a, order="C"))
    if t.dtype not in (torch.float32, torch.float64):
        t = t.to(torch.float64)
    if t.dim() == 2:
        t = t.unsqueeze(0)
    if t.dim() != 3 or t.shape[2] != 3:
        raise ValueError(f"points must have shape (B, N, 3); got {tuple(t.shape)}")
    if t.shape[1] < 1:
        raise BudgetOutOfRange("cloud is empty")
    if t.device != dev:
        t = t.to(dev, non_blocking=t.is_pinned())
    return t.contiguous()


def _out_dtype(x: torch.Tensor, precision) -> torch.dtype:
    """dtype of the selection distances (= the arithmetic) for coordinates x."""
    if precision is None:
        return x.dtype
    want = {"f64": torch.float64, "float64": torch.float64, torch.float64: torch.float64,
            "f32": torch.float32, "float32": torch.float32, torch.float32: torch.float32}.get(
                precision)
    if want is None:
        raise ValueError(f"precision must be None, 'f32' or 'f64'; got {precision!r}")
    if want == torch.float32 and x.dtype == torch.float64:
        raise ValueError("binary32 arithmetic on float64 coordinates would round the cloud")
    return want


def _shape(xyz) -> tuple[int, int]:
    """(B, N) of a (B, N, 3) or (N, 3) input without touching the device, so
    argument errors surface before any CUDA requirement."""
    shp = tuple(xyz.shape) if hasattr(xyz, "shape") else np.shape(xyz)
    if len(shp) == 2:
        shp = (1,) + shp
    if len(shp) != 3 or shp[2] != 3:
        raise ValueError(f"points must have shape (B, N, 3); got {shp}")
    return int(shp[0]), int(shp[1])


def _seed_array(seed_index, B: int) -> np.ndarray:
    return np.broadcast_to(np.asarray(seed_index, dtype=np.int64), (B,))


def _check_seeds(seeds: np.ndarray, n: int) -> None:
    bad = (seeds < 0) | (seeds >= n)
    if bad.any():
        s = int(seeds[np.flatnonzero(bad)[0]])
        raise SeedOutOfRange(f"seed index {s} not in [0, {n})")


def fps_batch(xyz, m: int, seed_index=0, *, device=None,
              precision=None) -> tuple[BatchSample, SamplerStats]:
    """Exhaustive FPS of every cloud (fps_core.py:185-196)."""
    B, n = _shape(xyz)
    if not 1 <= m <= n:
        raise BudgetOutOfRange(f"m={m} not in [1, {n}]")
    seeds = _seed_array(seed_index, B)
    _check_seeds(seeds, n)
    x = as_device_batch(xyz, device)
    order = torch.empty((B, m), dtype=torch.int64, device=x.device)
    sel = torch.empty((B, m), dtype=_out_dtype(x, precision), device=x.device)
    _device.greedy(x, n, m, _device.seeds_tensor(seeds, B, x.device), order, sel)
    return (BatchSample(order, sel, m),
            SamplerStats(distance_evals=n * (m - 1), iterations=m, candidates=n))


def _fps_prune_checks(B: int, n: int, m1: int, cfg: PruneConfig, seeds: np.ndarray):
    """fps_prune.py:78-88 — returns (k, c)."""
    if not 1 <= m1 <= n:
        raise BudgetOutOfRange(f"m1={m1} not in [1, {n}]")
    _check_seeds(seeds, n)
    k = cfg.kernel_budget(m1)
    c = min(cfg.candidate_count(n, m1), n)   # candidate_prune(...).shape[0]
    if (seeds >= c).any():
        s = int(seeds[np.flatnonzero(seeds >= c)[0]])
        raise SeedNotInCandidates(
            f"seed index {s} was pruned (candidate count {c}); "
            "re-index the cloud or lower p")
    return k, c


def _fps_prune_device(x: torch.Tensor, m1: int, cfg: PruneConfig, seeds: np.ndarray,
                      n: int | None = None, precision=None):
    """``x`` holds at least the candidate prefix of every cloud; ``n`` is the
    logical cloud size (x.shape[1] when the whole cloud is on the device)."""
    B = x.shape[0]
    n = x.shape[1] if n is None else n
    k, c = _fps_prune_checks(B, n, m1, cfg, seeds)
    assert x.shape[1] >= c
    order = torch.empty((B, m1), dtype=torch.int64, device=x.device)
    sel = torch.empty((B, m1), dtype=_out_dtype(x, precision), device=x.device)
    # candidates are the store prefix [0, c): kernel positions == original indices
    _device.greedy(x, c, k, _device.seeds_tensor(seeds, B, x.device), order, sel)
    if m1 > k:
        if cfg.fill_mode is FillMode.DETERMINISTIC_SLICE:
            _device.fill_slice(order, sel, k, m1)
        else:
            _device.fill_random(order, sel, n, k, m1, cfg.rng_seed)
    return (BatchSample(order, sel, k),
            SamplerStats(distance_evals=c * (k - 1), iterations=k, candidates=c))


def fps_prune_batch(xyz, m1: int, cfg: PruneConfig, seed_index=0, *,
                    device=None, precision=None) -> tuple[BatchSample, SamplerStats]:
    """FPS-Prune for every cloud (fps_prune.py:68-111)."""
    B, n = _shape(xyz)
    seeds = _seed_array(seed_index, B)
    _fps_prune_checks(B, n, m1, cfg, seeds)
    return _fps_prune_device(as_device_batch(xyz, device), m1, cfg, seeds,
                             precision=precision)


def run_restricted_batch(xyz, index_map, m: int, seed_pos=0, *,
                         device=None, precision=None) -> tuple[BatchSample, SamplerStats]:
    """Exact FPS over xyz[b][index_map[b]] in map order, reported in original
    indices (fps_cache.py:189-201); the gather happens inside the kernel.

    ``index_map`` is (B, M) or (M,) (the same map for every cloud).  As the
    reference's ``points[index_map]`` (fps_cache.py:195): negative entries
    count from the end of the cloud, entries outside [-N, N) raise IndexError —
    checked before any kernel reads the cloud."""
    B, N = _shape(xyz)
    shp = tuple(np.shape(index_map))
    if len(shp) not in (1, 2) or (len(shp) == 2 and shp[0] != B):
        raise ValueError(f"index_map must have shape ({B}, M) or (M,); got {shp}")
    nm = int(shp[-1])
    if not 1 <= m <= nm:
        raise BudgetOutOfRange(f"m={m} not in [1, {nm}]")
    seeds = _seed_array(seed_pos, B)
    _check_seeds(seeds, nm)
    x = as_device_batch(xyz, device)
    imap = index_map if isinstance(index_map, torch.Tensor) else \
        torch.from_numpy(np.ascontiguousarray(np.asarray(index_map, dtype=np.int64)))
    if imap.dtype.is_floating_point or imap.dtype == torch.bool:
        raise IndexError("index_map must hold integers")
    imap = imap.to(x.device, torch.int64)
    if imap.dim() == 1:
        imap = imap.unsqueeze(0).expand(B, nm)
    lo, hi = torch.aminmax(imap)
    if int(lo) < -N or int(hi) >= N:
        bad = int(lo) if int(lo) < -N else int(hi)
        raise IndexError(f"index {bad} is out of bounds for a cloud of {N} points")
    if int(lo) < 0:
        imap = torch.where(imap < 0, imap + N, imap)
    return _run_restricted_device(x, imap.contiguous(), m, seeds, precision)


def _run_restricted_device(x: torch.Tensor, imap: torch.Tensor, m: int, seeds: np.ndarray,
                           precision=None) -> tuple[BatchSample, SamplerStats]:
    """run_restricted on a validated (B, M) int64 device map in [0, N)."""
    B, nm = x.shape[0], imap.shape[1]
    order = torch.empty((B, m), dtype=torch.int64, device=x.device)
    sel = torch.empty((B, m), dtype=_out_dtype(x, precision), device=x.device)
    _device.greedy(x, nm, m, _device.seeds_tensor(seeds, B, x.device), order, sel,
                   index_map=imap)
    return (BatchSample(order, sel, m),
            SamplerStats(distance_evals=nm * (m - 1), iterations=m, candidates=nm))


def _budgets(budgets) -> tuple[int, ...]:
    from .fps_cache import LayerBudgets
    if not isinstance(budgets, LayerBudgets):
        budgets = LayerBudgets(tuple(budgets))
    return budgets.budgets


def hierarchical_sample_batch(xyz, budgets: Sequence[int], cfg: PruneConfig, seed_index=0,
                              cache_enabled: bool = True, *, device=None, precision=None):
    """Every layer of the budget pyramid for every cloud
    (fps_cache.py:204-240).  Returns (layers, total, per_layer): with the cache
    on, layers 2..L are prefix views of layer 1 (zero distance evaluations);
    with it off, each layer re-runs exact FPS on the previous layer's points,
    seeded at position 0 (the reference's verification / exhaustive path)."""
    b = _budgets(budgets)
    B, n = _shape(xyz)
    if b[0] > n:
        raise BudgetExceedsCloud(f"M1={b[0]} exceeds cloud size {n}")
    seeds = _seed_array(seed_index, B)
    _fps_prune_checks(B, n, b[0], cfg, seeds)
    x = as_device_batch(xyz, device)
    layer1, stats1 = _fps_prune_device(x, b[0], cfg, seeds, precision=precision)
    layers, per_layer = [layer1], [stats1]
    if cache_enabled:
        stats1.cache_bytes = cache_footprint_bytes(b[0])
        for m in b[1:]:
            layers.append(BatchSample(layer1.indices[:, :m], layer1.selection_dist2[:, :m],
                                      min(layer1.fill_boundary, m)))
            per_layer.append(SamplerStats())
    else:
        zero = np.zeros(B, dtype=np.int64)
        for m in b[1:]:  # the previous layer's indices are valid by construction
            s, st = _run_restricted_device(x, layers[-1].indices, m, zero, precision)
            layers.append(s)
            per_layer.append(st)
    total = SamplerStats(
        distance_evals=sum(s.distance_evals for s in per_layer),
        iterations=sum(s.iterations for s in per_layer),
        candidates=sum(s.candidates for s in per_layer),
        cache_bytes=sum(s.cache_bytes for s in per_layer))
    return layers, total, per_layer


def hierarchical_sample_fused(xyz, budgets: Sequence[int], cfg: PruneConfig, seed_index=0,
                              cache_enabled: bool = True, *, device=None, precision=None):
    """hierarchical_sample_batch through ONE C-ABI call
    (ffps_hierarchical_sample): the greedy layer 1, its fill and, with the
    cache off, every restricted deeper layer are issued by the library on
    the current stream without returning to Python.  Same results and return
    value as hierarchical_sample_batch."""
    from . import _native
    b = _budgets(budgets)
    B, n = _shape(xyz)
    if b[0] > n:
        raise BudgetExceedsCloud(f"M1={b[0]} exceeds cloud size {n}")
    seeds = _seed_array(seed_index, B)
    k, c = _fps_prune_checks(B, n, b[0], cfg, seeds)
    x = as_device_batch(xyz, device)
    od = _out_dtype(x, precision)
    orders = [torch.empty((B, m), dtype=torch.int64, device=x.device)
              for m in (b if not cache_enabled else b[:1])]
    sels = [torch.empty((B, m), dtype=od, device=x.device)
            for m in (b if not cache_enabled else b[:1])]
    pcg = None
    if cfg.fill_mode is not FillMode.DETERMINISTIC_SLICE and b[0] > k:
        st = np.random.PCG64(cfg.rng_seed).state["state"]
        pcg = (int(st["state"]), int(st["inc"]))
    sel_code = torch.empty(0, dtype=od)
    with torch.cuda.device(x.device):
        _device._count(_native.hierarchical_sample(
            _device.dtype_code(x, sel_code), x.data_ptr(), B, x.shape[1], n, list(b), k, c,
            0 if pcg is None else 1, pcg, cache_enabled,
            _device.seeds_tensor(seeds, B, x.device).data_ptr(),
            [t.data_ptr() for t in orders] + [None] * (len(b) - len(orders)),
            [t.data_ptr() for t in sels] + [None] * (len(b) - len(sels)),
            torch.cuda.current_stream(x.device).cuda_stream))
    layer1 = BatchSample(orders[0], sels[0], k)
    stats1 = SamplerStats(distance_evals=c * (k - 1), iterations=k, candidates=c)
    layers, per_layer = [layer1], [stats1]
    if cache_enabled:
        stats1.cache_bytes = cache_footprint_bytes(b[0])
        for m in b[1:]:
            layers.append(BatchSample(layer1.indices[:, :m], layer1.selection_dist2[:, :m],
                                      min(k, m)))
            per_layer.append(SamplerStats())
    else:
        for li, m in enumerate(b[1:], 1):
            layers.append(BatchSample(orders[li], sels[li], m))
            per_layer.append(SamplerStats(distance_evals=b[li - 1] * (m - 1), iterations=m,
                                          candidates=b[li - 1]))
    total = SamplerStats(
        distance_evals=sum(s.distance_evals for s in per_layer),
        iterations=sum(s.iterations for s in per_layer),
        candidates=sum(s.candidates for s in per_layer),
        cache_bytes=sum(s.cache_bytes for s in per_layer))
    return layers, total, per_layer


_STREAMS: dict = {}


def _side_streams(dev: torch.device, n: int) -> list:
    """Cached side streams of ``dev`` for the chunked host pipeline."""
    have = _STREAMS.setdefault(dev.index, [])
    while len(have) < n:
        have.append(torch.cuda.Stream(dev))
    return have[:n]


def hierarchical_sample_host(points, budgets: Sequence[int], cfg: PruneConfig, seed_index=0,
                             cache_enabled: bool = True, *, device=None, out=None,
                             chunks: int = 4, precision=None):
    """End-to-end call from HOST buffers: ``points`` (B, N, 3) float32/float64
    numpy array or (preferably pinned) CPU tensor.  Copies the clouds to the
    device, runs the pipeline, copies every layer's indices and selection
    distances back and synchronises.  Returns (layers, total) with layers a
    list of (indices int64 (B, M_l), selection_dist2 (B, M_l), fill_boundary)
    host tensors; ``out`` may pass preallocated pinned (indices, sel) tensors
    of shape (B, M1) for layer 1 (deeper cache-on layers are views of it).

    With the cache on only the candidate prefix points[:, :c] is ever read
    (the greedy run is on points[:c], fps_prune.py:92; the fill and the cached
    layers are index-only), so only that prefix is copied.  The batch is split
    into ``chunks`` groups of clouds on separate streams so the copies of one
    group overlap the kernels of the others."""
    dev = _device.require_cuda(device)
    b = _budgets(budgets)
    B, N = _shape(points)
    if b[0] > N:
        raise BudgetExceedsCloud(f"M1={b[0]} exceeds cloud size {N}")
    seeds = _seed_array(seed_index, B)
    k, c = _fps_prune_checks(B, N, b[0], cfg, seeds)
    host = points if isinstance(points, torch.Tensor) else torch.from_numpy(
        np.ascontiguousarray(points))
    if not cache_enabled:
        x = host.to(dev, non_blocking=host.is_pinned())
        layers, total, _ = hierarchical_sample_batch(x, b, cfg, seed_index, False,
                                                     precision=precision)
        res = [(s.indices.to("cpu", non_blocking=True),
                s.selection_dist2.to("cpu", non_blocking=True), s.fill_boundary)
               for s in layers]
        torch.cuda.current_stream(dev).synchronize()
        return res, total
    pinned = host.is_pinned()
    if out is not None:
        hi, hs = out
    else:
        hi = torch.empty((B, b[0]), dtype=torch.int64, pin_memory=pinned)
        hs = torch.empty((B, b[0]), dtype=_out_dtype(host, precision), pin_memory=pinned)
    nch = max(1, min(chunks, B))
    bounds = [B * i // nch for i in range(nch + 1)]
    # one schedule for the whole batch (AUTO would otherwise decide per chunk)
    from . import _native
    sched = _device.current_schedule()
    if sched == "auto":
        sched = _native.auto_schedule(c, B, _device.dtype_code(
            host, torch.empty(0, dtype=_out_dtype(host, precision))))
    prev = _device.set_schedule(sched)
    try:
        main = torch.cuda.current_stream(dev)
        streams = [main] if nch == 1 else _side_streams(dev, nch)
        stats1 = None
        for i, st in enumerate(streams):
            lo, up = bounds[i], bounds[i + 1]
            if up <= lo:
                continue
            if st is not main:
                st.wait_stream(main)
            with torch.cuda.stream(st):
                if host.is_contiguous() and host.dtype in (torch.float32, torch.float64):
                    # one pitched copy of the candidate prefixes (no host staging)
                    x = torch.empty((up - lo, c, 3), dtype=host.dtype, device=dev)
                    _native.h2d_prefix(x.data_ptr(), host[lo:up].data_ptr(), up - lo, c, N,
                                       _device.dtype_code(x), st.cuda_stream)
                    if not pinned:
                        st.synchronize()  # pageable source: the copy is staged, keep it alive
                else:
                    x = host[lo:up, :c].to(dev, non_blocking=pinned)
                l1, stats1 = _fps_prune_device(x, b[0], cfg, seeds[lo:up], n=N,
                                               precision=precision)
                hi[lo:up].copy_(l1.indices, non_blocking=pinned)
                # the fill's selection distances are 0 by definition
                # (fps_prune.py:104-105): only the greedy part crosses PCIe
                if pinned:   # one pitched copy into the strided pinned rows
                    sd = l1.selection_dist2
                    _native.d2h_prefix(hs[lo:up].data_ptr(), hs.stride(0), sd.data_ptr(),
                                       sd.stride(0), up - lo, k, sd.element_size(),
                                       st.cuda_stream)
                else:
                    hs[lo:up, :k].copy_(l1.selection_dist2[:, :k])
        for st in streams:
            if st is not main:
                main.wait_stream(st)
    finally:
        _device.set_schedule(prev)
    if b[0] > k:
        hs[:, k:].zero_()   # on the host while the device works
    main.synchronize()
    stats1.cache_bytes = cache_footprint_bytes(b[0])
    res = [(hi[:, :m], hs[:, :m], min(k, m)) for m in b]
    total = SamplerStats(distance_evals=stats1.distance_evals, iterations=stats1.iterations,
                         candidates=stats1.candidates, cache_bytes=stats1.cache_bytes)
    return res, total
