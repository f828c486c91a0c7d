"""Exhaustive farthest point sampling — the reference's L2 kernel layer
(pkg/src/flashfps/fps_core.py) with its body moved to the device.

``run_kernel`` keeps the reference seam (fps_core.py:110-175): same
arguments, same (order, selection_dist2, distance_evals) triple, same
lowest-index tie rule, and — because the binary64 instantiation of the CUDA
kernel performs the same separately rounded operations — bit-identical
output.  ``threads`` is accepted and ignored: it may never change the output
(fps_core.py:115-117), and the device path has no host threads.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
from numpy.typing import NDArray

from . import _device
from .errors import BudgetOutOfRange, SeedOutOfRange
from .geometry import PointCloud

__all__ = ["OrderedSample", "SamplerStats", "run_kernel", "fps"]


@dataclass(frozen=True)
class OrderedSample:
    """Ordered selection over original indices (fps_core.py:29-56).

    ``selection_dist2[0]`` is +inf (the seed), entries from ``fill_boundary``
    on are budget fill with distance 0.  Arrays are owned, contiguous and
    read-only.
    """

    indices: NDArray[np.int64]
    selection_dist2: NDArray[np.float64]
    fill_boundary: int

    def __post_init__(self):
        idx = np.array(self.indices, dtype=np.int64, order="C")   # owned copy
        d2 = np.array(self.selection_dist2, dtype=np.float64, order="C")
        if idx.ndim != 1 or d2.shape != idx.shape:
            raise ValueError("indices and selection_dist2 must be 1-D and equal length")
        if not 0 <= self.fill_boundary <= idx.shape[0]:
            raise ValueError("fill_boundary out of range")
        idx.flags.writeable = False
        d2.flags.writeable = False
        object.__setattr__(self, "indices", idx)
        object.__setattr__(self, "selection_dist2", d2)

    def __len__(self) -> int:
        return int(self.indices.shape[0])


@dataclass
class SamplerStats:
    """Analytic work counters (fps_core.py:59-71): for a greedy run
    distance_evals == candidates * (iterations - 1)."""

    distance_evals: int = 0
    iterations: int = 0
    candidates: int = 0
    cache_bytes: int = 0


def run_kernel(points: NDArray[np.float64], m: int, seed_pos: int, threads: int = 1):
    """Greedy farthest-first selection of ``m`` points over ``points`` (n, 3),
    on the GPU (binary64 unless ``points`` is float32).  Returns
    ``(order int64[m], selection_dist2 float64[m], n*(m-1))`` with positions
    local to ``points`` (fps_core.py:110-175)."""
    del threads  # output never depends on it (fps_core.py:115-117)
    pts = np.asarray(points)
    if pts.dtype not in (np.float32, np.float64):
        pts = pts.astype(np.float64)
    n = int(pts.shape[0])
    if not 0 <= int(seed_pos) < n:
        # the reference indexes dist[seed_pos] (fps_core.py:130): IndexError
        # past the end; a negative position is rejected here as well, before
        # any kernel reads xyz[seed]
        raise IndexError(f"seed position {seed_pos} is out of bounds for {n} points")
    dev = _device.require_cuda()
    xyz = torch.from_numpy(np.array(pts, order="C")).to(dev).unsqueeze(0)
    order = torch.empty((1, m), dtype=torch.int64, device=dev)
    sel = torch.empty((1, m), dtype=xyz.dtype, device=dev)
    seeds = _device.seeds_tensor(seed_pos, 1, dev)
    _device.greedy(xyz, n, m, seeds, order, sel)
    return (order[0].cpu().numpy(), sel[0].to(torch.float64).cpu().numpy(),
            n * (m - 1))


def _check_budget_and_seed(n: int, m: int, seed_index: int) -> None:
    """fps_core.py:178-182."""
    if not 1 <= m <= n:
        raise BudgetOutOfRange(f"m={m} not in [1, {n}]")
    if not 0 <= seed_index < n:
        raise SeedOutOfRange(f"seed index {seed_index} not in [0, {n})")


def fps(cloud: PointCloud, m: int, seed_index: int = 0, *,
        threads: int = 1) -> tuple[OrderedSample, SamplerStats]:
    """Standard FPS of ``m`` points from ``seed_index`` (fps_core.py:185-196)."""
    _check_budget_and_seed(cloud.n, m, seed_index)
    order, sel_d2, evals = run_kernel(cloud.points, m, seed_index, threads)
    return (OrderedSample(order, sel_d2, fill_boundary=m),
            SamplerStats(distance_evals=evals, iterations=m, candidates=cloud.n))
