"""Point-network call-site adapter.

The paper integrates FlashFPS into PointNeXt / PointVector through
OpenPoints' sampling op: ``furthest_point_sample(xyz,
npoint)`` on a (B, N, 3) float32 CUDA tensor, returning (B, npoint) int32
indices on the device, and the set-abstraction stages call it once per stage
on the previous stage's points.  This module keeps that call shape on top of
the batched device API:

* ``furthest_point_sample(xyz, npoint)`` — one stage, seed index 0, the
  reference's farthest-first semantics (fps_core.py:110-175: lowest-index
  tie-break, separately rounded d2);
* ``flashfps_hierarchy(xyz, budgets, p)`` — the whole FlashFPS pyramid
  (FPS-Prune + FPS-Cache, fps_cache.py:204-240) as per-stage device index
  tensors (views of one (B, M1) buffer when the cache is on).

Neither synchronises the host: the kernels are stream-ordered on torch's
current stream and the results stay on the device for the grouping op that
follows.  ``precision="f64"`` runs the reference's binary64 arithmetic on the
float32 coordinates (bit-identical to the reference on the upcast cloud);
the default is binary32, the arithmetic of the CUDA op it replaces.
"""

from __future__ import annotations

from typing import Sequence

import torch

from .batched import fps_batch, hierarchical_sample_batch
from .fps_prune import PruneConfig

__all__ = ["furthest_point_sample", "flashfps_hierarchy"]


def _check_xyz(xyz: torch.Tensor) -> None:
    if not isinstance(xyz, torch.Tensor) or not xyz.is_cuda:
        raise TypeError("xyz must be a CUDA tensor of shape (B, N, 3)")
    if xyz.dim() != 3 or xyz.shape[2] != 3:
        raise ValueError(f"xyz must have shape (B, N, 3); got {tuple(xyz.shape)}")


def furthest_point_sample(xyz: torch.Tensor, npoint: int, *,
                          precision=None) -> torch.Tensor:
    """(B, npoint) int32 CUDA indices of farthest-first samples of every
    cloud, starting at point 0 (the OpenPoints op's signature)."""
    _check_xyz(xyz)
    x = xyz if xyz.is_contiguous() else xyz.contiguous()
    s, _ = fps_batch(x, int(npoint), 0, device=x.device, precision=precision)
    return s.indices.to(torch.int32)


def flashfps_hierarchy(xyz: torch.Tensor, budgets: Sequence[int], p: float = 0.75, *,
                       cache: bool = True, precision=None,
                       cfg: PruneConfig | None = None) -> list[torch.Tensor]:
    """FlashFPS sampling for every set-abstraction stage at once: returns one
    (B, M_l) int64 CUDA index tensor per budget (indices into the original
    cloud).  With ``cache`` the deeper stages are prefix views of stage 1
    (FPS-Cache, fps_cache.py:141-148) — zero extra kernels."""
    _check_xyz(xyz)
    x = xyz if xyz.is_contiguous() else xyz.contiguous()
    layers, _, _ = hierarchical_sample_batch(x, budgets, cfg or PruneConfig(p=p), 0, cache,
                                             device=x.device, precision=precision)
    return [s.indices for s in layers]
