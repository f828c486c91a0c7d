"""Multi-GPU: a batch of independent clouds sharded across ranks by cloud.

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch).  A single
cloud's greedy loop has a global argmax per iteration, so clouds are never
split across GPUs; every rank samples its own contiguous slice of the batch
with the single-GPU kernels and there is NO data-path collective.  The only
exchange is the final index gather of layer-1 indices (layers 2..L are prefix
views of layer 1 when the cache is on, so only layer 1 moves): an
``all_gather_into_tensor`` of (B_r, M1) indices per rank, sent as int32.

The reference has no multi-device code; the per-cloud
semantics are those of hierarchical_sample (fps_cache.py:204-240).
"""

from __future__ import annotations

from typing import Sequence

import torch
import torch.distributed as dist

from .fps_prune import PruneConfig

__all__ = ["shard_range", "gather_rows", "hierarchical_sample_sharded"]


def shard_range(batch: int, world: int, rank: int) -> tuple[int, int]:
    """Clouds [lo, hi) owned by ``rank``: contiguous, sizes differ by <= 1,
    lower ranks take the remainder."""
    if world < 1 or not 0 <= rank < world or batch < 0:
        raise ValueError(f"bad shard request batch={batch} world={world} rank={rank}")
    q, r = divmod(batch, world)
    lo = rank * q + min(rank, r)
    return lo, lo + q + (1 if rank < r else 0)


def gather_rows(local: torch.Tensor, batch: int, group=None) -> torch.Tensor:
    """Concatenate every rank's (B_r, ...) rows in rank order into (batch, ...).
    int64 rows are point indices (< 2^31) and travel as int32.

    Shards are padded to the largest shard so the collective is a single
    ``all_gather_into_tensor`` (NCCL); on backends without it (gloo) the list
    form is used.  Works on CPU tensors with gloo (tests) and CUDA tensors
    with NCCL (production)."""
    world = dist.get_world_size(group)
    rows = -(-batch // world) if batch else 0
    # int64 point indices travel as int32 (clouds hold < 2^31 points): half
    # the bytes on the wire; the result is int64 again
    wire = torch.int32 if local.dtype == torch.int64 else local.dtype
    pad = torch.zeros((rows,) + tuple(local.shape[1:]), dtype=wire, device=local.device)
    pad[: local.shape[0]].copy_(local)
    if dist.get_backend(group) == "nccl":
        out = torch.empty((world * rows,) + tuple(local.shape[1:]), dtype=wire,
                          device=local.device)
        dist.all_gather_into_tensor(out, pad, group=group)
        parts = list(out.split(rows)) if rows else [out] * world
    else:  # gloo: host tensors
        host = pad.cpu()
        parts = [torch.empty_like(host) for _ in range(world)]
        dist.all_gather(parts, host, group=group)
        parts = [p.to(local.device) for p in parts]
    keep = []
    for r in range(world):
        lo, hi = shard_range(batch, world, r)
        keep.append(parts[r][: hi - lo])
    return torch.cat(keep, 0).to(local.dtype)


def hierarchical_sample_sharded(xyz_local, budgets: Sequence[int], cfg: PruneConfig,
                                batch: int, seed_index=0, cache_enabled: bool = True,
                                group=None, gather: bool = True):
    """hierarchical_sample_batch on this rank's shard of a ``batch``-cloud job,
    then (``gather``) the layer-1 index gather to every rank.

    Returns (layers, total, gathered): ``layers``/``total`` as
    hierarchical_sample_batch for the local clouds, ``gathered`` the (batch,
    M1) int64 layer-1 indices of the whole job (None when gather=False)."""
    from .batched import hierarchical_sample_batch

    layers, total, _ = hierarchical_sample_batch(xyz_local, budgets, cfg, seed_index,
                                                 cache_enabled)
    gathered = gather_rows(layers[0].indices, batch, group) if gather else None
    return layers, total, gathered
