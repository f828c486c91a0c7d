"""Sampling-quality metric on the device: the covering radius
(reference pkg/src/flashfps/metrics.py:29-52).

``coverage_radius(sample, cloud)`` is the k-center objective a sample
achieves: max over cloud points of the distance to the nearest sampled point.
The per-pair squared distance is the kernels' own rounded formula, and max /
min are exact, so the value is bit-identical to the reference (which is what
lets the reference's tests check coverage(prefix k) == sqrt(sel_d2[k]) for an
exact farthest-first run, test_metrics.py:55-63).  The sweep runs in K5
(csrc/coverage.cu) over K0 spatial buckets with an exact box-box bound.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _device
from .batched import as_device_batch
from .fps_core import OrderedSample
from .geometry import PointCloud

__all__ = ["coverage_radius", "coverage_d2_batch", "coverage_radius_batch"]


def _as_index_array(sample) -> np.ndarray:
    if isinstance(sample, OrderedSample):
        return sample.indices
    return np.asarray(sample, dtype=np.int64)


def coverage_d2_batch(xyz, indices, *, device=None, precision=None) -> torch.Tensor:
    """Squared covering radius of every cloud: ``xyz`` (B, N, 3), ``indices``
    (B, M) int64 sample indices.  Returns (B,) on the device (max over points
    of min over samples of d2), in the input dtype — or binary64 with
    ``precision="f64"`` on float32 clouds (the reference's arithmetic)."""
    x = as_device_batch(xyz, device)
    idx = indices if isinstance(indices, torch.Tensor) else \
        torch.from_numpy(np.ascontiguousarray(np.asarray(indices, dtype=np.int64)))
    if idx.dim() == 1:
        idx = idx.unsqueeze(0)
    if idx.shape[0] != x.shape[0]:
        raise ValueError(f"indices batch {idx.shape[0]} != clouds {x.shape[0]}")
    if idx.shape[1] < 1:
        raise ValueError("sample must be nonempty")
    idx = idx.to(x.device, torch.int64)
    if idx.stride(-1) != 1:
        idx = idx.contiguous()
    bad = (idx < 0) | (idx >= x.shape[1])
    if bool(bad.any()):
        raise IndexError(f"sample index out of range for a cloud of {x.shape[1]} points")
    from .batched import _out_dtype
    out = torch.empty(x.shape[0], dtype=_out_dtype(x, precision), device=x.device)
    _device.coverage(x, idx, out)
    return out


def coverage_radius_batch(xyz, indices, *, device=None, precision=None) -> torch.Tensor:
    """(B,) float64 covering radii, sqrt taken in binary64 (metrics.py:52)."""
    return torch.sqrt(coverage_d2_batch(xyz, indices, device=device,
                                        precision=precision).to(torch.float64))


def coverage_radius(sample, cloud: PointCloud) -> float:
    """Max over all cloud points of the Euclidean distance to the nearest
    sampled point (metrics.py:45-52); binary64 throughout."""
    idx = _as_index_array(sample)
    if idx.size == 0:
        raise ValueError("sample must be nonempty")
    d2 = coverage_d2_batch(np.ascontiguousarray(cloud.points)[None], idx.reshape(1, -1))
    return math.sqrt(float(d2[0].item()))
