"""FPS-Prune: candidate pruning + iteration pruning + budget fill
(reference pkg/src/flashfps/fps_prune.py).

Candidate pruning keeps the cloud's first floor((1-p)N) points — a prefix
slice (fps_prune.py:54-65), so on the device it is only the point count the
greedy kernel is launched with; iteration pruning is the kernel's iteration
count floor((1-p)M1) (fps_prune.py:45-47), both computed here in IEEE double
exactly like the reference (e.g. p=0.9, M1=6000 gives 599, not 600).  The
slice fill (K2) and the seeded random fill (K2r, NumPy's
``default_rng(rng_seed).choice(pool, fill_n, replace=False)`` restated on the
device step for step, csrc/fill_random.cu) both run on the GPU.
"""

from __future__ import annotations

import enum
import math
from dataclasses import dataclass

import numpy as np
from numpy.typing import NDArray

from .errors import PruneLeavesNothing
from .fps_core import OrderedSample, SamplerStats
from .geometry import PointCloud

__all__ = ["FillMode", "PruneConfig", "candidate_prune", "fps_prune"]


class FillMode(enum.Enum):
    DETERMINISTIC_SLICE = "slice"
    SEEDED_RANDOM = "random"


def _check_ratio(p: float) -> None:
    if not 0.0 <= p < 1.0:
        raise ValueError(f"pruning ratio must be in [0, 1); got {p}")


@dataclass(frozen=True)
class PruneConfig:
    """Pruning ratio p in [0, 1) and the fill policy (fps_prune.py:30-51)."""

    p: float = 0.0
    fill_mode: FillMode = FillMode.DETERMINISTIC_SLICE
    rng_seed: int = 0

    def __post_init__(self):
        _check_ratio(self.p)

    def kernel_budget(self, m1: int) -> int:
        """Greedy iterations actually run: max(1, floor((1-p) * m1))."""
        return max(1, math.floor((1.0 - self.p) * m1))

    def candidate_count(self, n: int, m1: int) -> int:
        """Candidates admitted: max(kernel budget, floor((1-p) * n))."""
        return max(self.kernel_budget(m1), math.floor((1.0 - self.p) * n))


def candidate_prune(cloud: PointCloud, p: float, min_count: int = 1) -> NDArray[np.int64]:
    """Indices of the candidate prefix [0, c), c = max(min_count, floor((1-p)N))
    clamped to N (fps_prune.py:54-65)."""
    _check_ratio(p)
    c = max(int(min_count), math.floor((1.0 - p) * cloud.n))
    if c < 1:
        raise PruneLeavesNothing("candidate pruning left no candidates")
    return np.arange(min(c, cloud.n), dtype=np.int64)


def fps_prune(cloud: PointCloud, m1: int, cfg: PruneConfig, seed_index: int = 0, *,
              threads: int = 1) -> tuple[OrderedSample, SamplerStats]:
    """``m1`` samples: ``k`` greedy steps over the candidate prefix, then the
    budget fill from the whole cloud (fps_prune.py:68-111)."""
    del threads
    from . import batched  # device pipeline (single code path for 1 or B clouds)

    out, stats = batched.fps_prune_batch(cloud.points, m1, cfg, seed_index)
    return out.to_ordered(0), stats
