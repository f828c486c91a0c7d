"""B200-native FlashFPS hot path (arxiv 2604.17720).

Drop-in for the sampling entry points of the reference package
(pkg/src/flashfps/__init__.py:21-33): same names, arguments, return types and
exceptions; the greedy loop, the budget fill and the cache-off restricted
re-runs execute in hand-written sm_100a kernels behind the C ABI in
include/flashfps_b200.h.  ``batched`` adds the B-cloud device API used by the
benchmark and by point-network callers.
"""

from . import errors
from .batched import (BatchSample, fps_batch, fps_prune_batch, hierarchical_sample_batch,
                      hierarchical_sample_fused, hierarchical_sample_host, run_restricted_batch)
from .fps_cache import (BYTES_PER_ENTRY, CacheRecord, LayerBudgets, PrefixCheckResult,
                        cache_footprint, hierarchical_sample, hierarchical_sample_detailed,
                        prefix_reuse, read_cache, run_restricted, verify_prefix_property,
                        write_cache, write_cache_text)
from .fps_core import OrderedSample, SamplerStats, fps, run_kernel
from .fps_prune import FillMode, PruneConfig, candidate_prune, fps_prune
from .geometry import Point3, PointCloud, squared_distance, validate_cloud
from .metrics import coverage_d2_batch, coverage_radius, coverage_radius_batch
from .pnn import flashfps_hierarchy, furthest_point_sample

__version__ = "0.1.0"

__all__ = [
    "BYTES_PER_ENTRY", "BatchSample", "CacheRecord", "FillMode", "LayerBudgets",
    "OrderedSample", "Point3", "PointCloud", "PrefixCheckResult", "PruneConfig",
    "SamplerStats", "cache_footprint", "candidate_prune", "coverage_d2_batch",
    "coverage_radius", "coverage_radius_batch", "errors", "fps", "fps_batch",
    "flashfps_hierarchy", "fps_prune", "fps_prune_batch", "furthest_point_sample",
    "hierarchical_sample", "hierarchical_sample_batch",
    "hierarchical_sample_detailed", "hierarchical_sample_fused", "hierarchical_sample_host", "prefix_reuse", "read_cache",
    "run_kernel", "run_restricted", "run_restricted_batch", "squared_distance",
    "validate_cloud", "verify_prefix_property", "write_cache", "write_cache_text",
    "__version__",
]
