"""Edge cases of the public API on the device: argument checks that must
precede any kernel (the reference raises IndexError from NumPy indexing,
fps_cache.py:195, fps_core.py:130) and the AUTO schedule's fallback for
clouds whose bucket table exceeds shared memory."""

import numpy as np
import pytest
import torch

import paper_2604_17720_b200 as ffps
from oracle import oracle

pytestmark = pytest.mark.gpu


def test_restricted_index_map_is_checked(cuda):
    rng = np.random.default_rng(1)
    x = torch.from_numpy(rng.random((2, 500, 3))).cuda()
    good = np.stack([rng.permutation(500)[:100] for _ in range(2)])
    with pytest.raises(ValueError):      # batch mismatch
        ffps.run_restricted_batch(x, good[:1].repeat(3, 0), 10)
    for bad in (500, -501):
        m = good.copy()
        m[1, 7] = bad
        with pytest.raises(IndexError):
            ffps.run_restricted_batch(x, m, 10)
    # negative entries count from the end, as points[index_map] does
    neg = good.copy()
    neg[:, ::3] -= 500
    a, _ = ffps.run_restricted_batch(x, neg, 40)
    b, _ = ffps.run_restricted_batch(x, good, 40)
    assert torch.equal(a.indices, b.indices)
    assert torch.equal(a.selection_dist2, b.selection_dist2)
    # one 1-D map shared by every cloud
    c, _ = ffps.run_restricted_batch(x, good[0], 40)
    for i in range(2):
        wo, ws, _ = oracle.run_kernel(x[i].cpu().numpy(), 40, 0, index_map=good[0])
        assert np.array_equal(c.indices[i].cpu().numpy(), wo)
        assert np.array_equal(c.selection_dist2[i].cpu().numpy(), ws)


def test_run_kernel_seed_position_is_checked(cuda):
    pts = np.random.default_rng(2).random((50, 3))
    for seed in (50, -1):
        with pytest.raises(IndexError):
            ffps.run_kernel(pts, 5, seed)


@pytest.mark.parametrize("precision", ["f64", None])
def test_auto_falls_back_when_the_bucket_table_exceeds_shared_memory(cuda, precision):
    """1.5M points in binary64: no K1g configuration fits shared memory, AUTO
    runs the streaming kernel with HBM spill instead of failing."""
    rng = np.random.default_rng(3)
    pts = rng.random((1, 1_500_000, 3)).astype(np.float32 if precision else np.float64)
    s, _ = ffps.fps_batch(torch.from_numpy(pts).cuda(), 40, precision=precision)
    wo, ws = oracle.run_kernel_batch(pts.astype(np.float64), 40, np.zeros(1, np.int64))
    assert np.array_equal(s.indices.cpu().numpy(), wo)
    assert np.array_equal(s.selection_dist2.cpu().numpy(), ws)
