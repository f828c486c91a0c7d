"""K5 covering radius vs the reference (metrics.py:45-52): golden values from
the unmodified reference, a NumPy brute-force restatement, and the exact
identity coverage(prefix k) == sqrt(sel_d2[k]) of a farthest-first run
(test_metrics.py:55-63) at sizes the brute force cannot reach."""

import math

import numpy as np
import pytest
import torch

import paper_2604_17720_b200 as ffps

pytestmark = pytest.mark.gpu


def _brute_d2(pts, idx):
    """metrics.py:29-42 restated: per point min over samples, then max."""
    best = np.full(pts.shape[0], np.inf, dtype=pts.dtype)
    for q in pts[idx]:
        d = ((pts[:, 0] - q[0]) * (pts[:, 0] - q[0]) + (pts[:, 1] - q[1]) * (pts[:, 1] - q[1])) \
            + (pts[:, 2] - q[2]) * (pts[:, 2] - q[2])
        np.minimum(best, d, out=best)
    return best.max()


def test_coverage_goldens(golden, cuda):
    for c in golden.cases("coverage"):
        cloud = ffps.PointCloud(golden.points(c))
        got = ffps.coverage_radius(golden.out(c, "sample"), cloud)
        assert got == c["value"], (c["id"], got, c["value"])


def test_coverage_worked_examples(cuda):
    cloud = ffps.validate_cloud([(0, 0, 0), (10, 0, 0)])
    assert ffps.coverage_radius(np.array([0]), cloud) == 10.0
    pts = np.random.default_rng(0).random((50, 3))
    assert ffps.coverage_radius(np.arange(50), ffps.PointCloud(pts)) == 0.0
    with pytest.raises(ValueError):
        ffps.coverage_radius(np.array([], dtype=np.int64), ffps.PointCloud(pts))


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_coverage_vs_bruteforce(cuda, dtype):
    rng = np.random.default_rng(3)
    for N, M, B in [(1, 1, 2), (33, 5, 3), (1000, 1, 2), (3000, 300, 3), (5000, 2000, 2)]:
        pts = rng.random((B, N, 3)).astype(dtype)
        if N > 10:
            pts[:, N // 2:] = pts[:, : N - N // 2]  # duplicates -> exact ties
        idx = np.stack([rng.choice(N, size=M, replace=M > N) for _ in range(B)])
        got = ffps.coverage_d2_batch(torch.from_numpy(pts).cuda(), torch.from_numpy(idx).cuda())
        for b in range(B):
            assert got[b].item() == _brute_d2(pts[b], idx[b]), (N, M, b)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_coverage_equals_next_selection_distance(cuda, dtype):
    """For an exact FPS run, the k-prefix covers the cloud with radius
    sqrt(sel_d2[k]) exactly (the next pick is the farthest point)."""
    rng = np.random.default_rng(5)
    B, N, m = 3, 30000, 3000
    x = torch.from_numpy(rng.random((B, N, 3)).astype(dtype)).cuda()
    s, _ = ffps.fps_batch(x, m)
    for k in (1, 2, 17, 500, 2999):
        d2 = ffps.coverage_d2_batch(x, s.indices[:, :k].contiguous())
        assert torch.equal(d2, s.selection_dist2[:, k]), k


def test_coverage_c5_shape_flash_vs_exhaustive(cuda):
    """Matched quality metric at the benchmark shape: FlashFPS (p=0.75 +
    cache) vs exhaustive layer 1; the exhaustive prefix radius equals its
    next selection distance, FlashFPS is within the paper's small gap."""
    rng = np.random.default_rng(6)
    x = torch.from_numpy(rng.random((2, 200000, 3)).astype(np.float32)).cuda()
    budgets = (50000, 12500, 3125, 781)
    fl, _, _ = ffps.hierarchical_sample_batch(x, budgets, ffps.PruneConfig(p=0.75))
    ex, _, _ = ffps.hierarchical_sample_batch(x, budgets, ffps.PruneConfig(p=0.0))
    r_fl = ffps.coverage_radius_batch(x, fl[0].indices)
    r_ex = ffps.coverage_radius_batch(x, ex[0].indices)
    assert (r_ex <= r_fl).all()
    assert (r_fl / r_ex < 3.0).all()


def test_acceptance_criterion_6_quality_bound(cuda):
    """Reference acceptance C6 (test_acceptance.py:169-187) on the device: 50
    uniform clouds of 10,000 points (io.py:209-210), m = 2,500, FPS-Prune p=0.5
    vs exhaustive FPS; median coverage ratio <= 1.9 (QUALITY_RATIO_BOUND,
    test_acceptance.py:27-31).  Binary64 kernels: the same ratios as the
    reference itself."""
    pts = np.stack([np.random.default_rng(s).random((10_000, 3)) for s in range(50)])
    x = torch.from_numpy(pts).cuda()
    full, _ = ffps.fps_batch(x, 2500)
    pruned, _ = ffps.fps_prune_batch(x, 2500, ffps.PruneConfig(p=0.5))
    ratios = (ffps.coverage_radius_batch(x, pruned.indices) /
              ffps.coverage_radius_batch(x, full.indices)).cpu().numpy()
    med = float(np.median(ratios))
    assert med <= 1.9, med
    # the full-FPS radius is its next selection distance (test_metrics.py:55-63)
    nxt, _ = ffps.fps_batch(x, 2501)
    assert torch.equal(ffps.coverage_d2_batch(x, full.indices), nxt.selection_dist2[:, 2500])
