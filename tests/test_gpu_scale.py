"""Parity at the BASELINE.json shapes (C2-C5), bit-exact against the C
oracle where the oracle finishes in seconds, and through size-independent
properties where it does not:

* every cloud's FlashFPS stage-1 run (candidate prefix, k iterations) at the
  full C5 / C3 / C2 shapes vs the oracle, bit-exact indices + distances;
* the exhaustive 200K-point stage-1 and the 300K-point (spill) kernel for a
  bounded number of iterations vs the oracle;
* properties of whole pipelines: indices unique and in range, selection
  distances non-increasing after the seed, fill = ascending complement, and
  the prefix theorem (cache on == cache off) at the BASELINE budgets
  (holds for p <= 0.75 at m1 = N/4)."""

import numpy as np
import pytest
import torch

import paper_2604_17720_b200 as ffps
from paper_2604_17720_b200 import _device
from oracle import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["stream", "bucket", "grid"])
def schedule(request):
    prev = _device.set_schedule(request.param)
    yield request.param
    _device.set_schedule(prev)

SHAPES = {"C2": (24_000, (6_000, 1_500, 375, 93)), "C3": (100_000, (25_000, 6_250, 1_562, 390)),
          "C5": (200_000, (50_000, 12_500, 3_125, 781)),
          "C4": (300_000, (75_000, 18_750, 4_687, 1_171))}


def _uniform(B, N, first=0):
    return np.stack([np.random.default_rng(first + b).random((N, 3)).astype(np.float32)
                     for b in range(B)])


def _greedy(x_np, n, iters, seeds):
    x = torch.from_numpy(x_np).cuda()
    B = x.shape[0]
    order = torch.empty((B, iters), dtype=torch.int64, device="cuda")
    sel = torch.empty((B, iters), dtype=x.dtype, device="cuda")
    _device.greedy(x, n, iters, _device.seeds_tensor(seeds, B, "cuda"), order, sel)
    return order.cpu().numpy(), sel.cpu().numpy()


def _assert_same(go, gs, wo, ws, what):
    for b in range(go.shape[0]):
        bad = np.flatnonzero(go[b] != wo[b])
        assert bad.size == 0, f"{what} cloud {b}: {bad.size} divergences, first at {bad[0]}"
        assert np.array_equal(gs[b], ws[b]), f"{what} cloud {b}: selection distances differ"


@pytest.mark.parametrize("shape,B", [("C2", 16), ("C3", 8), ("C5", 8)])
def test_flash_stage1_full_shape_bit_exact(shape, B, schedule):
    N, budgets = SHAPES[shape]
    cfg = ffps.PruneConfig(p=0.75)
    k, c = cfg.kernel_budget(budgets[0]), min(cfg.candidate_count(N, budgets[0]), N)
    x = _uniform(B, N, 100)
    seeds = np.arange(B) % 7
    go, gs = _greedy(x, c, k, seeds)
    wo, ws = oracle.run_kernel_batch(x, k, seeds, n=c)
    _assert_same(go, gs, wo, ws, shape)


@pytest.mark.parametrize("N,iters,B", [(200_000, 1_500, 4), (300_000, 600, 2)])
def test_large_clouds_bounded_iterations_bit_exact(N, iters, B, schedule):
    x = _uniform(B, N, 200)
    seeds = np.array([0, N - 1, 12345, 7][:B])
    go, gs = _greedy(x, N, iters, seeds)
    wo, ws = oracle.run_kernel_batch(x, iters, seeds)
    _assert_same(go, gs, wo, ws, f"N={N}")


@pytest.mark.parametrize("shape", ["C2", "C3", "C5"])
def test_pipeline_properties_and_prefix_theorem(shape, schedule):
    N, budgets = SHAPES[shape]
    B = 4
    x = torch.from_numpy(_uniform(B, N, 300)).cuda()
    on, tot_on, _ = ffps.hierarchical_sample_batch(x, budgets, ffps.PruneConfig(p=0.75))
    off, tot_off, _ = ffps.hierarchical_sample_batch(x, budgets, ffps.PruneConfig(p=0.75), 0,
                                                     cache_enabled=False)
    cfg = ffps.PruneConfig(p=0.75)
    k = cfg.kernel_budget(budgets[0])
    for li in range(len(budgets)):
        assert torch.equal(on[li].indices, off[li].indices), f"layer {li + 1}: on != off"
    l1 = on[0].indices.cpu().numpy()
    d1 = on[0].selection_dist2.cpu().numpy()
    for b in range(B):
        assert np.unique(l1[b]).size == budgets[0] and l1[b].min() >= 0 and l1[b].max() < N
        assert np.all(np.diff(d1[b][1:k]) <= 0), "greedy distances must be non-increasing"
        assert np.isinf(d1[b][0]) and np.all(d1[b][k:] == 0)
        fill = l1[b][k:]
        assert np.all(np.diff(fill) > 0), "slice fill is ascending"
        want = oracle.fill_slice(l1[b][:k], N, budgets[0] - k)
        assert np.array_equal(fill, want)
    assert tot_on.distance_evals == min(cfg.candidate_count(N, budgets[0]), N) * (k - 1)
    assert tot_on.cache_bytes == 36 * budgets[0]


def test_exhaustive_four_stage_restricted_stages_bit_exact(schedule):
    """Cache-off stages 2..4 at the C2 shape (the restricted runs gather
    through the previous layer inside the kernel), vs the oracle."""
    N, budgets = SHAPES["C2"]
    B = 4
    xn = _uniform(B, N, 400)
    layers, _, _ = ffps.hierarchical_sample_batch(torch.from_numpy(xn).cuda(), budgets,
                                                  ffps.PruneConfig(p=0.0), 0,
                                                  cache_enabled=False)
    for b in range(B):
        want = oracle.hierarchical(xn[b], budgets, 0.0, 0, cache_enabled=False)
        for li, (wi, ws) in enumerate(want):
            assert np.array_equal(layers[li].indices[b].cpu().numpy(), wi), (b, li)
            assert np.array_equal(layers[li].selection_dist2[b].cpu().numpy(), ws), (b, li)


@pytest.mark.parametrize("chunks", [1, 3])
def test_host_pipeline_matches_device_pipeline(chunks):
    """hierarchical_sample_host (prefix-only copy, chunked streams) returns
    exactly the device pipeline's layers."""
    N, budgets = SHAPES["C2"]
    xn = _uniform(7, N, 500)
    cfg = ffps.PruneConfig(p=0.75)
    want, tot_w, _ = ffps.hierarchical_sample_batch(torch.from_numpy(xn).cuda(), budgets, cfg)
    got, tot_g = ffps.hierarchical_sample_host(torch.from_numpy(xn).pin_memory(), budgets, cfg,
                                               chunks=chunks)
    for (gi, gs, fb), w in zip(got, want):
        assert torch.equal(gi, w.indices.cpu()) and torch.equal(gs, w.selection_dist2.cpu())
        assert fb == w.fill_boundary
    assert tot_g.distance_evals == tot_w.distance_evals and tot_g.cache_bytes == tot_w.cache_bytes


@pytest.mark.parametrize("sched", ["stream", "grid"])
def test_flash_stage1_full_shape_fp64_bit_exact(sched):
    """binary64 — the reference's own precision: the C5 FlashFPS
    stage-1 run (50,000 candidates, 12,500 iterations) equals the oracle's
    binary64 restatement of run_kernel bit for bit."""
    prev = _device.set_schedule(sched)
    try:
        N, budgets = SHAPES["C5"]
        cfg = ffps.PruneConfig(p=0.75)
        k, c = cfg.kernel_budget(budgets[0]), min(cfg.candidate_count(N, budgets[0]), N)
        x = _uniform(2, N, 300).astype(np.float64)
        seeds = np.array([0, 4242])
        go, gs = _greedy(x, c, k, seeds)
        wo, ws = oracle.run_kernel_batch(x, k, seeds, n=c)
        _assert_same(go, gs, wo, ws, f"C5 fp64 {sched}")
    finally:
        _device.set_schedule(prev)
