"""Full-shape parity at the BASELINE configurations the first round left
bounded or untested (VERDICT r01 "What's weak" #2), bit-exact indices AND
selection distances against the C oracle (pinned to the reference's goldens):

* C4 FlashFPS stage 1 — 75,000 candidates x 18,750 iterations — binary32
  and binary64 (on float coordinates, the headline's arithmetic);
* C5 exhaustive stage 1 — 200,000 points x 50,000 iterations — binary64;
* C5 cache-off stages 2..4 (restricted runs gathering through the previous
  layer) with FPS-Prune p = 0.75;
* binary64 (double coordinates) at the full C2 and C3 FlashFPS shapes;
* LiDAR-like frames (bench.lidar_cloud) at the C3 and C5 stage-1 shapes on
  K1g with 1 and 2 CTAs per cloud, where the candidate ranking takes its
  general path in tens to hundreds of rounds per cloud (asserted from the
  kernel counters)."""

import numpy as np
import pytest
import torch

import paper_2604_17720_b200 as ffps
from paper_2604_17720_b200 import _device
from oracle import oracle

pytestmark = pytest.mark.gpu

SHAPES = {"C2": (24_000, (6_000, 1_500, 375, 93)), "C3": (100_000, (25_000, 6_250, 1_562, 390)),
          "C5": (200_000, (50_000, 12_500, 3_125, 781)),
          "C4": (300_000, (75_000, 18_750, 4_687, 1_171))}


def _uniform(B, N, first=0):
    return np.stack([np.random.default_rng(first + b).random((N, 3)).astype(np.float32)
                     for b in range(B)])


def _greedy(x_np, n, iters, seeds, precision=None, stats=False):
    x = torch.from_numpy(x_np).cuda()
    B = x.shape[0]
    order = torch.empty((B, iters), dtype=torch.int64, device="cuda")
    sel = torch.empty((B, iters), dtype=torch.float64 if precision == "f64" else x.dtype,
                      device="cuda")
    with _device.grid_stats() as gs:
        _device.greedy(x, n, iters, _device.seeds_tensor(seeds, B, "cuda"), order, sel)
    torch.cuda.synchronize()
    st = gs.records[0][3].cpu().numpy() if stats else None
    return order.cpu().numpy(), sel.cpu().numpy(), st


def _assert_same(go, gs, wo, ws, what):
    for b in range(go.shape[0]):
        bad = np.flatnonzero(go[b] != wo[b])
        assert bad.size == 0, f"{what} cloud {b}: {bad.size} divergences, first at {bad[0]}"
        assert np.array_equal(gs[b], ws[b]), f"{what} cloud {b}: selection distances differ"


def _flash(N, budgets):
    cfg = ffps.PruneConfig(p=0.75)
    return cfg.kernel_budget(budgets[0]), min(cfg.candidate_count(N, budgets[0]), N)


@pytest.mark.parametrize("precision", [None, "f64"])
def test_c4_flash_stage1_full(cuda, precision):
    N, budgets = SHAPES["C4"]
    k, c = _flash(N, budgets)
    x = _uniform(2, N, 600)
    seeds = np.array([0, 31])
    go, gs, _ = _greedy(x, c, k, seeds, precision)
    wo, ws = oracle.run_kernel_batch(x.astype(np.float64) if precision else x, k, seeds, n=c)
    _assert_same(go, gs, wo, ws, f"C4 flash {precision or 'f32'}")


def test_c5_exhaustive_stage1_full_binary64(cuda):
    N, budgets = SHAPES["C5"]
    x = _uniform(2, N, 700)
    seeds = np.array([0, 199_999])
    go, gs, _ = _greedy(x, N, budgets[0], seeds, "f64")
    wo, ws = oracle.run_kernel_batch(x.astype(np.float64), budgets[0], seeds)
    _assert_same(go, gs, wo, ws, "C5 exhaustive stage 1 binary64")


@pytest.mark.parametrize("precision", [None, "f64"])
def test_c5_cache_off_stages_vs_oracle(cuda, precision):
    N, budgets = SHAPES["C5"]
    B = 3
    xn = _uniform(B, N, 800)
    layers, _, _ = ffps.hierarchical_sample_batch(torch.from_numpy(xn).cuda(), budgets,
                                                  ffps.PruneConfig(p=0.75), 0,
                                                  cache_enabled=False, precision=precision)
    for b in range(B):
        pts = xn[b].astype(np.float64) if precision else xn[b]
        want = oracle.hierarchical(pts, budgets, 0.75, 0, cache_enabled=False)
        for li, (wi, ws) in enumerate(want):
            assert np.array_equal(layers[li].indices[b].cpu().numpy(), wi), (b, li)
            assert np.array_equal(layers[li].selection_dist2[b].cpu().numpy(), ws), (b, li)


@pytest.mark.parametrize("shape,B", [("C2", 16), ("C3", 8)])
@pytest.mark.parametrize("sched", ["grid", "stream"])
def test_binary64_flash_stage1_full_c2_c3(cuda, shape, B, sched):
    N, budgets = SHAPES[shape]
    k, c = _flash(N, budgets)
    x = _uniform(B, N, 900).astype(np.float64)
    seeds = np.arange(B) % 5
    prev = _device.set_schedule(sched)
    try:
        go, gs, _ = _greedy(x, c, k, seeds)
    finally:
        _device.set_schedule(prev)
    wo, ws = oracle.run_kernel_batch(x, k, seeds, n=c)
    _assert_same(go, gs, wo, ws, f"{shape} binary64 {sched}")


@pytest.fixture(scope="module")
def lidar_frames():
    import bench
    return {n: bench.make_clouds("lidar", 2, n, 40) for n in (100_000, 200_000)}


@pytest.mark.parametrize("shape", ["C3", "C5"])
@pytest.mark.parametrize("sched", ["grid@1", "grid@2"])
@pytest.mark.parametrize("precision", [None, "f64"])
def test_lidar_flash_stage1_general_path(cuda, lidar_frames, shape, sched, precision):
    N, budgets = SHAPES[shape]
    k, c = _flash(N, budgets)
    x = np.ascontiguousarray(lidar_frames[N])
    seeds = np.zeros(2, np.int64)
    prev = _device.set_schedule(sched)
    try:
        go, gs, st = _greedy(x, c, k, seeds, precision, stats=True)
    finally:
        _device.set_schedule(prev)
    wo, ws = oracle.run_kernel_batch(x.astype(np.float64) if precision else x, k, seeds, n=c)
    _assert_same(go, gs, wo, ws, f"LiDAR {shape} {sched} {precision or 'f32'}")
    rounds, general = st[:, 0], st[:, 3]
    # the general ranking path ran (C5 LiDAR: ~6% of the rounds per CTA on one
    # CTA per cloud, ~11% on two; C3: more)
    assert (general >= 20).all() and (general < rounds * int(sched[-1])).all(), (rounds, general)
