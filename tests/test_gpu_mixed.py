"""FFPS_F32_F64 — float32 coordinates, the reference's binary64 arithmetic.

The reference upcasts every cloud to float64 (geometry.py:52-54) and computes
in binary64 (fps_core.py:74-83).  For a float32 cloud the upcast is exact, so
the build may keep the coordinates float32 in HBM, L2 and shared memory and
still reproduce the reference bit for bit, as long as every rounded operation
runs in binary64.  Bar: indices AND selection distances equal the binary64
oracle (pinned to the reference's goldens, tests/test_oracle.py) on the
upcast cloud, under every schedule (K1g natively; the others on a widened
copy of the cloud)."""

import numpy as np
import pytest
import torch

import paper_2604_17720_b200 as ffps
from oracle import oracle
from test_gpu_parity import SCHEDULES, _cloud, _Sched

pytestmark = pytest.mark.gpu


@pytest.fixture(params=SCHEDULES)
def schedule(request):
    with _Sched(request.param):
        yield request.param


def _check_mixed(xyz32, m, seeds, n=None, index_map=None):
    assert xyz32.dtype == np.float32
    xd = torch.from_numpy(xyz32).cuda()
    B = xyz32.shape[0]
    wide = xyz32.astype(np.float64)
    if index_map is None:
        nn = n or xyz32.shape[1]
        order = torch.empty((B, m), dtype=torch.int64, device="cuda")
        sel = torch.empty((B, m), dtype=torch.float64, device="cuda")
        from paper_2604_17720_b200 import _device
        _device.greedy(xd, nn, m, _device.seeds_tensor(seeds, B, "cuda"), order, sel)
        go, gs = order.cpu().numpy(), sel.cpu().numpy()
        wo, ws = oracle.run_kernel_batch(wide, m, seeds, n=nn)
    else:
        s, _ = ffps.run_restricted_batch(xd, torch.from_numpy(index_map).cuda(), m, seeds,
                                         precision="f64")
        assert s.selection_dist2.dtype == torch.float64
        go, gs = s.indices.cpu().numpy(), s.selection_dist2.cpu().numpy()
        wo, ws = oracle.run_kernel_batch(wide, m, seeds, index_map=index_map)
    for b in range(B):
        bad = np.flatnonzero(go[b] != wo[b])
        assert bad.size == 0, f"cloud {b}: first divergence at {bad[0]} of {m}"
        assert np.array_equal(gs[b], ws[b]), f"cloud {b}: selection distances differ"


@pytest.mark.parametrize("kind", ["uniform", "ties", "grid", "collinear"])
def test_mixed_random_batches_vs_binary64_oracle(cuda, kind, schedule):
    rng = np.random.default_rng(hash(("mixed", kind)) % 2**32)
    for N, m, B in [(1, 1, 2), (33, 33, 2), (1000, 250, 3), (1728, 1728, 1), (5000, 1300, 2),
                    (20000, 700, 2), (60000, 400, 2)]:
        if kind == "grid":
            N = min(N, 1728)
            m = min(m, N)
        if schedule in ("stream", "small") and N > 20000:
            continue  # slow schedules: covered up to 20K points
        seeds = rng.integers(0, N, size=B)
        _check_mixed(_cloud(rng, B, N, kind, np.float32), m, seeds)


@pytest.mark.parametrize("sched", ["grid@1", "grid@2", "grid@4", "grid@1/km8",
                                   "grid@2/km8", "grid@4/km8"])
def test_mixed_grid_sizes_ties_and_restricted(cuda, sched):
    """K1g's float-coordinate instances on every bucket size class (32/64/128
    points per bucket), massive ties, candidate prefixes and restricted runs."""
    with _Sched(sched):
        rng = np.random.default_rng(31)
        for N, m, B, kind in [(31, 31, 2, "ties"), (1728, 900, 2, "grid"), (20000, 3000, 2, "ties"),
                              (140000, 300, 1, "uniform"), (300000, 200, 1, "ties")]:
            _check_mixed(_cloud(rng, B, N, kind, np.float32), min(m, N),
                         rng.integers(0, N, size=B))
        pts = np.zeros((2, 20000, 3), np.float32)
        pts[:, :400] = rng.random((2, 400, 3))      # 98% duplicates: truncated rounds
        _check_mixed(pts, 3000, np.array([0, 19999]))
        xyz = _cloud(rng, 3, 30000, "uniform", np.float32)
        _check_mixed(xyz, 2000, np.zeros(3, np.int64), n=7500)
        imap = np.stack([rng.permutation(30000)[:12000] for _ in range(3)])
        _check_mixed(xyz, 1500, np.array([0, 5, 11999]), index_map=imap)


@pytest.mark.parametrize("p", [0.0, 0.75])
@pytest.mark.parametrize("cache", [True, False])
def test_mixed_hierarchy_vs_binary64_oracle(cuda, p, cache):
    rng = np.random.default_rng(int(p * 100) + 7 * cache)
    budgets = (6000, 1500, 375, 93)
    xyz = _cloud(rng, 3, 24000, "uniform", np.float32)
    layers, total, _ = ffps.hierarchical_sample_batch(torch.from_numpy(xyz).cuda(), budgets,
                                                      ffps.PruneConfig(p=p), 0, cache,
                                                      precision="f64")
    for b in range(3):
        want = oracle.hierarchical(xyz[b].astype(np.float64), budgets, p, 0, cache)
        for li, (wi, ws) in enumerate(want):
            assert np.array_equal(layers[li].indices[b].cpu().numpy(), wi), (b, li)
            assert np.array_equal(layers[li].selection_dist2[b].cpu().numpy(), ws), (b, li)


def test_mixed_equals_float64_run_and_host_pipeline(cuda):
    """Mixed == the all-double kernels on the upcast cloud (device API) ==
    the host pipeline from pinned float32 buffers (fills included)."""
    rng = np.random.default_rng(3)
    budgets = (12500, 3125, 781, 195)
    xyz = _cloud(rng, 4, 50000, "uniform", np.float32)
    xd = torch.from_numpy(xyz).cuda()
    a, _, _ = ffps.hierarchical_sample_batch(xd, budgets, ffps.PruneConfig(p=0.75), 0, True,
                                             precision="f64")
    b, _, _ = ffps.hierarchical_sample_batch(xd.double(), budgets, ffps.PruneConfig(p=0.75))
    assert torch.equal(a[0].indices, b[0].indices)
    assert torch.equal(a[0].selection_dist2, b[0].selection_dist2)
    res, _ = ffps.hierarchical_sample_host(torch.from_numpy(xyz).pin_memory(), budgets,
                                           ffps.PruneConfig(p=0.75), precision="f64")
    assert torch.equal(res[0][0], a[0].indices.cpu())
    assert res[0][1].dtype == torch.float64
    assert torch.equal(res[0][1], a[0].selection_dist2.cpu())
    cfg = ffps.PruneConfig(p=0.75, fill_mode=ffps.FillMode.SEEDED_RANDOM, rng_seed=3)
    ra, _ = ffps.fps_prune_batch(xd, 12500, cfg, precision="f64")
    rb, _ = ffps.fps_prune_batch(xd.double(), 12500, cfg)
    assert torch.equal(ra.indices, rb.indices) and torch.equal(ra.selection_dist2,
                                                               rb.selection_dist2)


def test_mixed_coverage_equals_binary64(cuda):
    rng = np.random.default_rng(4)
    xyz = _cloud(rng, 3, 30000, "uniform", np.float32)
    xd = torch.from_numpy(xyz).cuda()
    s, _ = ffps.fps_batch(xd, 3001, precision="f64")
    idx = s.indices[:, :3000].contiguous()
    got = ffps.coverage_d2_batch(xd, idx, precision="f64")
    assert got.dtype == torch.float64
    assert torch.equal(got, ffps.coverage_d2_batch(xd.double(), idx))
    assert torch.equal(got, s.selection_dist2[:, 3000])   # metrics/kernel identity


@pytest.mark.parametrize("kd", ["cl1", "cl2", "global"])
def test_mixed_kd_build_variants(cuda, kd, monkeypatch):
    """K0 on float coordinates writing binary64 running distances, in each
    K0 configuration."""
    if kd == "global":
        monkeypatch.setenv("FFPS_KD_STAGE", "0")
    else:
        monkeypatch.setenv("FFPS_KD_CL", kd[-1])
    with _Sched("grid"):
        rng = np.random.default_rng(37)
        for N, m, B in [(65, 40, 2), (3000, 700, 80), (60000, 500, 2)]:
            _check_mixed(_cloud(rng, B, N, "ties", np.float32), m, rng.integers(0, N, size=B))


def test_precision_argument_checks(cuda):
    x = torch.zeros((1, 10, 3), dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError):
        ffps.fps_batch(x, 3, precision="f32")
    with pytest.raises(ValueError):
        ffps.fps_batch(x.float(), 3, precision="f16")


@pytest.mark.parametrize("precision", [None, "f64"])
@pytest.mark.parametrize("cache", [True, False])
@pytest.mark.parametrize("fill", ["slice", "random"])
def test_fused_hierarchy_abi_equals_python_pipeline(cuda, precision, cache, fill):
    """ffps_hierarchical_sample (one C call for the whole pyramid) returns
    exactly hierarchical_sample_batch's layers and counters."""
    rng = np.random.default_rng(17)
    xd = torch.from_numpy(_cloud(rng, 5, 24000, "ties", np.float32)).cuda()
    cfg = ffps.PruneConfig(p=0.75, rng_seed=9, fill_mode=ffps.FillMode.DETERMINISTIC_SLICE
                           if fill == "slice" else ffps.FillMode.SEEDED_RANDOM)
    budgets = (6000, 1500, 375, 93)
    seeds = np.array([0, 5, 17, 3, 100])
    a, ta, pa = ffps.hierarchical_sample_batch(xd, budgets, cfg, seeds, cache, precision=precision)
    b, tb, pb = ffps.hierarchical_sample_fused(xd, budgets, cfg, seeds, cache, precision=precision)
    for la, lb in zip(a, b):
        assert torch.equal(la.indices, lb.indices)
        assert torch.equal(la.selection_dist2, lb.selection_dist2)
        assert la.fill_boundary == lb.fill_boundary
    assert vars(ta) == vars(tb) and [vars(x) for x in pa] == [vars(x) for x in pb]
