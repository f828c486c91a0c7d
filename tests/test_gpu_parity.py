"""Parity of the CUDA path (through the public API / C ABI) with the
reference's golden vectors and with the CPU oracle.  Bar: bit-exact indices
AND selection distances (integer/index work and exactly reproduced float
arithmetic — no tolerance)."""

import os

import numpy as np
import pytest
import torch

import paper_2604_17720_b200 as ffps
from paper_2604_17720_b200 import _native
from oracle import oracle

pytestmark = pytest.mark.gpu


class _Sched:
    """Run under one schedule: set_schedule(name); "grid@c" = K1g with c CTAs
    per cloud, plain "grid" lets the library pick 1/2/4 from the batch."""

    def __init__(self, name):
        self.name = name

    def __enter__(self):
        from paper_2604_17720_b200 import _device
        name, _, km = self.name.partition("/km")  # "grid@2/km8": K1g with KM = 8
        self.prev_km = os.environ.pop("FFPS_GRID_KM", None)
        if km:
            os.environ["FFPS_GRID_KM"] = km
        self.prev = _device.set_schedule(name)
        return self

    def __exit__(self, *exc):
        from paper_2604_17720_b200 import _device
        _device.set_schedule(self.prev)
        os.environ.pop("FFPS_GRID_KM", None)
        if self.prev_km is not None:
            os.environ["FFPS_GRID_KM"] = self.prev_km


SCHEDULES = ["stream", "small", "bucket", "grid", "grid@1", "grid@2", "grid@4", "grid@2/km8"]


@pytest.fixture(params=SCHEDULES)
def schedule(request):
    """Run the test under each greedy schedule (K1 streaming, K1s small-cloud
    (n <= 8192, else streaming), K0+K1b bucketed, K1g multi-winner with 1/2
    CTAs per cloud)."""
    with _Sched(request.param):
        yield request.param


# ---------------------------------------------------------------- golden (fp64)
def test_fps_matches_reference_goldens(golden, cuda, schedule):
    for c in golden.cases("fps"):
        cloud = ffps.PointCloud(golden.points(c))
        s, st = ffps.fps(cloud, c["m"], c["seed"])
        assert np.array_equal(s.indices, golden.out(c, "indices")), c["id"]
        assert np.array_equal(s.selection_dist2, golden.out(c, "sel")), c["id"]
        assert [st.distance_evals, st.iterations, st.candidates] == c["stats"]
        assert s.fill_boundary == c["m"]


def test_fps_prune_matches_reference_goldens(golden, cuda, schedule):
    for c in golden.cases("prune"):
        cfg = ffps.PruneConfig(p=c["p"], fill_mode=ffps.FillMode(c["fill"]),
                               rng_seed=c.get("rng_seed", 0))
        s, st = ffps.fps_prune(ffps.PointCloud(golden.points(c)), c["m1"], cfg, c["seed"])
        assert np.array_equal(s.indices, golden.out(c, "indices")), c["id"]
        assert np.array_equal(s.selection_dist2, golden.out(c, "sel")), c["id"]
        assert s.fill_boundary == c["fill_boundary"]
        assert [st.distance_evals, st.iterations, st.candidates] == c["stats"]


def test_hierarchy_matches_reference_goldens(golden, cuda, schedule):
    for c in golden.cases("hier"):
        samples, st = ffps.hierarchical_sample(ffps.PointCloud(golden.points(c)), c["budgets"],
                                               ffps.PruneConfig(p=c["p"]), c["seed"],
                                               cache_enabled=c["cache"])
        for li, s in enumerate(samples):
            assert np.array_equal(s.indices, golden.out(c, f"L{li}_indices")), (c["id"], li)
            assert np.array_equal(s.selection_dist2, golden.out(c, f"L{li}_sel")), (c["id"], li)
        assert [s.fill_boundary for s in samples] == c["fill_boundaries"]
        assert [st.distance_evals, st.iterations, st.candidates, st.cache_bytes] == c["stats"]


def test_prefix_property_goldens(golden, cuda):
    for c in golden.cases("prefix"):
        res = ffps.verify_prefix_property(ffps.PointCloud(golden.points(c)), c["m1"], c["m2"],
                                          c["seed"])
        assert bool(res.ok) == c["ok"] and res.ok


def test_fp32_goldens(golden, cuda, schedule):
    for c in golden.cases("fps32"):
        pts = torch.from_numpy(golden.points(c).astype(np.float32)).cuda()
        s, _ = ffps.fps_batch(pts, c["m"], c["seed"])
        assert s.selection_dist2.dtype == torch.float32
        assert np.array_equal(s.indices[0].cpu().numpy(), golden.out(c, "indices")), c["id"]
        assert np.array_equal(s.selection_dist2[0].cpu().numpy(), golden.out(c, "sel")), c["id"]


# ------------------------------------------------------------ worked examples
COLLINEAR = [(0, 0, 0), (1, 0, 0), (2, 0, 0), (3, 0, 0), (10, 0, 0)]


def test_collinear_and_tiny_clouds(cuda, schedule):
    s, st = ffps.fps(ffps.validate_cloud(COLLINEAR), 5, 0)
    assert s.indices.tolist() == [0, 4, 3, 1, 2]
    assert s.selection_dist2[1:].tolist() == [100.0, 9.0, 1.0, 1.0]
    assert st.distance_evals == 20
    s, st = ffps.fps(ffps.validate_cloud([(1, 2, 3)]), 1, 0)
    assert s.indices.tolist() == [0] and np.isinf(s.selection_dist2[0])
    assert st.distance_evals == 0
    s, _ = ffps.fps(ffps.validate_cloud([(0, 0, 0), (5, 0, 0)]), 2, 0)
    assert s.indices.tolist() == [0, 1] and s.selection_dist2[1] == 25.0
    s, _ = ffps.fps_prune(ffps.validate_cloud(COLLINEAR), 5, ffps.PruneConfig(p=0.5), 0)
    assert s.indices.tolist() == [0, 1, 2, 3, 4]


# ------------------------------------------------- randomized vs the oracle
def _check_batch(xyz, m, seeds, n=None, index_map=None):
    xyz_d = torch.from_numpy(xyz).cuda()
    B = xyz.shape[0]
    if index_map is None:
        nn = n or xyz.shape[1]
        order = torch.empty((B, m), dtype=torch.int64, device="cuda")
        sel = torch.empty((B, m), dtype=xyz_d.dtype, device="cuda")
        from paper_2604_17720_b200 import _device
        _device.greedy(xyz_d, nn, m, _device.seeds_tensor(seeds, B, "cuda"), order, sel)
        go, gs = order.cpu().numpy(), sel.cpu().numpy()
        wo, ws = oracle.run_kernel_batch(xyz, m, seeds, n=nn)
    else:
        s, _ = ffps.run_restricted_batch(xyz_d, torch.from_numpy(index_map).cuda(), m, seeds)
        go, gs = s.indices.cpu().numpy(), s.selection_dist2.cpu().numpy()
        wo, ws = oracle.run_kernel_batch(xyz, m, seeds, index_map=index_map)
    for b in range(B):
        bad = np.flatnonzero(go[b] != wo[b])
        assert bad.size == 0, f"cloud {b}: first divergence at {bad[0]} of {m}"
        assert np.array_equal(gs[b], ws[b]), f"cloud {b}: selection distances differ"


def _cloud(rng, B, N, kind, dtype):
    pts = rng.random((B, N, 3))
    if kind == "ties":
        for b in range(B):
            dup = pts[b][rng.integers(0, N, size=N // 2)]
            pts[b] = np.vstack([pts[b][: N - N // 2], dup])[rng.permutation(N)]
    elif kind == "grid":  # massive exact ties of distances
        g = np.stack(np.meshgrid(*(np.arange(12),) * 3, indexing="ij"), -1).reshape(-1, 3)
        pts = np.broadcast_to(g[rng.permutation(len(g))[:N]] * 0.25, (B, N, 3)).copy()
    elif kind == "collinear":
        pts = np.zeros((B, N, 3))
        pts[:, :, 0] = np.arange(N)
    return np.ascontiguousarray(pts.astype(dtype))


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("kind", ["uniform", "ties", "grid", "collinear"])
def test_random_batches_vs_oracle(cuda, dtype, kind, schedule):
    rng = np.random.default_rng(hash((kind, dtype().itemsize)) % 2**32)
    for N, m, B in [(1, 1, 3), (2, 2, 2), (33, 33, 2), (257, 100, 3), (1000, 250, 4),
                    (1728, 1728, 1), (5000, 1300, 3)]:
        if kind == "grid" and N > 1728:
            N = 1728
        seeds = rng.integers(0, N, size=B)
        _check_batch(_cloud(rng, B, N, kind, dtype), m, seeds)


# (plan "threads,register slots,smem slots,{C}", cluster sizes, has a spill variant)
FORCED = {
    np.float32: [("256,2,0,{C}", [1, 2, 3, 4, 7, 8, 16], False),
                 ("256,16,24,{C}", [1, 2, 5], False), ("256,14,36,{C}", [1, 3, 4], True),
                 ("512,14,36,{C}", [1, 2], True), ("256,8,0,{C}", [1, 16], False),
                 ("128,28,72,{C}", [1, 2, 4], False), ("128,10,36,{C}", [1, 3, 9], False),
                 ("256,8,20,{C}", [2, 7], False), ("256,4,16,{C}", [1, 10], False)],
    np.float64: [("256,2,0,{C}", [1, 2, 5, 16], False), ("256,8,8,{C}", [1, 3], False),
                 ("256,6,18,{C}", [1, 2, 4], True), ("512,6,18,{C}", [1, 2], True)],
}


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_every_kernel_configuration(cuda, dtype, monkeypatch):
    """Each compiled (threads, register slots, smem slots) configuration at
    several cluster sizes, including forced spill (capacity < n)."""
    rng = np.random.default_rng(7)
    for fmt, clusters, spills in FORCED[dtype]:
        for C in clusters:
            monkeypatch.setenv("FFPS_FORCE_PLAN", fmt.format(C=C))
            nt, p, s, _ = (int(v) for v in fmt.format(C=C).split(","))
            cap = nt * (p + s) * C
            sizes = {max(2, cap // 3), cap} | ({cap + 777} if spills else set())
            for N in sorted(sizes):
                m = min(N, 97)
                xyz = _cloud(rng, 2, N, "ties" if C % 2 else "uniform", dtype)
                _check_batch(xyz, m, rng.integers(0, N, size=2))


def test_restricted_runs_vs_oracle(cuda, schedule):
    rng = np.random.default_rng(11)
    for dtype in (np.float32, np.float64):
        xyz = _cloud(rng, 3, 3000, "ties", dtype)
        imap = np.stack([rng.permutation(3000)[:1200] for _ in range(3)])
        _check_batch(xyz, 300, np.array([0, 5, 1199]), index_map=imap)


def test_candidate_prefix_runs_vs_oracle(cuda, schedule):
    rng = np.random.default_rng(12)
    xyz = _cloud(rng, 4, 6000, "uniform", np.float32)
    _check_batch(xyz, 375, np.zeros(4, np.int64), n=1500)


@pytest.mark.parametrize("p", [0.0, 0.25, 0.5, 0.75, 0.9])
@pytest.mark.parametrize("cache", [True, False])
def test_hierarchy_batch_vs_oracle(cuda, p, cache, schedule):
    rng = np.random.default_rng(int(p * 100) + cache)
    budgets = (1500, 375, 93, 23)
    xyz = _cloud(rng, 3, 6000, "uniform", np.float32)
    layers, total, per = ffps.hierarchical_sample_batch(torch.from_numpy(xyz).cuda(), budgets,
                                                        ffps.PruneConfig(p=p), 0,
                                                        cache_enabled=cache)
    for b in range(3):
        want = oracle.hierarchical(xyz[b], budgets, p, 0, cache)
        for li, (wi, ws) in enumerate(want):
            assert np.array_equal(layers[li].indices[b].cpu().numpy(), wi), (b, li)
            assert np.array_equal(layers[li].selection_dist2[b].cpu().numpy(), ws), (b, li)
    k = oracle.kernel_budget(p, 1500)
    c = oracle.candidate_count(p, 6000, 1500)
    assert per[0].distance_evals == c * (k - 1) and layers[0].fill_boundary == k


def test_random_fill_matches_reference_semantics(cuda):
    rng = np.random.default_rng(5)
    pts = rng.random((400, 3))
    cfg = ffps.PruneConfig(p=0.5, fill_mode=ffps.FillMode.SEEDED_RANDOM, rng_seed=1)
    a, _ = ffps.fps_prune(ffps.PointCloud(pts), 100, cfg, 0)
    k = a.fill_boundary
    order, _, _ = oracle.run_kernel(pts[:200], k, 0)
    remaining = np.ones(400, bool)
    remaining[order] = False
    fill = np.random.default_rng(1).choice(np.flatnonzero(remaining), size=100 - k,
                                           replace=False)
    assert np.array_equal(a.indices, np.concatenate([order, fill]))
    assert (a.selection_dist2[k:] == 0).all()


def test_fill_slice_kernel_vs_oracle(cuda):
    rng = np.random.default_rng(9)
    for k, m1, n in [(1, 2, 10), (12, 50, 200), (1500, 6000, 24000), (70000, 300000, 300000)]:
        B = 2
        order = torch.full((B, m1), -1, dtype=torch.int64)
        for b in range(B):
            order[b, :k] = torch.from_numpy(rng.permutation(n)[:k])
        od = order.cuda()
        sd = torch.full((B, m1), 7.0, dtype=torch.float32, device="cuda")
        from paper_2604_17720_b200 import _device
        _device.fill_slice(od, sd, k, m1)
        for b in range(B):
            want = oracle.fill_slice(order[b, :k].numpy(), n, m1 - k)
            assert np.array_equal(od[b, k:].cpu().numpy(), want), (k, m1, b)
            assert (sd[b, k:] == 0).all() and (sd[b, :k] == 7.0).all()


# ------------------------------------------------------------- error behaviour
def test_errors_raised_before_device_work(cuda):
    cloud = ffps.validate_cloud(COLLINEAR)
    with pytest.raises(ffps.errors.BudgetOutOfRange):
        ffps.fps(cloud, 0)
    with pytest.raises(ffps.errors.BudgetOutOfRange):
        ffps.fps(cloud, 6)
    with pytest.raises(ffps.errors.SeedOutOfRange):
        ffps.fps(cloud, 3, 5)
    with pytest.raises(ffps.errors.SeedNotInCandidates):
        ffps.fps_prune(ffps.PointCloud(np.random.default_rng(0).random((10, 3))), 4,
                       ffps.PruneConfig(p=0.5), 7)
    with pytest.raises(ffps.errors.BudgetExceedsCloud):
        ffps.hierarchical_sample(cloud, (8, 2), ffps.PruneConfig())


def test_auto_schedule_choices(cuda):
    """AUTO's measured thresholds (abi.cu auto_algo / grid_cluster) on the
    B200's SM count: 4 CTAs per cloud for >= 40K-point clouds while the
    batch's 4-CTA clusters are all resident (32 are), else 2 while batch * 2
    <= SMs, else 1; small / stream / bucket below."""
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    F32, F64, MIX = _native.F32, _native.F64, _native.F32_F64
    for dt in (F32, F64, MIX):
        assert _native.auto_schedule(50_000, 32, dt) == "grid@4"
        assert _native.auto_schedule(50_000, sms // 4 + 1, dt) == "grid@2"
        assert _native.auto_schedule(40_000, 8, dt) == "grid@4"
        assert _native.auto_schedule(39_999, 8, dt) == "grid@2"
        assert _native.auto_schedule(50_000, sms // 2 + 1, dt) == "grid@1"
    assert _native.auto_schedule(4_000, 8, F64) == "small"
    assert _native.auto_schedule(8_000, 8, F64) == "grid@1"
    assert _native.auto_schedule(8_000, 8, F32) == "small"
    assert _native.auto_schedule(9_000, 8, F32) == "stream"
    assert _native.auto_schedule(9_000, 64, F32) == "bucket"


def test_grid_plan_bucket_size_rule(cuda):
    """K1g's bucket size class (abi.cu pick_grid): the smallest class whose
    per-CTA table holds at most 800 buckets, under AUTO's cluster choice."""
    F64 = _native.F32_F64
    p = _native.grid_plan(F64, 50_000, 64)           # C5 headline: 2 CTAs, 782 buckets / CTA
    assert (p["cl"], p["ppl"], p["buckets"]) == (2, 1, 1563)
    p = _native.grid_plan(F64, 75_000, 64)           # 1,172 -> 586 buckets of 64 points / CTA
    assert (p["cl"], p["ppl"]) == (2, 2)
    p = _native.grid_plan(F64, 150_000, 64)
    assert (p["cl"], p["ppl"]) == (2, 4)
    p = _native.grid_plan(F64, 75_000, 16)           # 4 CTAs: 586 buckets of 32 points / CTA
    assert (p["cl"], p["ppl"]) == (4, 1)
    p = _native.grid_plan(F64, 50_000, 8, "grid@1")
    assert p["cl"] == 1 and (p["buckets"] + p["cl"] - 1) // p["cl"] <= 800
    assert p["smem"] > 0
    with pytest.raises(ffps.errors.KernelError):
        _native.grid_plan(F64, 50_000, 8, "stream")


def test_abi_rejects_bad_arguments(cuda):
    lib = _native.load()
    rc = lib.ffps_run_kernel(0, 1, 1, 10, 10, 11, 1, None, 0, 1, 1, 11, None)
    assert rc == -1 and b"not in" in lib.ffps_last_error()
    rc = lib.ffps_run_kernel(7, 1, 1, 10, 10, 5, 1, None, 0, 1, 1, 5, None)
    assert rc == -1
    assert lib.ffps_fill_slice(0, 1, 1, 1, 10, 5, 4, None) == -1


@pytest.mark.parametrize("sched", ["bucket", "grid@1", "grid@2", "grid@4", "grid@1/km8",
                                   "grid@2/km8", "grid@4/km8"])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_bucketed_schedule_sizes_and_ties(cuda, dtype, sched):
    """K0+K1b / K1g forced on every size class: n below / at / above
    one bucket, bucket sizes 32/64/128 (n up to 140K), heavy exact ties."""
    with _Sched(sched):
        rng = np.random.default_rng(21)
        for N, m, B, kind in [(1, 1, 2, "uniform"), (31, 31, 2, "ties"), (32, 20, 2, "grid"),
                              (33, 33, 1, "collinear"), (1728, 900, 2, "grid"),
                              (5000, 600, 2, "ties"), (20000, 300, 2, "uniform"),
                              (140000, 200, 1, "ties")]:
            if kind == "grid":
                N = min(N, 1728)
            _check_batch(_cloud(rng, B, N, kind, dtype), min(m, N), rng.integers(0, N, size=B))


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("sched", ["grid@1", "grid@2", "grid@4", "grid@2/km8",
                                   "grid@4/km8"])
def test_multi_winner_degenerate_ties(cuda, dtype, sched):
    """K1g when hundreds of bucket keys tie (identical points, exhausted
    buckets): the candidate list overflows and rounds fall back to one exact
    winner; results must still match the oracle."""
    with _Sched(sched):
        rng = np.random.default_rng(23)
        for N, m in [(8000, 600), (20000, 3000)]:
            pts = np.zeros((2, N, 3))
            pts[:, : N // 50] = rng.random((2, N // 50, 3))  # 2% distinct, 98% duplicates
            _check_batch(np.ascontiguousarray(pts.astype(dtype)), m, np.array([0, N - 1]))


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("n,m1,p,rng_seed", [
    (24000, 6000, 0.75, 0),      # tail partial Fisher-Yates (pop > 10000, fill > pop // 50)
    (200000, 50000, 0.75, 3),    # C5 shape; seed 3 hits Lemire's rejection loop
    (30000, 30000, 0.5, 5),      # tail with pop == fill (slot 0 keeps its value)
    (5000, 2000, 0.5, 1),        # Floyd + shuffle (pop <= 10000)
    (60000, 1100, 0.05, 2),      # Floyd with pop > 10000, fill <= pop // 50
    (3000, 3000, 0.5, 7),        # Floyd with pop == fill
])
@pytest.mark.parametrize("sequential", [False, True])
def test_seeded_random_fill_matches_numpy(cuda, n, m1, p, rng_seed, dtype, sequential,
                                          monkeypatch):
    """K2r: FillMode.SEEDED_RANDOM on the device equals
    np.random.default_rng(rng_seed).choice(pool, m1 - k, replace=False) of the
    reference (fps_prune.py:96-103) for every cloud, bit for bit — through the
    warp-parallel generator and through its sequential backup."""
    if sequential:
        monkeypatch.setenv("FFPS_FILL_SEQUENTIAL", "1")
    rng = np.random.default_rng(41)
    B = 3
    pts = rng.random((B, n, 3)).astype(dtype)
    cfg = ffps.PruneConfig(p=p, fill_mode=ffps.FillMode.SEEDED_RANDOM, rng_seed=rng_seed)
    out, _ = ffps.fps_prune_batch(torch.from_numpy(pts).cuda(), m1, cfg, seed_index=0)
    k = out.fill_boundary
    idx = out.indices.cpu().numpy()
    sel = out.selection_dist2.cpu().numpy()
    for b in range(B):
        remaining = np.ones(n, dtype=bool)
        remaining[idx[b, :k]] = False
        want = np.random.default_rng(rng_seed).choice(np.flatnonzero(remaining), size=m1 - k,
                                                      replace=False)
        assert np.array_equal(idx[b, k:], want), (n, m1, p, b)
        assert (sel[b, k:] == 0).all()


@pytest.mark.parametrize("kd", ["cl1", "cl2", "global"])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_kd_bucket_build_variants(cuda, kd, dtype, monkeypatch):
    """K0-kd in each configuration — CTA phase on one CTA or a 2-CTA cluster
    (FFPS_KD_CL), leaf phase staged in shared memory or on the global arrays
    (FFPS_KD_STAGE=0) — feeds K1g with the same exact results, including a
    batch too large for 2 CTAs per cloud, restricted (index-mapped) runs and
    ragged sizes around the bucket size."""
    if kd == "global":
        monkeypatch.setenv("FFPS_KD_STAGE", "0")
    else:
        monkeypatch.setenv("FFPS_KD_CL", kd[-1])
    with _Sched("grid"):
        rng = np.random.default_rng(29)
        for N, m, B, kind in [(31, 31, 3, "uniform"), (65, 40, 2, "ties"), (3000, 700, 80, "uniform"),
                              (20000, 900, 2, "ties"), (60000, 500, 2, "uniform")]:
            _check_batch(_cloud(rng, B, N, kind, dtype), min(m, N), rng.integers(0, N, size=B))
        xyz = _cloud(rng, 2, 9000, "uniform", dtype)
        imap = np.stack([rng.permutation(9000)[:5000] for _ in range(2)])
        _check_batch(xyz, 800, np.array([0, 17]), index_map=imap)
