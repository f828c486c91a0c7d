"""Host-side arithmetic of bench.py: the per-launch unit counts equal the
reference's distance_evals and the CPU sample runs."""

import numpy as np

import bench


def test_stage_units_match_reference_counters():
    b = bench.BUDGETS[200_000]
    exh = bench.stage_units(200_000, b, 0.0, False)
    flash = bench.stage_units(200_000, b, 0.75, True)
    assert sum(c * (m - 1) for c, m in exh) == 10_666_237_500
    assert sum(c * (m - 1) for c, m in flash) == 624_950_000
    assert sum(m for _, m in exh) == 66_406 and flash == [(50_000, 12_500)]
    for n, want in [(24_000, 153_565_500), (100_000, 2_666_488_868),
                    (300_000, 23_999_221_290)]:
        assert sum(c * (m - 1) for c, m in bench.stage_units(n, bench.BUDGETS[n], 0, False)) \
            == want


def test_clouds_are_deterministic():
    a = bench.make_clouds("uniform", 2, 1000, 5)
    assert a.dtype == np.float32 and a.shape == (2, 1000, 3)
    assert np.array_equal(a[1], np.random.default_rng(6).random((1000, 3)).astype(np.float32))
    l1 = bench.lidar_cloud(5000, 3)
    assert l1.shape == (5000, 3) and np.isfinite(l1).all()
    assert np.array_equal(l1, bench.lidar_cloud(5000, 3))


def test_cpu_sample_runs():
    for dtype in ("f64", "f32"):
        dt, cnt = bench.cpu_pipeline_sample(24_000, bench.BUDGETS[24_000], 0.75, 2, "uniform", 2,
                                            dtype)
        assert cnt == 2 and dt > 0


def test_shards_cover_the_global_batch():
    """Strong scaling splits the BASELINE global batch of 64 by cloud; --batch
    gives B clouds per rank (weak)."""
    for world in (1, 2, 4, 8):
        got = [bench.shard(bench.parse([]), world, r) for r in range(world)]
        assert sum(c for _, c, _, _ in got) == 64
        assert [f for f, _, _, _ in got] == [64 // world * r for r in range(world)]
        assert all(gb == 64 and sc == "strong" for _, _, gb, sc in got)
    f, c, gb, sc = bench.shard(bench.parse(["--batch", "16"]), 4, 3)
    assert (f, c, gb, sc) == (48, 16, 64, "weak")


def test_gpus_flag_must_match_world(monkeypatch):
    """--gpus is authoritative: a torchrun world of another size fails loudly."""
    import pytest
    monkeypatch.setenv("WORLD_SIZE", "2")
    monkeypatch.setattr("sys.argv", ["bench.py", "--gpus", "4"])
    with pytest.raises(SystemExit) as ei:
        bench.main()
    assert "WORLD_SIZE=2" in str(ei.value)
