"""The verify suites (reference verify.py:52-153) on the device: the
reference's own settings pass, the results equal the reference's on the
recorded small settings, the device brute-force oracle equals the C oracle,
and the suites run well beyond the reference's CPU sizes."""

import json
import os

import numpy as np
import pytest

from oracle import oracle
from paper_2604_17720_b200 import verify as V

pytestmark = pytest.mark.gpu
SUITE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "suite")


def test_device_brute_force_oracle_matches_c_oracle(cuda):
    rng = np.random.default_rng(3)
    for n, m in [(1, 1), (7, 7), (500, 120), (1024, 256)]:
        pts = rng.random((n, 3))
        pts[n // 2:] = pts[: n - n // 2]     # exact ties
        wi, ws = V.fps_oracle_device(pts, m, n - 1)
        oi, os_, _ = oracle.run_kernel(pts, m, n - 1)
        assert np.array_equal(wi, oi) and np.array_equal(ws, os_)


def test_results_equal_the_reference_suites(cuda):
    with open(os.path.join(SUITE, "verify_trials.json")) as fh:
        want = json.load(fh)["results"]
    got = (V.run_suites("prefix", 12, 1024, 7) + V.run_suites("oracle", 12, 256, 3)
           + [V.run_counters_suite(20000, rng_seed=5)])
    assert [(r.name, r.trials, r.passed) for r in got] == \
        [(w["name"], w["trials"], w["passed"]) for w in want]
    assert all(r.ok for r in got), [r.failures[:1] for r in got]


def test_acceptance_criterion_1_settings(cuda):
    """test_acceptance.py:47-62: `verify --suite prefix --trials 100 --rng-seed 7`."""
    r, = V.run_suites("prefix", 100, None, 7)
    assert r.ok and r.passed == 100, r.failures[:1]


def test_suites_beyond_reference_scale(cuda):
    """Sizes the reference's CPU suites do not reach: prefix trials up to
    60K points, counters on 1M points."""
    r = V.run_prefix_suite(6, 60_000, 11, min_n=20_000)
    assert r.ok, r.failures[:1]
    c = V.run_counters_suite(1_000_000, rng_seed=2)
    assert c.ok, c.failures


def test_acceptance_criterion_2_settings(cuda):
    """test_acceptance.py:65-79: `verify --suite oracle --trials 50 --max-n 1024
    --rng-seed 11`."""
    r, = V.run_suites("oracle", 50, 1024, 11)
    assert r.ok and r.passed == 50, r.failures[:1]


def test_acceptance_criterion_4_desk_scale_speedup(cuda):
    """test_acceptance.py:104-131: fps_prune (p = 0.75) at least 2.5x faster
    than fps, wall clock, N = 262,144 -> m = 65,536, through the reference
    API (binary64 PointCloud in, host arrays out)."""
    import statistics
    import time

    import paper_2604_17720_b200 as ffps
    cloud = ffps.PointCloud(np.random.default_rng(1).random((262_144, 3)))
    ffps.fps(ffps.PointCloud(np.random.default_rng(2).random((8192, 3))), 2048, 0)  # warm-up
    t0 = time.perf_counter_ns()
    ffps.fps(cloud, 65_536, 0)
    base = time.perf_counter_ns() - t0
    cfg = ffps.PruneConfig(p=0.75)
    ffps.fps_prune(cloud, 65_536, cfg, 0)
    runs = []
    for _ in range(3):
        t0 = time.perf_counter_ns()
        ffps.fps_prune(cloud, 65_536, cfg, 0)
        runs.append(time.perf_counter_ns() - t0)
    speedup = base / statistics.median(runs)
    print(f"criterion 4: fps {base / 1e6:.1f} ms, fps_prune {statistics.median(runs) / 1e6:.1f} ms,"
          f" {speedup:.2f}x")
    assert speedup >= 2.5, speedup
