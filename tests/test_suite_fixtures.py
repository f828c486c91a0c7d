"""CPU checks of the fixtures recorded from the reference's own suites
(tests/golden/make_suite_golden.py): every recorded call decodes (uniform
clouds regenerate from their recipe, SHA-256 checked) and the device port of
the verify suites (paper_2604_17720_b200/verify.py) draws exactly the
reference's trial streams — same flavors, sizes, seeds and trial clouds."""

import hashlib
import json
import os

import numpy as np

from paper_2604_17720_b200 import verify as V

SUITE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "suite")


def test_recorded_reference_calls_decode():
    import test_gpu_reference_suite as R
    n = 0
    for r in R.META["records"]:
        for a in r["args"]:
            R.dec(a)
        n += 1
    assert n >= 900
    assert {r["fn"] for r in R.META["records"]} >= {"fps", "fps_prune", "hierarchical_sample",
                                                   "verify_prefix_property", "coverage_radius",
                                                   "prefix_reuse"}


def test_verify_port_draws_the_reference_trial_streams():
    with open(os.path.join(SUITE, "verify_trials.json")) as fh:
        ref = json.load(fh)
    streams = {}
    for tr in ref["trials"]:
        key = (tr["suite"], tr["rng_seed"])
        if key not in streams:
            streams[key] = np.random.default_rng(tr["rng_seed"])
        rng = streams[key]
        flavor = V._FLAVORS[tr["t"] % len(V._FLAVORS)]
        if tr["suite"] == "prefix":
            n = int(rng.integers(64, (1024 if tr["rng_seed"] == 0 else 4096) + 1))
        else:
            n = int(rng.integers(2, (1024 if tr["rng_seed"] == 0 else 512) + 1))
            m = int(rng.integers(1, min(256, n) + 1))
            assert m == tr["m"]
        cs = int(rng.integers(0, 2**31))
        cloud = V._trial_cloud(flavor, n, cs, rng)
        seed_index = int(rng.integers(0, n))
        assert (flavor, n, cs, seed_index) == (tr["flavor"], tr["n"], tr["cloud_seed"],
                                               tr["seed_index"])
        assert hashlib.sha256(cloud.points.tobytes()).hexdigest()[:20] == tr["sha"], tr
