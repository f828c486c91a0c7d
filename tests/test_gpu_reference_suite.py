"""The reference's OWN test suites, replayed through the drop-in on the GPU.

tests/golden/make_suite_golden.py ran the unmodified reference's hot-path
test modules (pkg/tests/test_fps_core.py, test_fps_prune.py,
test_fps_cache.py, test_metrics.py and the in-process acceptance criteria 3,
6 and 7 of test_acceptance.py) against the unmodified reference and recorded
every call those tests made into the library's public entry points (fps,
fps_prune, hierarchical_sample, verify_prefix_property, prefix_reuse,
coverage_radius, candidate_prune): arguments, outputs, or the exception class.
The reference cannot travel to the GPU box, so its assertions are checked
through their inputs and outputs instead: each reference test becomes one
case here that replays its calls through this package and requires
bit-identical outputs (indices, selection distances, fill boundaries,
counters, prefix-check results, covering radii) and the same exception
classes.  Uniform-cube clouds are regenerated from their recipe
(reference io.py:209-210) and checked by SHA-256.
"""

from __future__ import annotations

import hashlib
import json
import os

import numpy as np
import pytest

import paper_2604_17720_b200 as ffps

pytestmark = pytest.mark.gpu

SUITE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "suite")
with open(os.path.join(SUITE, "calls.json")) as _fh:
    META = json.load(_fh)
TESTS = sorted({r["test"] for r in META["records"]})
_ARRAYS = None


def arrays():
    global _ARRAYS
    if _ARRAYS is None:
        _ARRAYS = np.load(os.path.join(SUITE, "calls.npz"))
    return _ARRAYS


def arr(ref) -> np.ndarray:
    if isinstance(ref, dict):  # uniform-cube recipe, io.py:209-210
        a = np.random.default_rng(ref["seed"]).random((ref["n"], 3)) * 1.0
        h = hashlib.sha256(a.tobytes() + str(a.dtype).encode() + str(a.shape).encode())
        assert h.hexdigest()[:20] == ref["sha"], "cloud recipe drifted"
        return a
    return arrays()[ref]


def dec(v):
    if not isinstance(v, dict):
        return v
    t = v["t"]
    if t == "cloud":
        return ffps.PointCloud(arr(v["a"]))
    if t == "arr":
        return arr(v["a"])
    if t == "cfg":
        return ffps.PruneConfig(p=v["p"], fill_mode=ffps.FillMode(v["fill"]),
                                rng_seed=v["rng_seed"])
    if t == "enum":
        return getattr(ffps, v["cls"])(v["v"])
    if t == "sample":
        return ffps.OrderedSample(arr(v["i"]), arr(v["s"]), fill_boundary=v["fb"])
    if t == "budgets":
        return ffps.LayerBudgets(tuple(v["v"]))
    if t == "cache":
        return ffps.CacheRecord(dec(v["layer1"]), v["n"], arr(v["pts"]), v["fp"])
    if t in ("list", "tuple"):
        seq = [dec(x) for x in v["v"]]
        return seq if t == "list" else tuple(seq)
    raise ValueError(t)


def check(want, got, where):
    if not isinstance(want, dict):
        if isinstance(want, float):
            assert isinstance(got, float) and (got == want or (np.isnan(got) and np.isnan(want))), \
                (where, want, got)
        else:
            assert got == want, (where, want, got)
        return
    t = want["t"]
    if t == "sample":
        assert isinstance(got, ffps.OrderedSample), where
        wi, ws = arr(want["i"]), arr(want["s"])
        bad = np.flatnonzero(np.asarray(got.indices) != wi) if got.indices.shape == wi.shape else [0]
        assert len(bad) == 0, f"{where}: indices differ first at {bad[0]}"
        assert np.array_equal(got.selection_dist2, ws), f"{where}: selection_dist2 differ"
        assert got.fill_boundary == want["fb"], where
    elif t == "stats":
        assert [got.distance_evals, got.iterations, got.candidates, got.cache_bytes] == want["v"], \
            where
    elif t == "prefix":
        assert (bool(got.ok), got.first_divergence, got.expected_index, got.actual_index) == \
            (want["ok"], want["first"], want["exp"], want["act"]), where
    elif t == "arr":
        assert np.array_equal(np.asarray(got), arr(want["a"])), where
    elif t in ("list", "tuple"):
        assert len(got) == len(want["v"]), where
        for i, (w, g) in enumerate(zip(want["v"], got)):
            check(w, g, f"{where}[{i}]")
    else:
        raise ValueError(t)


def test_suite_fixture_is_complete():
    recs = META["records"]
    assert len(recs) >= 900 and not any("skipped" in r for r in recs)
    assert "passed" in META["pytest_summary"] and "failed" not in META["pytest_summary"]


@pytest.mark.parametrize("nodeid", TESTS)
def test_reference_test_replays_bit_exact(cuda, nodeid):
    recs = [r for r in META["records"] if r["test"] == nodeid]
    for i, r in enumerate(recs):
        fn = getattr(ffps, r["fn"])
        args = [dec(a) for a in r["args"]]
        kwargs = {k: dec(v) for k, v in r["kwargs"].items()}
        where = f"{nodeid} call {i} {r['fn']}"
        if "raises" in r:
            with pytest.raises(Exception) as ei:
                fn(*args, **kwargs)
            assert type(ei.value).__name__ == r["raises"], (where, repr(ei.value))
            continue
        check(r["result"], fn(*args, **kwargs), where)
