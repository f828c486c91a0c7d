"""pytest plugin used ONLY by make_suite_golden.py, in this container, while
the reference's own test modules run against the unmodified reference
(PYTHONPATH=/root/reference/pkg/src).  It wraps the reference's public
hot-path entry points and records every top-level call a reference test
makes — arguments, result or exception class — so that
tests/test_gpu_reference_suite.py can replay the reference suite's calls
through the drop-in on the GPU (the reference itself cannot travel there).
"""

from __future__ import annotations

import enum
import functools
import hashlib
import json
import os

import numpy as np

OUT = os.environ.get("FFPS_SUITE_OUT", "")
# entry points of the hot path the reference tests call
FNS = ("fps", "fps_prune", "hierarchical_sample", "hierarchical_sample_detailed",
       "run_restricted", "verify_prefix_property", "prefix_reuse", "run_kernel",
       "coverage_radius", "candidate_prune")
MAX_ELEMS = 1_000_000          # larger arrays are not stored (the call is listed as skipped)

RECORDS: list = []
ARRAYS: dict = {}
RECIPES: dict = {}   # sha -> uniform-cube recipe of clouds made by the reference's generate()
_depth = [0]
_test = [None]


class TooBig(Exception):
    pass


def _sha(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.tobytes() + str(a.dtype).encode() + str(a.shape).encode()).hexdigest()


def _key(a):
    """Array reference: a uniform-cube recipe (regenerated at replay, io.py:209-210)
    when the reference's generate() produced it, else a stored array."""
    h = _sha(a)
    if h in RECIPES:
        return dict(RECIPES[h], sha=h[:20])
    a = np.ascontiguousarray(a)
    if a.size > MAX_ELEMS:
        raise TooBig(a.shape)
    k = "a" + h[:20]
    ARRAYS.setdefault(k, a.copy())
    return k


def enc(v):
    import flashfps as F
    if v is None or isinstance(v, (bool, int, float, str)):
        return v
    if isinstance(v, (np.integer,)):
        return int(v)
    if isinstance(v, (np.floating,)):
        return float(v)
    if isinstance(v, F.PointCloud):
        return {"t": "cloud", "a": _key(v.points)}
    if isinstance(v, np.ndarray):
        return {"t": "arr", "a": _key(v)}
    if isinstance(v, F.PruneConfig):
        return {"t": "cfg", "p": v.p, "fill": v.fill_mode.value, "rng_seed": v.rng_seed}
    if isinstance(v, enum.Enum):
        return {"t": "enum", "cls": type(v).__name__, "v": v.value}
    if isinstance(v, F.OrderedSample):
        return {"t": "sample", "i": _key(v.indices), "s": _key(v.selection_dist2),
                "fb": int(v.fill_boundary)}
    if isinstance(v, F.SamplerStats):
        return {"t": "stats", "v": [v.distance_evals, v.iterations, v.candidates, v.cache_bytes]}
    if isinstance(v, F.LayerBudgets):
        return {"t": "budgets", "v": [int(x) for x in v.budgets]}
    if isinstance(v, F.CacheRecord):
        return {"t": "cache", "layer1": enc(v.layer1), "n": int(v.source_cloud_size),
                "pts": _key(v.points), "fp": int(v.footprint_bytes)}
    if type(v).__name__ == "PrefixCheckResult":
        return {"t": "prefix", "ok": bool(v.ok), "first": v.first_divergence,
                "exp": v.expected_index, "act": v.actual_index}
    if isinstance(v, (list, tuple)):
        return {"t": "list" if isinstance(v, list) else "tuple", "v": [enc(x) for x in v]}
    raise TypeError(f"cannot encode {type(v).__name__}")


def _wrap(name, fn):
    @functools.wraps(fn)
    def w(*args, **kwargs):
        if _depth[0] > 0:
            return fn(*args, **kwargs)
        _depth[0] += 1
        rec = {"test": _test[0], "fn": name}
        try:
            try:
                rec["args"] = [enc(a) for a in args]
                rec["kwargs"] = {k: enc(v) for k, v in kwargs.items()}
            except (TooBig, TypeError) as e:
                rec["skipped"] = f"{type(e).__name__}: {e}"
            try:
                out = fn(*args, **kwargs)
            except Exception as e:
                rec["raises"] = type(e).__name__
                raise
            if "skipped" not in rec:
                try:
                    rec["result"] = enc(out)
                except (TooBig, TypeError) as e:
                    rec["skipped"] = f"{type(e).__name__}: {e}"
            return out
        finally:
            RECORDS.append(rec)
            _depth[0] -= 1
    return w


def _wrap_generate(orig):
    @functools.wraps(orig)
    def g(spec):
        cloud = orig(spec)
        if spec.kind.name == "UNIFORM_CUBE" and spec.side == 1.0:
            RECIPES[_sha(cloud.points)] = {"recipe": "uniform_cube", "n": int(spec.n),
                                           "seed": int(spec.rng_seed)}
        return cloud
    return g


def pytest_configure(config):
    import importlib

    import flashfps as F
    import flashfps.io as FIO
    gen = _wrap_generate(FIO.generate)
    F.generate = FIO.generate = gen
    mods = [F] + [importlib.import_module(f"flashfps.{m}")
                  for m in ("fps_core", "fps_prune", "fps_cache", "metrics")]
    for name in FNS:
        orig = getattr(F, name, None)
        if orig is None:
            continue
        w = _wrap(name, orig)
        for m in mods:
            if getattr(m, name, None) is orig:
                setattr(m, name, w)


def pytest_runtest_setup(item):
    _test[0] = item.nodeid


def pytest_unconfigure(config):
    if not OUT:
        return
    os.makedirs(OUT, exist_ok=True)
    np.savez_compressed(os.path.join(OUT, "calls.npz"), **ARRAYS)
    with open(os.path.join(OUT, "calls.json"), "w") as fh:
        json.dump({"records": RECORDS}, fh, indent=0)
