"""Generate the golden vectors in tests/golden/ from the UNMODIFIED reference.

Run in the build container only (it imports /root/reference/pkg/src, which
does not exist on the GPU box):

    python tests/golden/make_golden.py

Outputs ``golden.npz`` (indices / selection distances / stats) and
``manifest.json`` (one entry per case: operation, cloud recipe + SHA-256,
parameters, output keys).  Clouds are regenerated at test time from their
recipe (tests/golden/clouds.py) and checked against the stored SHA-256;
literal clouds (collinear worked example etc.) are stored verbatim.

fp64 cases come from the reference itself (``fps``, ``fps_prune``,
``hierarchical_sample``, ``verify_prefix_property``).  The reference has no
float32 path, so the ``fps32`` cases come from ``_run_kernel_f32_numpy`` below:
an independent NumPy-float32 restatement of fps_core.py:110-175 (NumPy float32
ufuncs are correctly rounded binary32 operations, no contraction).  They pin
the binary32 instantiation of the C oracle and of the CUDA kernel.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

import flashfps as ref  # noqa: E402  (the unmodified reference)
from flashfps.fps_prune import FillMode  # noqa: E402

from clouds import digest, make_cloud  # noqa: E402

COLLINEAR = np.array([(0, 0, 0), (1, 0, 0), (2, 0, 0), (3, 0, 0), (10, 0, 0)], dtype=float)


def _run_kernel_f32_numpy(points32: np.ndarray, m: int, seed: int):
    """Independent binary32 restatement of fps_core.py:110-175 in NumPy."""
    xs = np.ascontiguousarray(points32[:, 0], dtype=np.float32)
    ys = np.ascontiguousarray(points32[:, 1], dtype=np.float32)
    zs = np.ascontiguousarray(points32[:, 2], dtype=np.float32)
    n = xs.shape[0]
    order = np.empty(m, dtype=np.int64)
    sel = np.empty(m, dtype=np.float32)
    dist = np.full(n, np.inf, dtype=np.float32)
    order[0] = seed
    sel[0] = np.inf
    dist[seed] = -np.inf
    out = np.empty(n, dtype=np.float32)
    scr = np.empty(n, dtype=np.float32)
    px, py, pz = xs[seed], ys[seed], zs[seed]
    for k in range(1, m):
        np.subtract(xs, px, out=out)
        np.multiply(out, out, out=out)
        np.subtract(ys, py, out=scr)
        np.multiply(scr, scr, out=scr)
        np.add(out, scr, out=out)
        np.subtract(zs, pz, out=scr)
        np.multiply(scr, scr, out=scr)
        np.add(out, scr, out=out)
        np.minimum(dist, out, out=dist)
        j = int(np.argmax(dist))
        order[k] = j
        sel[k] = dist[j]
        dist[j] = -np.inf
        px, py, pz = xs[j], ys[j], zs[j]
    return order, sel


def main():
    arrays: dict[str, np.ndarray] = {}
    cases: list[dict] = []

    def cloud_entry(kind, n, seed):
        pts = make_cloud(kind, n, seed)
        return pts, {"kind": kind, "n": n, "seed": seed, "sha": digest(pts)}

    def add(case, **outs):
        cid = f"c{len(cases)}"
        case["id"] = cid
        case["outputs"] = {}
        for k, v in outs.items():
            key = f"{cid}__{k}"
            arrays[key] = np.asarray(v)
            case["outputs"][k] = key
        cases.append(case)

    # ---- literal worked examples (test_fps_core.py:20-41, test_fps_prune.py:55-63)
    arrays["lit__collinear"] = COLLINEAR
    arrays["lit__two"] = np.array([(0, 0, 0), (5, 0, 0)], dtype=float)
    arrays["lit__single"] = np.array([(1, 2, 3)], dtype=float)
    for lit, m, seed in (("collinear", 5, 0), ("collinear", 3, 2), ("two", 2, 0),
                         ("single", 1, 0)):
        cloud = ref.PointCloud(arrays[f"lit__{lit}"])
        s, st = ref.fps(cloud, m, seed)
        add({"op": "fps", "literal": f"lit__{lit}", "m": m, "seed": seed,
             "stats": [st.distance_evals, st.iterations, st.candidates]},
            indices=s.indices, sel=s.selection_dist2)
    for m1, p in ((4, 0.5), (5, 0.5)):
        cloud = ref.PointCloud(COLLINEAR)
        s, st = ref.fps_prune(cloud, m1, ref.PruneConfig(p=p), 0)
        add({"op": "prune", "literal": "lit__collinear", "m1": m1, "p": p, "seed": 0,
             "fill": "slice", "fill_boundary": s.fill_boundary,
             "stats": [st.distance_evals, st.iterations, st.candidates]},
            indices=s.indices, sel=s.selection_dist2)

    # ---- randomized fps vs reference (mirrors test_fps_core.py:50-61 at larger n)
    rng = np.random.default_rng(20260418)
    kinds = ["uniform", "ties", "clusters", "uniform32", "ties"]
    for t in range(30):
        kind = kinds[t % len(kinds)]
        n = int(rng.integers(2, 3000))
        m = int(rng.integers(1, min(n, 700) + 1))
        seed = int(rng.integers(0, n))
        pts, cl = cloud_entry(kind, n, 1000 + t)
        s, st = ref.fps(ref.PointCloud(pts), m, seed)
        add({"op": "fps", "cloud": cl, "m": m, "seed": seed,
             "stats": [st.distance_evals, st.iterations, st.candidates]},
            indices=s.indices, sel=s.selection_dist2)

    # ---- benchmark-shaped fps on fp32-representable inputs (BASELINE config 1, C2 stage 1)
    for kind, n, m, seed in (("uniform32", 4096, 1024, 0), ("uniform32", 4096, 1024, 1),
                             ("ties", 4096, 4096, 7), ("uniform32", 24000, 6000, 0)):
        pts, cl = cloud_entry(kind, n, seed)
        s, st = ref.fps(ref.PointCloud(pts), m, 0)
        add({"op": "fps", "cloud": cl, "m": m, "seed": 0,
             "stats": [st.distance_evals, st.iterations, st.candidates]},
            indices=s.indices, sel=s.selection_dist2)

    # ---- fps_prune (slice + random fill) vs reference (test_fps_prune.py:74-88 style)
    for t in range(24):
        n = int(rng.integers(1, 2500))
        m1 = int(rng.integers(1, n + 1))
        p = float(rng.choice([0.0, 0.25, 0.3, 0.5, 0.6, 0.75, 0.8, 0.9,
                              float(rng.uniform(0, 0.999))]))
        fill = "random" if t % 3 == 2 else "slice"
        kind = kinds[t % len(kinds)]
        pts, cl = cloud_entry(kind, n, 5000 + t)
        cfg = ref.PruneConfig(p=p, fill_mode=FillMode.SEEDED_RANDOM if fill == "random"
                              else FillMode.DETERMINISTIC_SLICE, rng_seed=7 + t)
        k = cfg.kernel_budget(m1)
        c = min(cfg.candidate_count(n, m1), n)
        seed = int(rng.integers(0, c))
        s, st = ref.fps_prune(ref.PointCloud(pts), m1, cfg, seed)
        add({"op": "prune", "cloud": cl, "m1": m1, "p": p, "seed": seed, "fill": fill,
             "rng_seed": 7 + t, "fill_boundary": s.fill_boundary,
             "stats": [st.distance_evals, st.iterations, st.candidates]},
            indices=s.indices, sel=s.selection_dist2)

    # ---- hierarchical cache on / off (test_fps_cache.py:37-81, C2-shaped pyramids)
    hier = [("uniform32", 2400, (600, 150, 37, 9), 0.0, 0),
            ("uniform32", 2400, (600, 150, 37, 9), 0.25, 0),
            ("uniform32", 2400, (600, 150, 37, 9), 0.5, 0),
            ("uniform32", 2400, (600, 150, 37, 9), 0.75, 0),
            ("ties", 1000, (250, 62, 15), 0.75, 3),
            ("clusters", 1500, (375, 93, 23, 5), 0.5, 11),
            ("uniform32", 2400, (600, 150, 37, 9), 0.9, 0),     # prefix theorem breaks
            ("uniform32", 24000, (6000, 1500, 375, 93), 0.75, 0)]
    for kind, n, budgets, p, seed in hier:
        pts, cl = cloud_entry(kind, n, 77)
        for cache in (True, False):
            if n > 20000 and not cache:
                continue
            samples, st = ref.hierarchical_sample(ref.PointCloud(pts), budgets,
                                                  ref.PruneConfig(p=p), seed,
                                                  cache_enabled=cache)
            outs = {}
            for li, s in enumerate(samples):
                outs[f"L{li}_indices"] = s.indices
                outs[f"L{li}_sel"] = s.selection_dist2
            add({"op": "hier", "cloud": cl, "budgets": list(budgets), "p": p, "seed": seed,
                 "cache": cache, "fill_boundaries": [s.fill_boundary for s in samples],
                 "stats": [st.distance_evals, st.iterations, st.candidates, st.cache_bytes]},
                **outs)

    # ---- prefix property under ties (test_fps_cache.py:109-120)
    for seed in range(4):
        pts, cl = cloud_entry("ties", 256, seed)
        res = ref.verify_prefix_property(ref.PointCloud(pts), 64, 32, seed_index=seed * 11 % 256)
        add({"op": "prefix", "cloud": cl, "m1": 64, "m2": 32, "seed": seed * 11 % 256,
             "ok": bool(res.ok)})

    # ---- float32 restatement goldens (pin the binary32 oracle / kernel)
    for kind, n, m, seed in (("uniform32", 4096, 1024, 0), ("ties", 3000, 900, 5),
                             ("clusters", 5000, 1250, 2), ("uniform32", 24000, 6000, 0)):
        pts, cl = cloud_entry(kind, n, seed)
        o, s = _run_kernel_f32_numpy(pts.astype(np.float32), m, 0)
        add({"op": "fps32", "cloud": cl, "m": m, "seed": 0}, indices=o, sel=s)

    # ---- coverage radius (metrics.py:45-52) of fps / fps_prune / random samples
    arrays["lit__line"] = np.array([(0, 0, 0), (10, 0, 0)], dtype=float)
    add({"op": "coverage", "literal": "lit__line", "sample": "given",
         "value": ref.coverage_radius(np.array([0]), ref.PointCloud(arrays["lit__line"]))},
        sample=np.array([0]))
    for t, (kind, n, m, how) in enumerate((("uniform", 50, 50, "all"),
                                           ("uniform", 3000, 300, "fps"),
                                           ("ties", 2000, 400, "fps"),
                                           ("clusters", 4000, 500, "prune"),
                                           ("uniform32", 6000, 700, "random"),
                                           ("ties", 1500, 1, "random"),
                                           ("uniform32", 24000, 1500, "prune"))):
        pts, cl = cloud_entry(kind, n, 9000 + t)
        cloud = ref.PointCloud(pts)
        if how == "all":
            idx = np.arange(n)
        elif how == "fps":
            idx = ref.fps(cloud, m, 0)[0].indices
        elif how == "prune":
            idx = ref.fps_prune(cloud, m, ref.PruneConfig(p=0.75), 0)[0].indices
        else:
            idx = np.random.default_rng(t).choice(n, size=m, replace=False)
        add({"op": "coverage", "cloud": cl, "sample": how,
             "value": ref.coverage_radius(idx, cloud)}, sample=idx)

    # ---- FPSC v1 cache wire format (fps_cache.py:26-33, :82-116), reference bytes
    for t, (kind, n, m1, p) in enumerate((("uniform", 200, 50, 0.4), ("ties", 64, 20, 0.0),
                                          ("uniform32", 1000, 250, 0.75))):
        pts, cl = cloud_entry(kind, n, 7000 + t)
        cloud = ref.PointCloud(pts)
        sample, _ = ref.fps_prune(cloud, m1, ref.PruneConfig(p=p), 0)
        cache = ref.CacheRecord.from_sample(cloud, sample)
        blob = cache.to_bytes()
        back = ref.CacheRecord.from_bytes(blob)
        add({"op": "fpsc", "cloud": cl, "m1": m1, "p": p, "fill_boundary": sample.fill_boundary,
             "back_fill_boundary": back.layer1.fill_boundary,
             "footprint": cache.footprint_bytes},
            indices=sample.indices, sel=sample.selection_dist2,
            blob=np.frombuffer(blob, dtype=np.uint8))

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    meta = {"numpy": np.__version__, "reference": "/root/reference/pkg (flashfps "
            f"{ref.__version__})", "cases": cases}
    with open(os.path.join(HERE, "manifest.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    print(f"{len(cases)} cases written")


if __name__ == "__main__":
    main()
