#!/usr/bin/env python
"""Record the reference's OWN test suites as replayable fixtures.

Runs the unmodified reference's test modules for the hot path
(/root/reference/pkg/tests: test_fps_core, test_fps_prune, test_fps_cache,
test_metrics, and the acceptance criteria that call the library in-process)
against the unmodified reference (PYTHONPATH=/root/reference/pkg/src), with
the recording plugin suite_recorder.py wrapping the public hot-path entry
points.  Every top-level call those tests make — arguments, outputs or the
exception raised — lands in tests/golden/suite/{calls.json, calls.npz}.
tests/test_gpu_reference_suite.py replays them through this package on the
GPU (the Python reference cannot travel to the GPU box) and requires
bit-identical outputs and the same exception classes.

Run in this container only (needs /root/reference):
    python tests/golden/make_suite_golden.py
"""

from __future__ import annotations

import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg"
OUT = os.path.join(HERE, "suite")
MODULES = ["test_fps_core.py", "test_fps_prune.py", "test_fps_cache.py", "test_metrics.py",
           "test_acceptance.py"]
# acceptance criteria that run the library in-process (1, 2 and 8 drive the
# CLI in subprocesses, 4 and 5 are wall-clock / distribution studies whose
# library calls are covered by the others)
ACCEPTANCE = "criterion_3 or criterion_6 or criterion_7"


def main() -> None:
    env = dict(os.environ, PYTHONPATH=f"{REF}/src{os.pathsep}{HERE}", FFPS_SUITE_OUT=OUT)
    args = [sys.executable, "-m", "pytest", "-q", "-p", "suite_recorder", "-p",
            "no:cacheprovider", "--rootdir", REF]
    args += [os.path.join(REF, "tests", m) for m in MODULES]
    args += ["-k", f"not test_acceptance or {ACCEPTANCE}"]
    proc = subprocess.run(args, env=env, cwd=REF, capture_output=True, text=True)
    print(proc.stdout[-2000:], proc.stderr[-2000:])
    with open(os.path.join(OUT, "calls.json")) as fh:
        meta = json.load(fh)
    meta["generated_by"] = "tests/golden/make_suite_golden.py"
    meta["reference_tests"] = MODULES
    meta["acceptance_selection"] = ACCEPTANCE
    meta["pytest_summary"] = proc.stdout.strip().splitlines()[-1] if proc.stdout.strip() else ""
    with open(os.path.join(OUT, "calls.json"), "w") as fh:
        json.dump(meta, fh, indent=0)
    recs = meta["records"]
    print(f"{len(recs)} calls recorded, {sum('skipped' in r for r in recs)} skipped, "
          f"{sum('raises' in r for r in recs)} raising")


def record_verify_trials() -> None:
    """The reference verify suites' trial streams (verify.py:52-105): trial
    parameters and a digest of every trial cloud, for seeds 0 and 7, plus
    the suites' own results on small settings — so the device port
    (paper_2604_17720_b200/verify.py) can be checked against them."""
    code = r"""
import hashlib, json, sys
import numpy as np
from flashfps import verify as V
out = {"trials": [], "results": []}
for suite, rng_seed, trials, max_n in (("prefix", 0, 12, 1024), ("prefix", 7, 12, 4096),
                                       ("oracle", 0, 12, 1024), ("oracle", 3, 12, 512)):
    rng = np.random.default_rng(rng_seed)
    for t in range(trials):
        flavor = V._FLAVORS[t % len(V._FLAVORS)]
        if suite == "prefix":
            n = int(rng.integers(64, max_n + 1)); m = None
        else:
            n = int(rng.integers(2, max_n + 1)); m = int(rng.integers(1, min(256, n) + 1))
        cs = int(rng.integers(0, 2**31))
        cloud = V._trial_cloud(flavor, n, cs, rng)
        seed_index = int(rng.integers(0, n))
        out["trials"].append({"suite": suite, "rng_seed": rng_seed, "t": t, "flavor": flavor,
                              "n": n, "m": m, "cloud_seed": cs, "seed_index": seed_index,
                              "sha": hashlib.sha256(cloud.points.tobytes()).hexdigest()[:20]})
for r in V.run_suites("prefix", 12, 1024, 7) + V.run_suites("oracle", 12, 256, 3) + \
        [V.run_counters_suite(20000, rng_seed=5)]:
    out["results"].append({"name": r.name, "trials": r.trials, "passed": r.passed})
json.dump(out, sys.stdout)
"""
    env = dict(os.environ, PYTHONPATH=f"{REF}/src")
    proc = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                          check=True)
    with open(os.path.join(OUT, "verify_trials.json"), "w") as fh:
        fh.write(proc.stdout)
    print("verify trial streams recorded")


if __name__ == "__main__":
    main()
    record_verify_trials()
