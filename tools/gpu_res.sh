#!/bin/bash
# grid@8 (resident bucket points, 8-CTA clusters): parity + strong-scaling timings + trace
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
TAG=${1:-res}
{
cat > /tmp/res_parity.py <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, "tests")
from test_gpu_mixed import _check_mixed
from test_gpu_parity import _check_batch, _cloud, _Sched
rng = np.random.default_rng(5)
with _Sched("grid@8"):
    for N, m, B, kind in [(31, 31, 2, "ties"), (300, 200, 2, "uniform"), (1728, 900, 2, "grid"), (20000, 3000, 2, "ties"),
                          (50000, 12500, 3, "uniform"), (100000, 2000, 2, "uniform"), (300000, 300, 1, "ties")]:
        x = _cloud(rng, B, N, kind, np.float32)
        seeds = rng.integers(0, N, size=B)
        _check_batch(x, m, seeds); _check_mixed(x, m, seeds)
        print("ok", N, m, B, kind, flush=True)
    pts = np.zeros((2, 20000, 3), np.float32); pts[:, :400] = rng.random((2, 400, 3))
    _check_mixed(pts, 3000, np.array([0, 19999])); _check_batch(pts, 3000, np.array([0, 19999]))
    xyz = _cloud(rng, 3, 30000, "uniform", np.float32)
    imap = np.stack([rng.permutation(30000)[:12000] for _ in range(3)])
    _check_mixed(xyz, 1500, np.array([0, 5, 11999]), index_map=imap)
    print("ok ties/restricted", flush=True)
PY
timeout 900 python /tmp/res_parity.py 2>&1 | tail -12
timeout 600 python tools/sweep_strong.py --batches 8 16 18 --scheds grid@2 grid@8 2>&1
for prec in f32 f64; do echo "-- $prec grid@8 B=8"; timeout 120 python tools/trace_multi.py --sched grid@8 --batch 8 --precision $prec | grep -A7 "rounds \[9"; done
} > gpurun_out/${TAG}.txt 2>&1
echo done
