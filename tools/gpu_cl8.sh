#!/bin/bash
# 8 CTAs per cloud (K1g, 8 lists of 8 exchanged): parity + strong-scaling shapes
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
OUT=gpurun_out/${1:-cl8}.txt
{
timeout 900 python -m pytest tests -m gpu -q -x -k "grid or mixed or adversarial or auto" 2>&1 | tail -3
for shape in "50000 12500" "75000 18750" "100000 25000"; do
  set -- $shape
  timeout 900 python tools/sweep_strong.py --n $1 --iters $2 --batches 4 8 16 --scheds grid@4 grid@8 2>&1
done
for pr in f64 f32; do
  echo "-- grid@8 $pr"
  timeout 600 python tools/trace_multi.py --batch 8 --sched grid@8 --precision $pr 2>&1 | grep -A6 "^rounds \[9"
done
python - <<'PY'
import paper_2604_17720_b200 as f
from paper_2604_17720_b200 import _native as n
for b in (8, 16, 18, 32, 33, 36, 37, 40):
    print("auto", b, n.auto_schedule(50000, b, n.F32_F64))
PY
} > $OUT 2>&1
echo done
