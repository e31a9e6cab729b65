#!/bin/bash
# k_improve tuning sweep (G lanes per vertex x U edges in flight) + phase breakdown.
mkdir -p gpurun_out
out=gpurun_out/sweep_${1:-r01}.log; : > $out
for G in 1 2 4 8; do for U in 1 2 4 8; do
  echo "G=$G U=$U $(OCM_IMPROVE_G=$G OCM_IMPROVE_U=$U timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["value"], d["roofline"]["avg_launch_ms"], d["roofline"]["frac"])')" >> $out
done; done
OCM_PHASES=1 timeout 300 python scripts/profile_solve.py --solves 3 >> $out 2>&1
