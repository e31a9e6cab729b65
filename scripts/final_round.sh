#!/bin/bash
# End-of-round GPU pass: tests, smoke, bench lines for every BASELINE config,
# the reference arm, the ncu launch list and ncu --set full captures of k_solve
# at configs 2, 4, 5.  usage: gpurun -- 'bash scripts/final_round.sh <tag>'
set -u
TAG=${1:-r02_final}
NCU_BIG=${NCU_BIG:-1}  # 0: skip the config-4/5 captures (large reports)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_$TAG.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.log 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
timeout 1200 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.log 2>&1; echo "reference rc=$?"
for c in 1 3 4 5; do
  timeout 1200 python bench.py --config $c > gpurun_out/bench_cfg${c}_$TAG.log 2>&1; echo "cfg$c rc=$?"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/launches_$TAG.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_solve -s 1 -c 1 \
   -o gpurun_out/solve_cfg2_$TAG -f python scripts/profile_solve.py --solves 1 > gpurun_out/ncu2_$TAG.log 2>&1; echo "ncu2 rc=$?"
[ "$NCU_BIG" = 1 ] && timeout 900 ncu --set full --clock-control none -k regex:k_solve -s 1 -c 1 \
   -o gpurun_out/solve_cfg4_$TAG -f python scripts/profile_solve.py --solves 1 --kind powerlaw-hubs --n 64000000 > gpurun_out/ncu4_$TAG.log 2>&1; echo "ncu4 rc=$?"
[ "$NCU_BIG" = 1 ] && timeout 1200 ncu --set full --clock-control none -k regex:k_solve -s 1 -c 1 \
   -o gpurun_out/solve_cfg5_$TAG -f python scripts/profile_solve.py --solves 1 --kind uniform --n 250000000 > gpurun_out/ncu5_$TAG.log 2>&1; echo "ncu5 rc=$?"
