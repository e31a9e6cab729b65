#!/bin/bash
# One gpurun call: GPU parity tests, smoke, bench, reference arm, launch list, ncu --set full on k_solve.
# usage: gpurun -- 'bash scripts/gpu_round.sh <tag> [what...]'   what in {tests,smoke,bench,reference,fused,launches,full}
set -u
TAG=${1:-r01}; shift || true
WHAT=${@:-tests smoke bench reference launches full}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_$TAG.txt 2>&1
for w in $WHAT; do
case $w in
tests) timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "tests rc=$?" ;;
smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" ;;
bench) timeout 900 python bench.py > gpurun_out/bench_$TAG.log 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"; tail -1 gpurun_out/bench_$TAG.log ;;
launches) timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/launches_$TAG.log 2>&1; echo "launches rc=$?" ;;
reference) timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.log 2>&1; echo "reference rc=$?"; tail -1 gpurun_out/bench_ref_$TAG.log ;;
fused) timeout 900 python bench.py --lane fused --no-cpu-baseline > gpurun_out/bench_fused_$TAG.log 2>&1; echo "fused rc=$?"; tail -1 gpurun_out/bench_fused_$TAG.log ;;
full) timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_solve -s 1 -c 1 \
   -o gpurun_out/solve_$TAG -f python scripts/profile_solve.py --solves 1 > gpurun_out/full_$TAG.log 2>&1; echo "full rc=$?" ;;
esac
done
