#!/bin/bash
# One gpurun call: GPU parity tests, smoke, bench, launch list, ncu --set full on k_improve.
# usage: gpurun -- 'bash scripts/gpu_round.sh <tag> [what...]'   what in {tests,smoke,bench,launches,full}
set -u
TAG=${1:-r01}; shift || true
WHAT=${@:-tests smoke bench launches full}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_$TAG.txt 2>&1
for w in $WHAT; do
case $w in
tests) timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "tests rc=$?" ;;
smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" ;;
bench) timeout 900 python bench.py > gpurun_out/bench_$TAG.log 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"; tail -1 gpurun_out/bench_$TAG.log ;;
launches) timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches_$TAG.csv python scripts/profile_solve.py --solves 1 > gpurun_out/launches_$TAG.log 2>&1; echo "launches rc=$?" ;;
full) timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_improve -s 20 -c 3 \
   -o gpurun_out/improve_$TAG -f python scripts/profile_solve.py --solves 1 > gpurun_out/full_$TAG.log 2>&1; echo "full rc=$?" ;;
esac
done
