bash scripts/gpu_round.sh r01i tests
tail -5 gpurun_out/pytest_gpu_r01i.log
OCM_PHASES=1 timeout 120 python scripts/profile_solve.py --solves 1 > gpurun_out/phases_r01i.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_r01i.log 2> gpurun_out/bench_r01i.err; tail -1 gpurun_out/bench_r01i.log | head -c 3000
