OCM_PREP_TIMING=1 timeout 120 python scripts/e2e_breakdown.py > gpurun_out/e2e_r01z.log 2>&1; tail -6 gpurun_out/e2e_r01z.log
OCM_PHASES=1 timeout 120 python scripts/profile_solve.py --solves 2 > gpurun_out/phases_r01z.log 2>&1
bash scripts/gpu_round.sh r01z tests
tail -3 gpurun_out/pytest_gpu_r01z.log
