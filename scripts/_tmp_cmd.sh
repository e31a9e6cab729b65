bash scripts/gpu_round.sh r01m tests
tail -22 gpurun_out/pytest_gpu_r01m.log
OCM_PHASES=1 timeout 120 python scripts/profile_solve.py --solves 2 > gpurun_out/phases_r01m.log 2>&1
OCM_PHASES=1 timeout 120 python scripts/profile_solve.py --solves 1 --objective max >> gpurun_out/phases_r01m.log 2>&1
