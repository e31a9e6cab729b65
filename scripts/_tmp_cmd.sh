OCM_PREP_TIMING=1 timeout 120 python scripts/e2e_breakdown.py > gpurun_out/e2e_r01o.log 2>&1
cat gpurun_out/e2e_r01o.log
