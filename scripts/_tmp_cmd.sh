for v in default mb3 indeg; do
  if [ $v = default ]; then unset OCM_LIB; else export OCM_LIB=$PWD/paper_1111_0627_b200/lib/libocm_b200_$v.so; fi
  echo "== $v" >> gpurun_out/phases_r01g.log
  OCM_PHASES=1 timeout 120 python scripts/profile_solve.py --solves 1 >> gpurun_out/phases_r01g.log 2>&1
done
unset OCM_LIB
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_solve -s 1 -c 1 -o gpurun_out/solve_r01g -f python scripts/profile_solve.py --solves 1 > gpurun_out/ncu_r01g.log 2>&1
