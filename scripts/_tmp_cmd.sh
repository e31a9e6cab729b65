for g in 1 2 1 2; do
  echo "== G=$g" >> gpurun_out/gab_r01x.log
  OCM_IMPROVE_G=$g OCM_PHASES=1 timeout 120 python scripts/profile_solve.py --solves 2 >> gpurun_out/gab_r01x.log 2>&1
done
timeout 900 python bench.py > gpurun_out/bench_r01x.log 2> gpurun_out/bench_r01x.err; echo "bench rc=$?"; tail -c 2500 gpurun_out/bench_r01x.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01x.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/launches_r01x.log 2>&1; echo launches rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_solve -s 1 -c 1 -o gpurun_out/solve_r01x -f python scripts/profile_solve.py --solves 1 > gpurun_out/ncu_r01x.log 2>&1; echo ncu rc=$?
