cat > /tmp/w1.py <<'PY'
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_1111_0627_b200 as P
from paper_1111_0627_b200.sharded import ShardSession, LocalComm, solve_sharded
spec = P.Generator(sys.argv[1], n=int(sys.argv[2]), deg=8, dmax=100000, seed=5)
if sys.argv[3] == "full":
    s = P.Session.generated(spec)
    print("full ok", s.solve().mu_exact, flush=True)
    sys.exit(0)
sh = ShardSession(spec, P.SolveOptions(), 0, int(sys.argv[3]))
(sol,) = solve_sharded([sh], LocalComm())
print("ok", sol.mu_exact, sol.stats.spf_passes, flush=True)
PY
for args in "uniform 50000 1" "uniform 1000 1" "powerlaw 50000 1" "uniform 50000 full"; do
  echo "== $args" >> gpurun_out/w1_r01w.log
  timeout 60 python /tmp/w1.py $args >> gpurun_out/w1_r01w.log 2>&1 || echo "rc=$?" >> gpurun_out/w1_r01w.log
done
cat gpurun_out/w1_r01w.log
bash scripts/gpu_round.sh r01w tests
tail -3 gpurun_out/pytest_gpu_r01w.log
OCM_PHASES=1 timeout 120 python scripts/profile_solve.py --solves 2 > gpurun_out/phases_r01w.log 2>&1
OCM_PHASES=1 timeout 120 python scripts/profile_solve.py --solves 1 --objective max >> gpurun_out/phases_r01w.log 2>&1
