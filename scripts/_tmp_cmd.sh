cat > /tmp/big.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import paper_1111_0627_b200 as P
kind, n = sys.argv[1], int(sys.argv[2])
spec = P.Generator(kind, n=n, deg=8, dmax=1 << 20, seed=1111_0627)
s = P.Session.generated(spec, P.SolveOptions(objective="min"))
sol = s.solve()
print(kind, n, sol.stats.device_ms, sol.stats.spf_passes, sol.stats.host_prep_ms, file=sys.stderr)
PY
for cfg in "uniform 1000000" "powerlaw 64000000" "uniform 250000000"; do
  for gu in "1 4" "1 8" "2 4" "2 8"; do
    set -- $gu
    echo "== $cfg G=$1 U=$2" >> gpurun_out/big_r01k.log
    OCM_IMPROVE_G=$1 OCM_IMPROVE_U=$2 OCM_PHASES=1 timeout 300 python /tmp/big.py $cfg >> gpurun_out/big_r01k.log 2>&1
  done
done
