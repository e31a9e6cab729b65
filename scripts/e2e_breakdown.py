"""Wall-time breakdown of the end-to-end call (ocm_solve on a host graph):
upload, region split, packing, solve. Run with OCM_PREP_TIMING=1."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1111_0627_b200 as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
g = P.generate_uniform(n, 8, 1, 100, 1111_0627)
P.solve(g)  # pins the host arrays, warms the pool
for _ in range(3):
    t0 = time.perf_counter()
    s = P.solve(g, P.SolveOptions(objective="min"))
    t1 = time.perf_counter()
    print(f"e2e_ms={1e3 * (t1 - t0):.3f} device_ms={s.stats.device_ms:.3f} "
          f"prep_ms={s.stats.host_prep_ms:.3f} h2d={s.stats.h2d_bytes}", file=sys.stderr)
