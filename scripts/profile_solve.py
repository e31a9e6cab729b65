"""Profiling driver: one warm-up solve + N measured solves of the benchmark
graph (uniform n=1e6, deg 8). Use under ncu or with OCM_PHASES=1."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1111_0627_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--deg", type=int, default=8)
ap.add_argument("--seed", type=int, default=1111_0627)
ap.add_argument("--solves", type=int, default=1)
ap.add_argument("--objective", default="min")
ap.add_argument("--warmup", type=int, default=1)
ap.add_argument("--kind", default="uniform",
                help="generator kind (graph built in HBM, except uniform graphs up to 10^7 vertices)")
ap.add_argument("--dmax", type=int, default=1 << 20)
a = ap.parse_args()
if a.kind == "uniform" and a.n <= 10_000_000:
    g = P.generate_uniform(a.n, a.deg, 1, 100, a.seed)
    s = P.Session(g, P.SolveOptions(objective=a.objective))
else:
    s = P.Session.generated(P.Generator(a.kind, n=a.n, deg=a.deg, dmax=a.dmax, seed=a.seed),
                            P.SolveOptions(objective=a.objective))
for _ in range(a.warmup):
    s.solve()
for _ in range(a.solves):
    sol = s.solve()
    print(sol.mu_exact, sol.stats, file=sys.stderr)
