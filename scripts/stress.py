"""Stress run for the persistent kernel's grid barrier and the late round-2
phases (connected-vertex bitmap, block-cooperative attach): many
back-to-back solves on resident sessions must repeat the first solve's
answer exactly, and random graphs solved under different grid sizes and
bitmap settings must agree with each other and with the oracle.

    python scripts/stress.py [--config2 500] [--config4 10] [--graphs 200]
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
import paper_1111_0627_b200 as P  # noqa: E402


def key(sol):
    return (str(sol.mu_exact) if sol.exact else sol.mu, tuple(sol.cycle_vertices),
            sol.stats.spf_passes, sol.stats.outer_iters)


def resident(spec, reps, label):
    t0 = time.time()
    sess = {o: P.Session.generated(spec, P.SolveOptions(objective=o)) for o in ("min", "max")}
    first = {o: key(sess[o].solve()) for o in sess}
    bad = 0
    for _ in range(reps):
        for o in sess:
            bad += key(sess[o].solve()) != first[o]
    certs = {o: sess[o].certify() for o in sess}
    viol = sum(c["key_violations"] + c["policy_violations"] + c["cycle_violations"]
               for c in certs.values())
    print(f"{label}: {2 * reps} solves, mismatches {bad}, certificate violations {viol}, "
          f"{time.time() - t0:.1f}s", flush=True)
    return bad + viol


def graphs(count):
    rng = np.random.default_rng(1111)
    bad = 0
    t0 = time.time()
    for i in range(count):
        kind = ["uniform", "powerlaw", "powerlaw-hubs", "powerlaw-web"][i % 4]
        n = int(rng.integers(50, 20000))
        deg = int(rng.integers(1, 12))
        lo = int(rng.integers(-100, 50))
        spec = P.Generator(kind, n=n, deg=deg, dmax=max(2, n // 2), wlo=lo, whi=lo + int(rng.integers(1, 200)),
                           seed=int(rng.integers(1 << 30)))
        g = P.generate(spec)
        s, d, w = g.edges()
        if i % 5 == 4:  # float lane
            w = w / 8 + 0.125
            g = P.build_graph(g.n, (s, d, w))
        objective = "max" if i % 2 else "min"
        res = []
        for env in ({}, {"OCM_GRID": "37"}, {"OCM_CBITS_MIN_N": "0"}, {"OCM_GRID": "150", "OCM_CBITS_MIN_N": "0"}):
            for k, v in env.items():
                os.environ[k] = v
            try:
                res.append(key(P.Session(g, P.SolveOptions(objective=objective)).solve()))
            finally:
                for k in env:
                    os.environ.pop(k, None)
        ok = all(r == res[0] for r in res)
        if i % 10 == 0:  # and against the oracle
            ref = O.oracle_solve(g.n, s, d, w, objective, "tarjan")
            ok &= tuple(ref.cycle) == res[0][1]
        bad += not ok
    print(f"random graphs: {count} x 4 settings, mismatches {bad}, {time.time() - t0:.1f}s", flush=True)
    return bad


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config2", type=int, default=500)
    ap.add_argument("--config4", type=int, default=10)
    ap.add_argument("--graphs", type=int, default=200)
    a = ap.parse_args()
    bad = resident(P.Generator("uniform", n=1_000_000, deg=8, seed=1111_0627), a.config2, "config 2")
    bad += resident(P.Generator("powerlaw-hubs", n=64_000_000, deg=8, dmax=1 << 20, seed=1111_0627),
                    a.config4, "config 4")
    bad += graphs(a.graphs)
    print("TOTAL mismatches", bad)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
