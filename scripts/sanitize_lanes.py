"""Small solves over every device lane, for compute-sanitizer (memcheck,
racecheck, synccheck, initcheck):

    compute-sanitizer --tool racecheck python scripts/sanitize_lanes.py [lane ...]

Lanes: exact (uniform + power-law with the heavy path), float, sccoff,
staged (TMA-staged improvement pass forced on), wide (128-bit keys forced
on; and a weight of 2^40), hot (shared-memory hub table forced on), csr
(ocm_solve_csr from pageable arrays: the staging ring), certify, sharded,
fused, cbits (connected-vertex bitmap forced on), heavyattach (block-
cooperative attach of high-degree pending vertices). Each checks its answer against the oracle or the plain exact lane."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
import paper_1111_0627_b200 as P  # noqa: E402

LANES = sys.argv[1:] or ["exact", "float", "sccoff", "staged", "wide", "hot", "csr", "certify",
                         "sharded", "fused", "cbits", "heavyattach"]


def check(g, opt, env=None):
    for k, v in (env or {}).items():
        os.environ[k] = v
    try:
        s = P.Session(g, opt)
        sol = s.solve()
        s.values()
    finally:
        for k in (env or {}):
            os.environ.pop(k, None)
    src, dst, w = g.edges()
    ref = O.oracle_solve(g.n, src, dst, w, opt.objective, opt.scc)
    assert sol.has_cycle == ref.has_cycle and sol.cycle_vertices == ref.cycle, (opt, env)
    if sol.exact:
        assert (sol.mu_exact.numerator, sol.mu_exact.denominator) == (ref.mu_num, ref.mu_den)
    return s


uni = P.generate(P.Generator("uniform", n=3000, deg=8, seed=1))
plaw = P.generate(P.Generator("powerlaw-hubs", n=3000, deg=4, dmax=2000, seed=2))
for lane in LANES:
    for objective in ("min", "max"):
        o = P.SolveOptions(objective=objective)
        if lane == "exact":
            check(uni, o)
            check(plaw, o, {"OCM_HEAVY_DEG": "16"})
        elif lane == "float":
            s, d, w = uni.edges()
            check(P.build_graph(uni.n, (s, d, w / 8 + 0.125)), o)
        elif lane == "sccoff":
            check(uni, P.SolveOptions(objective=objective, scc="off"))
        elif lane == "staged":
            check(plaw, o, {"OCM_STAGED": "1", "OCM_HEAVY_DEG": "16"})
            check(uni, o, {"OCM_STAGED": "1"})
        elif lane == "wide":
            check(uni, o, {"OCM_WIDE": "1"})
            s, d, w = uni.edges()
            w2 = w.copy()
            w2[::7] *= 2.0 ** 33
            check(P.build_graph(uni.n, (s, d, w2)), o)
        elif lane == "hot":
            check(plaw, o, {"OCM_HOT": "1", "OCM_HOT_SLOTS": "64"})
        elif lane == "csr":
            idx, t, w = uni.csr()
            sol = P.solve_csr(uni.n, idx.astype(np.uint32), t, w, o)
            assert sol.mu_exact == P.solve(uni, o).mu_exact
            # int32 narrowing of pageable weights, and its fallback
            wf = w.copy()
            wf[-1] = 2.5
            sol = P.solve_csr(uni.n, idx.astype(np.uint32), t, wf, o)
            assert not sol.exact
        elif lane == "cbits":
            check(uni, o, {"OCM_CBITS_MIN_N": "0"})
            check(plaw, o, {"OCM_CBITS_MIN_N": "0"})
            s, d, w = plaw.edges()
            check(P.build_graph(plaw.n, (s, d, w / 8 + 0.125)), o, {"OCM_CBITS_MIN_N": "0"})
        elif lane == "heavyattach":
            dense = P.generate(P.Generator("powerlaw", n=1500, deg=64, dmax=1500, seed=3))
            check(dense, o)
            check(dense, o, {"OCM_CBITS_MIN_N": "0"})
        elif lane == "certify":
            s = check(uni, o)
            c = s.certify()
            assert c["key_violations"] == c["policy_violations"] == c["cycle_violations"] == 0
        elif lane in ("sharded", "fused"):
            from paper_1111_0627_b200.sharded import (LocalComm, ShardSession, connect_local,
                                                      solve_fused, solve_sharded)
            shards = [ShardSession(uni, o, r, 2) for r in range(2)]
            if lane == "fused":
                os.environ["OCM_GRID"] = str(148 * 4 // 2)
                connect_local(shards)
                sols = solve_fused(shards)
            else:
                sols = solve_sharded(shards, LocalComm())
            ref = P.solve(uni, o)
            assert all(x.mu_exact == ref.mu_exact for x in sols)
    print(f"{lane}: ok", flush=True)
