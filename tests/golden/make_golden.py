"""Generate golden vectors from the UNMODIFIED reference library.

Run in the build container (needs /root/reference and `make -C oracle ref`):

    python tests/golden/make_golden.py

Writes tests/golden/golden.json. Each case stores its edge list (so the
fixture is self-contained and the reference is not needed at test time) and
what the reference's ocm::solve (proj/src/solve.cpp:198, lanes howard and
howard-par) and HowardPar's final value plane (proj/include/ocm/howard_par.hpp:544)
return for it. Values are stored as exact scalars value*den = wsum*den -
steps*num (integer graphs) or doubles (float graphs): the reference's
region-concurrent lane keeps a global plane parity, so a region that finished
early may export its quiet-pass plane, whose (wsum, steps) pairs differ from
the propagated ones while the scalar values are equal.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")


def fixtures():
    """The reference's hand fixtures, proj/tests/support/test_graphs.hpp."""
    return {
        "two_cycle": (2, [(0, 1, 2), (1, 0, 4)]),
        "self_loop": (1, [(0, 0, 5)]),
        "unit_cycle_graph": (4, [(0, 1, 1), (1, 2, 1), (2, 3, 1), (3, 0, 1), (1, 3, 1), (2, 0, 1)]),
        "two_component_graph": (4, [(0, 1, 2), (1, 0, 4), (2, 3, 1), (3, 2, 2), (1, 2, 0)]),
        "diamond_dag": (4, [(0, 1, 1), (0, 2, 2), (1, 3, 3), (2, 3, -1)]),
        "four_component_graph": (7, [(0, 1, 1), (1, 4, 1), (4, 5, 2), (5, 1, 3), (1, 2, 0),
                                     (2, 3, 1), (3, 2, 2), (3, 6, 1), (5, 6, 4)]),
        # proj/tests/test_howard_par.cpp:315 (winning 2-cycle, losing 2-cycle, tail)
        "broadcast_restore": (5, [(0, 1, 1), (1, 0, 1), (2, 3, 3), (3, 2, 3), (4, 0, 0)]),
        # proj/tests/test_howard_par.cpp:158 (3-cycle with a 3-vertex tail)
        "cycle_with_tail": (6, [(0, 1, 1), (1, 2, 1), (2, 0, 1), (3, 0, 1), (4, 3, 1), (5, 4, 1)]),
        "parallel_edges": (3, [(0, 1, 5), (0, 1, 1), (1, 2, 2), (2, 0, 3), (2, 0, -4), (1, 1, 7)]),
        "float_two_cycle": (2, [(0, 1, 2.5), (1, 0, 4.25)]),
    }


def random_cases(rng, count, max_n, wlo, whi, deg_cap, dyadic_every=0, sc=False):
    out = []
    for i in range(count):
        n = int(rng.integers(1, max_n + 1))
        if sc:  # strongly connected: permutation cycle + extras (test_graphs.hpp:97)
            perm = rng.permutation(n)
            edges = [(int(perm[j]), int(perm[(j + 1) % n]), int(rng.integers(wlo, whi + 1)))
                     for j in range(n)]
            extra = int(rng.integers(0, deg_cap * n + 1))
        else:
            edges = []
            extra = int(rng.integers(0, deg_cap * n + 1))
        for _ in range(extra):
            edges.append((int(rng.integers(0, n)), int(rng.integers(0, n)),
                          int(rng.integers(wlo, whi + 1))))
        if dyadic_every and i % dyadic_every == 0:
            edges = [(u, v, w / 8 + 0.125) for (u, v, w) in edges]
        out.append((n, edges))
    return out


def record(name, n, edges):
    src = np.array([e[0] for e in edges], np.uint32)
    dst = np.array([e[1] for e in edges], np.uint32)
    w = np.array([e[2] for e in edges], np.float64)
    case = {"name": name, "n": n, "src": src.tolist(), "dst": dst.tolist(), "w": w.tolist(),
            "results": {}}
    for objective in ("min", "max"):
        for scc in ("tarjan", "off"):
            if n == 0:
                continue
            seq = O.ref_solve(n, src, dst, w, "howard", objective, scc)
            par = O.ref_solve(n, src, dst, w, "howard-par", objective, scc)
            assert (seq.has_cycle, seq.mu_num, seq.mu_den, seq.mu, seq.cycle) == \
                (par.has_cycle, par.mu_num, par.mu_den, par.mu, par.cycle)
            r = {"has_cycle": par.has_cycle, "exact": par.exact, "mu_num": par.mu_num,
                 "mu_den": par.mu_den, "mu": par.mu, "cycle": par.cycle,
                 "outer_iters": par.outer_iters, "spf_passes": par.spf_passes,
                 "regions": par.regions, "trivial_regions": par.trivial_regions,
                 "seq_outer_iters": seq.outer_iters, "seq_spf_passes": seq.spf_passes}
            if scc == "tarjan":
                v = O.ref_values(n, src, dst, w, objective)
                if par.exact or (len(w) and np.all(np.floor(w) == w)):
                    # exact Python integers: with weights up to 2^52 the
                    # products leave int64 (the wide device lane's range)
                    key = [int(a) * int(b) - int(c) * int(d) for a, b, c, d in
                           zip(v.wsum, v.lam_den, v.steps, v.lam_num)]
                    r["value_key"] = key
                    r["lam_num"] = v.lam_num.tolist()
                    r["lam_den"] = v.lam_den.tolist()
                else:
                    r["fval"] = v.fval.tolist()
                    r["lam_f"] = v.lam_f.tolist()
                r["succ_vertex"] = [int(x) for x in v.succ_vertex]
            case["results"][f"{objective}/{scc}"] = r
    return case


def main():
    if not O.ref_available():
        sys.exit("reference library not built: run `make -C oracle ref` first")
    cases = []
    for name, (n, edges) in fixtures().items():
        cases.append(record(name, n, edges))
    rng = np.random.default_rng(20111106)
    for i, (n, e) in enumerate(random_cases(rng, 120, 10, -9, 9, 4, dyadic_every=5)):
        cases.append(record(f"random_{i}", n, e))
    for i, (n, e) in enumerate(random_cases(rng, 40, 12, -9, 9, 3, sc=True)):
        cases.append(record(f"random_sc_{i}", n, e))
    for i, (n, e) in enumerate(random_cases(rng, 12, 60, 1, 100, 3)):
        cases.append(record(f"medium_{i}", n, e))
    # the reference's full ExactMode range (graph.cpp:15: integral |w| < 2^53):
    # weights of 2^40 and 2^48 -- the device's wide exact lane (2^48 keeps the
    # Hamiltonian weight 2n(max|w|+1)+1 of --scc off below 2^53 for n <= 8)
    wrng = np.random.default_rng(53)
    for i, (n, e) in enumerate(random_cases(wrng, 24, 10, -(1 << 40), 1 << 40, 4)):
        cases.append(record(f"wide40_{i}", n, e))
    for i, (n, e) in enumerate(random_cases(wrng, 12, 8, -(1 << 48) + 1, (1 << 48) - 1, 3, sc=True)):
        cases.append(record(f"wide48_sc_{i}", n, e))
    with open(OUT, "w") as f:
        json.dump({"generator": "tests/golden/make_golden.py",
                   "reference": "proj/src/solve.cpp via oracle/_ref/libocm_ref.so",
                   "cases": cases}, f, separators=(",", ":"))
    print(f"wrote {len(cases)} cases to {OUT} ({os.path.getsize(OUT)} bytes)")


if __name__ == "__main__":
    main()
