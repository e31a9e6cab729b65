"""Reference outputs for BASELINE configs 4 and 5 at their FULL sizes.

Run on a large-memory host (the GPU box: ~40 B/edge for the reference's
Graph plus the EdgeInput copy its build_graph makes, 40 GB for config 4 and
80 GB for config 5 -- more than this build container's 62 GB):

    python tests/golden/make_config_golden_full.py --out gpurun_out/config_golden_full.json

then merge into tests/golden/config_golden.json with --merge.  Same recipe as
make_config_golden.py (oracle generators at bench.py's seed, the UNMODIFIED
reference library oracle/_ref, ocm::solve, proj/src/solve.cpp:198) except the
lane: howard-par (HowardPar on the BSP engine, proj/src/solve.cpp:57, all
host cores) instead of run_howard_seq, which at ~1.2*10^7 edge-passes/s would
need 1-3 h per objective.  Both graphs have exactly one non-trivial region,
so howard-par's statistics (max over regions) are those of the one region's
policy iteration, and the mean and cycle are the solve's result either way.
The graph is built once and min, max solved one after the other; results are
written after every solve so a cut-off run keeps what finished.
"""
from __future__ import annotations

import argparse
import json
import os
import resource
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import oracle as O  # noqa: E402
from make_config_golden import SEED, OUT, graph_sha  # noqa: E402

FULL = {
    "4": dict(kind="powerlaw-hubs", n=64_000_000, deg=8, dmax=1 << 20),
    "5": dict(kind="uniform", n=250_000_000, deg=8),
}


def graph(c):
    if c["kind"] == "uniform":
        s, d, w = O.generate_uniform(c["n"], c["deg"], 1, 100, SEED)
    else:
        s, d, w = O.generate_powerlaw(c["n"], c["deg"], c["dmax"], 1, 100, SEED, hubs=1)
    return c["n"], s, d, w


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="4,5")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "config_golden_full.json"))
    ap.add_argument("--merge", action="store_true", help="merge --out into config_golden.json")
    ap.add_argument("--mem-gb", type=int, default=170)
    a = ap.parse_args()
    if a.merge:
        with open(OUT) as f:
            gold = json.load(f)
        with open(a.out) as f:
            full = json.load(f)
        for k, v in full["configs"].items():
            if set(v["results"]) == {"min", "max"}:
                gold["configs"][k] = v
        with open(OUT, "w") as f:
            json.dump(gold, f, indent=1)
        print("merged", sorted(full["configs"]), "into", OUT)
        return
    # fail with MemoryError instead of driving the host out of memory
    resource.setrlimit(resource.RLIMIT_AS, (a.mem_gb << 30, a.mem_gb << 30))
    out = {"seed": SEED, "reference": "oracle/_ref (unmodified proj/src compiled in place)",
           "configs": {}}
    if os.path.exists(a.out):
        with open(a.out) as f:
            out = json.load(f)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    for cfg in a.configs.split(","):
        c = FULL[cfg]
        t0 = time.time()
        n, s, d, w = graph(c)
        ent = out["configs"].setdefault(cfg, {"results": {}})
        ent.update({"spec": c, "lane": "howard-par (HowardPar, proj/src/solve.cpp:57; "
                    f"{os.cpu_count()} host cores)", "n": int(n), "m": int(len(s)),
                    "sha256": graph_sha(n, s, d, w)})
        t1 = time.time()
        g = O.RefGraph(n, s, d, w)
        del s, d, w
        print(cfg, f"n={n} m={ent['m']} gen+sha {t1 - t0:.0f}s build {time.time() - t1:.0f}s",
              flush=True)
        for objective in ("min", "max"):
            if objective in ent["results"]:
                continue
            t0 = time.time()
            r = g.solve("howard-par", objective, "tarjan")
            res = {"has_cycle": r.has_cycle, "exact": r.exact, "mu_num": r.mu_num,
                   "mu_den": r.mu_den, "mu": r.mu, "cycle": [int(x) for x in r.cycle],
                   "outer_iters": r.outer_iters, "spf_passes": r.spf_passes,
                   "regions": r.regions, "trivial_regions": r.trivial_regions,
                   "nontrivial_regions": r.regions - r.trivial_regions,
                   "ref_solve_ms": r.solve_ms, "ref_wall_s": time.time() - t0}
            ent["results"][objective] = res
            with open(a.out, "w") as f:
                json.dump(out, f, indent=1)
            print(cfg, objective, f"{r.mu_num}/{r.mu_den}", r.spf_passes, r.regions,
                  f"{r.solve_ms / 1e3:.0f} s", flush=True)
        del g


if __name__ == "__main__":
    main()
