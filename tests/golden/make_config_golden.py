"""Reference outputs on the BASELINE configurations' own graphs.

Run in the build container (needs /root/reference and `make -C oracle`):

    python tests/golden/make_config_golden.py [--jobs 8]

Builds each workload with the ORACLE's bit-identical generators (no import of
the product package) at bench.py's seed, solves it with the UNMODIFIED
reference library (oracle/_ref: ocm::solve, proj/src/solve.cpp:198, lane
howard = run_howard_seq, solve.cpp:43, which is also what the reference CLI
runs by default), min and max, and writes tests/golden/config_golden.json:
per config the graph's SHA-256 (so a test can prove it solved the same
graph), region counts, and per objective mu as a rational, the optimal
cycle, outer iterations and improvement passes, plus the reference's solve
wall time on this container (8 cores; informational).

Configs (BASELINE.json "configs"; bench.py CONFIGS):
  1   uniform 10^4 x 4
  2   uniform 10^6 x 8 (the metric's workload)
  3   server scenario, 19 clients (1.05*10^7 states, 2.0*10^8 edges; the
      reference's generator stops at 5*10^6 states, model_gen.hpp:65, so the
      graph comes from the oracle's restatement of generate_model and is fed
      to the reference's solve directly)
  4s  power-law in+out-degree ("powerlaw-hubs") at n = 10^6 -- config 4's
      generator at a size the reference solves in about a minute. Config 4
      itself (6.4*10^7 vertices, ~10^9 edges) is written by
      make_config_golden_full.py (memory-mapped inputs, ~1.5-3 h per
      objective); config 5 (2*10^9 edges, ~80 GB in the reference's
      representation) fits neither this container nor the time budget.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "config_golden.json")
SEED = 1111_0627  # bench.py SEED

CONFIGS = {
    "1": dict(kind="uniform", n=10_000, deg=4),
    "2": dict(kind="uniform", n=1_000_000, deg=8),
    "3": dict(kind="model", scenario="server", clients=19),
    "4s": dict(kind="powerlaw-hubs", n=1_000_000, deg=8, dmax=1 << 20),
    # the same config-2 graph through the reference's other options: float
    # weights (w/8 + 1/8: FloatMode, exact dyadic inputs) and --scc off
    # (the Hamiltonian-augmented single region, solve.cpp:48)
    "2f": dict(kind="uniform", n=1_000_000, deg=8, weights="float"),
    "2off": dict(kind="uniform", n=1_000_000, deg=8, scc="off"),
}


def graph(cfg):
    c = CONFIGS[cfg]
    if c["kind"] == "uniform":
        s, d, w = O.generate_uniform(c["n"], c["deg"], 1, 100, SEED)
        if c.get("weights") == "float":
            w = w / 8 + 0.125
        return c["n"], s, d, w
    if c["kind"] == "model":
        return O.generate_model(c["scenario"], c["clients"])
    s, d, w = O.generate_powerlaw(c["n"], c["deg"], c["dmax"], 1, 100, SEED,
                                  hubs={"powerlaw": 0, "powerlaw-hubs": 1, "powerlaw-web": 3}[c["kind"]])
    return c["n"], s, d, w


def graph_sha(n, s, d, w):
    h = hashlib.sha256()
    h.update(np.uint64(n).tobytes())
    for a in (s, d, w):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def solve(job):
    cfg, objective = job
    n, s, d, w = graph(cfg)
    t0 = time.time()
    r = O.ref_solve(n, s, d, w, "howard", objective, CONFIGS[cfg].get("scc", "tarjan"))
    wall = time.time() - t0
    trace = None
    if CONFIGS[cfg].get("scc") == "off":
        # one region by construction: the reference's lambda after every
        # policy iteration (HowardPar::run(trace), howard_par.hpp:588)
        tr = O.ref_lambda_trace(n, s, d, w, objective, "off")
        trace = [[x.numerator, x.denominator] if hasattr(x, "numerator") else x for x in tr]
    return cfg, objective, {
        "has_cycle": r.has_cycle, "exact": r.exact, "mu_num": r.mu_num, "mu_den": r.mu_den,
        "mu": r.mu, "cycle": [int(x) for x in r.cycle], "outer_iters": r.outer_iters,
        "spf_passes": r.spf_passes, "regions": r.regions, "trivial_regions": r.trivial_regions,
        "ref_solve_ms": r.solve_ms, "ref_wall_s": wall,
        **({"lambda_trace": trace} if trace is not None else {})}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--jobs", type=int, default=min(8, os.cpu_count() or 1))
    ap.add_argument("--configs", default=",".join(CONFIGS))
    a = ap.parse_args()
    cfgs = a.configs.split(",")
    out = {"seed": SEED, "reference": "oracle/_ref (unmodified proj/src compiled in place)",
           "lane": "howard (run_howard_seq, proj/src/solve.cpp:43)", "configs": {}}
    if os.path.exists(OUT):
        with open(OUT) as f:
            out["configs"] = json.load(f).get("configs", {})
    for cfg in cfgs:
        n, s, d, w = graph(cfg)
        out["configs"][cfg] = {"spec": CONFIGS[cfg], "n": int(n), "m": int(len(s)),
                               "sha256": graph_sha(n, s, d, w), "results": {}}
        del s, d, w
    jobs = [(c, o) for c in cfgs for o in ("min", "max")]
    with ProcessPoolExecutor(a.jobs) as ex:
        for cfg, objective, res in ex.map(solve, jobs):
            # one non-trivial region => howard-par's stats (max over regions)
            # equal howard's (sum over regions)
            res["nontrivial_regions"] = res["regions"] - res["trivial_regions"]
            out["configs"][cfg]["results"][objective] = res
            print(cfg, objective, f"{res['mu_num']}/{res['mu_den']}", res["spf_passes"],
                  f"{res['ref_solve_ms'] / 1e3:.1f} s", flush=True)
    with open(OUT, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
