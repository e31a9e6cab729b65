"""Reference outputs for BASELINE config 4 (and 5, given the memory) at its
FULL size.

    python tests/golden/make_config_golden_full.py --configs 4 --spill /tmp/ocm_spill
    python tests/golden/make_config_golden_full.py --merge

Same recipe as make_config_golden.py (the oracle's generators at bench.py's
seed, the UNMODIFIED reference library oracle/_ref, ocm::solve,
proj/src/solve.cpp:198, lane howard = run_howard_seq, solve.cpp:43), with
three changes for the size: the graph is built once and min and max are
solved concurrently on two threads over it (ocm::solve only reads the
Graph); --spill writes the generated edge arrays to disk and hands the
reference memory-mapped copies, so the resident peak is the reference's own
Graph plus the EdgeInput copy its build_graph makes (~40 B/edge: 40 GB for
config 4, 80 GB for config 5 -- config 4 fits this 62 GB build container,
config 5 does not); results are written after every solve. Measured: the
reference needs ~35 min (min, 24 passes) and ~70 min (max, 45 passes) for
config 4 at ~1.1*10^7 edge-passes/s; its howard-par lane on 16 host threads
did not finish the min solve within 50 minutes on the GPU box (a 1-hour
call limit), so the sequential lane is the one recorded.
"""
from __future__ import annotations

import argparse
import json
import os
import resource
import sys
import threading
import time

import numpy as np

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


def spill(arrays, where):
    """Write the arrays to disk and return read-only memory maps of them."""
    os.makedirs(where, exist_ok=True)
    out = []
    for i, a in enumerate(arrays):
        path = os.path.join(where, f"a{i}.npy")
        np.save(path, a)
        out.append(np.load(path, mmap_mode="r"))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="4")
    ap.add_argument("--out", default=os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                  "config_golden_full.json"))
    ap.add_argument("--merge", action="store_true", help="merge --out into config_golden.json")
    ap.add_argument("--lane", default="howard", choices=["howard", "howard-par"])
    ap.add_argument("--spill", default=None, help="directory for memory-mapped edge arrays")
    ap.add_argument("--mem-gb", type=int, default=58)
    a = ap.parse_args()
    if a.merge:
        with open(OUT) as f:
            gold = json.load(f)
        with open(a.out) as f:
            full = json.load(f)
        for k, v in full["configs"].items():
            if v["results"]:  # objectives still running are simply absent
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
    lock = threading.Lock()
    lane = {"howard": "howard (run_howard_seq, proj/src/solve.cpp:43)",
            "howard-par": f"howard-par (HowardPar, proj/src/solve.cpp:57; {os.cpu_count()} host cores)"}
    for cfg in a.configs.split(","):
        c = FULL[cfg]
        t0 = time.time()
        n, s, d, w = graph(c)
        ent = out["configs"].setdefault(cfg, {"results": {}})
        ent.update({"spec": c, "lane": lane[a.lane], "n": int(n), "m": int(len(s)),
                    "sha256": graph_sha(n, s, d, w)})
        if a.spill:
            s, d, w = spill((s, d, w), a.spill)
        t1 = time.time()
        g = O.RefGraph(n, s, d, w)
        del s, d, w
        print(cfg, f"n={n} m={ent['m']} gen+sha {t1 - t0:.0f}s build {time.time() - t1:.0f}s",
              flush=True)

        def one(objective):
            t0 = time.time()
            r = g.solve(a.lane, objective, "tarjan")
            res = {"has_cycle": r.has_cycle, "exact": r.exact, "mu_num": r.mu_num,
                   "mu_den": r.mu_den, "mu": r.mu, "cycle": [int(x) for x in r.cycle],
                   "outer_iters": r.outer_iters, "spf_passes": r.spf_passes,
                   "regions": r.regions, "trivial_regions": r.trivial_regions,
                   "nontrivial_regions": r.regions - r.trivial_regions,
                   "ref_solve_ms": r.solve_ms, "ref_wall_s": time.time() - t0}
            with lock:
                ent["results"][objective] = res
                with open(a.out, "w") as f:
                    json.dump(out, f, indent=1)
                print(cfg, objective, f"{r.mu_num}/{r.mu_den}", r.spf_passes, r.regions,
                      f"{r.solve_ms / 1e3:.0f} s", flush=True)

        ts = [threading.Thread(target=one, args=(o,)) for o in ("min", "max")
              if o not in ent["results"]]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        del g


if __name__ == "__main__":
    main()
