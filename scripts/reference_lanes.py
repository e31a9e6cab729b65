"""Which of the reference's own CPU lanes is fastest on the benchmark graph?
Times ocm::solve (oracle/_ref: the unmodified reference compiled in place)
with lane howard (run_howard_seq, single thread) and lane howard-par with
the seq schedule and with the par schedule on every host thread, on the
uniform generator (bench.py's seed), min objective.

usage: python scripts/reference_lanes.py [n] [--skip-par-seq]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 250_000
cpus = len(os.sched_getaffinity(0))
print(f"# reference lanes, uniform n={n} deg 8 (bench.py seed), min objective; host cpus {cpus}")
s, d, w = O.generate_uniform(n, 8, 1, 100, 1111_0627)
runs = [("howard", "seq", 1)]
if "--skip-par-seq" not in sys.argv:
    runs.append(("howard-par", "seq", 1))
runs += [("howard-par", "par", cpus), ("howard-par", "par", cpus)]
for algo, sched, workers in runs:
    r = O.ref_solve(n, s, d, w, algo, "min", "tarjan", sched, workers)
    print(f"{algo} schedule={sched} workers={workers} solve_ms={r.solve_ms:.1f} "
          f"spf_passes={r.spf_passes} mu={r.mu_num}/{r.mu_den}", flush=True)
