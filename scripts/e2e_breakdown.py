"""Wall-time breakdown of the end-to-end calls on a host graph: ocm_solve (the
library's own pinned graph) and ocm_solve_csr (the reference's CSR arrays in
pageable memory, staged). Run with OCM_PREP_TIMING=1 for the per-stage split
of the upload / validation / region split / packing.

usage: python scripts/e2e_breakdown.py [n] [--model CLIENTS]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1111_0627_b200 as P  # noqa: E402

if "--model" in sys.argv:
    g = P.generate_model(P.server_scenario(), int(sys.argv[sys.argv.index("--model") + 1]),
                         max_states=1 << 31)
else:
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
    g = P.generate_uniform(n, 8, 1, 100, 1111_0627)
idx64, tgt, w = g.csr()
idx = idx64.astype(np.uint32)
# ocm_solve pins the graph's own arrays (cudaHostRegister); the CSR leg gets
# private pageable copies, as a reference ocm::Graph would be
tgt, w = tgt.copy(), w.copy()
# host memcpy rate of this box (pageable -> pageable), for reference
buf = np.empty_like(w)
t0 = time.perf_counter()
np.copyto(buf, w)
print(f"host_memcpy_GBps={w.nbytes / (time.perf_counter() - t0) / 1e9:.1f}", file=sys.stderr)
P.solve(g)  # pins the host arrays, warms the pool
P.solve_csr(g.n, idx, tgt, w)  # starts the staging ring
for name, call in (("ocm_solve", lambda: P.solve(g, P.SolveOptions(objective="min"))),
                   ("ocm_solve_csr", lambda: P.solve_csr(g.n, idx, tgt, w, P.SolveOptions(objective="min")))):
    for _ in range(3):
        t0 = time.perf_counter()
        s = call()
        t1 = time.perf_counter()
        print(f"{name}: e2e_ms={1e3 * (t1 - t0):.3f} device_ms={s.stats.device_ms:.3f} "
              f"prep_ms={s.stats.host_prep_ms:.3f} h2d={s.stats.h2d_bytes}", file=sys.stderr)
# the bench's e2e loop: min then max per step, timed per call
for step in range(4):
    for o in ("min", "max"):
        t0 = time.perf_counter()
        s = P.solve_csr(g.n, idx, tgt, w, P.SolveOptions(objective=o))
        t1 = time.perf_counter()
        print(f"step {step} {o}: e2e_ms={1e3 * (t1 - t0):.3f} device_ms={s.stats.device_ms:.3f} "
              f"prep_ms={s.stats.host_prep_ms:.3f}", file=sys.stderr)
