"""Product side of tests/golden/make_config_golden_full.py, on the GPU box:
the product's host generator's SHA-256 of configs 4/5 (must equal the
oracle's) and the device solve of the HBM-generated graph (bench.py's path),
min and max, as one JSON line per config."""
import hashlib
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1111_0627_b200 as P  # noqa: E402

SEED = 1111_0627
FULL = {"4": dict(kind="powerlaw-hubs", n=64_000_000, deg=8, dmax=1 << 20),
        "5": dict(kind="uniform", n=250_000_000, deg=8)}
for cfg in sys.argv[1].split(","):
    c = FULL[cfg]
    spec = P.Generator(c["kind"], n=c["n"], deg=c["deg"], dmax=c.get("dmax", 0), wlo=1, whi=100,
                       seed=SEED)
    g = P.generate(spec)
    h = hashlib.sha256()
    h.update(np.uint64(g.n).tobytes())
    for a in g.edges():
        h.update(np.ascontiguousarray(a).tobytes())
    del g
    res = {}
    for objective in ("min", "max"):
        s = P.Session.generated(spec, P.SolveOptions(algo="howard", objective=objective))
        sol = s.solve()
        cert = s.certify()
        res[objective] = {"mu": f"{sol.mu_exact.numerator}/{sol.mu_exact.denominator}",
                          "cycle_len": len(sol.cycle_vertices), "cycle_head": sol.cycle_vertices[:8],
                          "outer_iters": sol.stats.outer_iters, "spf_passes": sol.stats.spf_passes,
                          "regions": sol.stats.regions, "cert": cert}
        del s
    print(json.dumps({"config": cfg, "sha256": h.hexdigest(), "device": res}), flush=True)
