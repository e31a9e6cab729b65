"""Golden digests of the reference's model generator (run in the build container).

    python tests/golden/make_model_golden.py

Drives the UNMODIFIED reference's ocm::generate_model (proj/src/model_gen.cpp:90,
through oracle/_ref) for its three scenario constructors and records, per
(scenario, clients): n, m and SHA-256 digests of the edge arrays in edge-id
order, plus the reference's optimal min/max cycle means of the smaller models.
Writes tests/golden/model_golden.json.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "model_golden.json")
LOOP_COSTS = [1, 3, 2, 7, 5]


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    cases = []
    for kind, ks in (("worker", range(1, 11)), ("server", range(1, 13)), ("loop", range(1, 7))):
        for k in ks:
            n, s, d, w = O.ref_generate_model(kind, k, LOOP_COSTS if kind == "loop" else ())
            rec = {"kind": kind, "clients": k, "n": n, "m": int(len(s)), "src": digest(s),
                   "dst": digest(d), "w": digest(w)}
            if n <= 20000:
                for obj in ("min", "max"):
                    r = O.ref_solve(n, s, d, w, "howard", obj, "tarjan")
                    rec[obj] = [r.mu_num, r.mu_den, r.cycle[:64], len(r.cycle)]
            cases.append(rec)
    # the reference's bound: kMaxModelStates (model_gen.hpp:70)
    try:
        O.ref_generate_model("server", 19)
        bound = None
    except RuntimeError as e:
        bound = str(e).replace("reference: ", "")
    with open(OUT, "w") as f:
        json.dump({"loop_costs": LOOP_COSTS, "cases": cases, "too_large_message": bound}, f,
                  indent=0)
    print(f"wrote {len(cases)} model digests to {OUT}")


if __name__ == "__main__":
    main()
