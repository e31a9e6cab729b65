"""A/B of library variants (scripts/build_variant.sh) on the bench graphs:
median device ms of min and max solves per variant, variants interleaved
A B A B ... in fresh processes (OCM_LIB selects the library).

    python scripts/ab_variants.py --variants base,gbar --n 1000000 --deg 8 --rounds 3
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import json, os, statistics, sys
sys.path.insert(0, os.environ["ROOT"])
import paper_1111_0627_b200 as P
n, deg, k = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
kind = sys.argv[4]
spec = P.Generator(kind, n=n, deg=deg, dmax=1 << 20, wlo=1, whi=100, seed=1111_0627)
out = {}
for o in ("min", "max"):
    s = P.Session.generated(spec, P.SolveOptions(objective=o))
    for _ in range(3):
        s.solve()
    ms = [s.solve().stats.device_ms for _ in range(k)]
    sol = s.solve()
    out[o] = {"ms": statistics.median(ms), "mu": str(sol.mu_exact), "passes": sol.stats.spf_passes}
print(json.dumps(out))
'''


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--variants", default="base")
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--deg", type=int, default=8)
    ap.add_argument("--kind", default="uniform")
    ap.add_argument("--solves", type=int, default=15)
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--env", default="", help="extra KEY=VAL,... for every child")
    a = ap.parse_args()
    res = {}
    for r in range(a.rounds):
        for v in a.variants.split(","):
            env = dict(os.environ, ROOT=ROOT)
            for kv in filter(None, a.env.split(",")):
                k, val = kv.split("=", 1)
                env[k] = val
            name = v
            if ":" in v:  # variant:KEY=VAL (an env-only variant of a library)
                v, kv = v.split(":", 1)
                k, val = kv.split("=", 1)
                env[k] = val
            if v != "base":
                env["OCM_LIB"] = os.path.join(ROOT, "paper_1111_0627_b200", "lib", f"libocm_b200_{v}.so")
            p = subprocess.run([sys.executable, "-c", CHILD, str(a.n), str(a.deg), str(a.solves), a.kind],
                               env=env, capture_output=True, text=True, timeout=900)
            if p.returncode:
                print(name, "FAILED", p.stderr[-2000:], flush=True)
                continue
            d = json.loads(p.stdout.strip().splitlines()[-1])
            res.setdefault(name, []).append(d)
            print(f"round {r} {name:>16}: min {d['min']['ms']:.3f} ms ({d['min']['mu']}, {d['min']['passes']})"
                  f"  max {d['max']['ms']:.3f} ms ({d['max']['mu']}, {d['max']['passes']})", flush=True)
    for name, ds in res.items():
        mn = sorted(d["min"]["ms"] for d in ds)[len(ds) // 2]
        mx = sorted(d["max"]["ms"] for d in ds)[len(ds) // 2]
        print(f"== {name:>16}: min {mn:.3f}  max {mx:.3f}  sum {mn + mx:.3f} ms", flush=True)


if __name__ == "__main__":
    main()
