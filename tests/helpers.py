"""Shared checks for the parity tests (test infrastructure)."""
from __future__ import annotations

import json
import os
from fractions import Fraction

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden.json")


def golden_cases():
    with open(GOLDEN) as f:
        return json.load(f)["cases"]


def case_arrays(case):
    return (np.array(case["src"], np.uint32), np.array(case["dst"], np.uint32),
            np.array(case["w"], np.float64))


def random_graph(rng, max_n=10, wlo=-9, whi=9, deg_cap=4):
    n = int(rng.integers(1, max_n + 1))
    m = int(rng.integers(0, deg_cap * n + 1))
    return (n, rng.integers(0, n, m).astype(np.uint32), rng.integers(0, n, m).astype(np.uint32),
            rng.integers(wlo, whi + 1, m).astype(np.float64))


def is_closed_walk(n, src, dst, cycle):
    """Every consecutive pair of the cycle (cyclically) is an edge of the graph."""
    if not cycle:
        return False
    edges = set(zip(src.tolist(), dst.tolist()))
    return all((cycle[i], cycle[(i + 1) % len(cycle)]) in edges for i in range(len(cycle)))


def cycle_mean_exact(src, dst, w, cycle, objective="min"):
    """Best mean achievable along the vertex cycle using the cheapest (min) or
    dearest (max) parallel edge between consecutive vertices."""
    best = {}
    for u, v, x in zip(src.tolist(), dst.tolist(), w.tolist()):
        k = (u, v)
        if k not in best:
            best[k] = x
        else:
            best[k] = min(best[k], x) if objective == "min" else max(best[k], x)
    tot = sum(Fraction(best[(cycle[i], cycle[(i + 1) % len(cycle)])]) for i in range(len(cycle)))
    return tot / len(cycle)
