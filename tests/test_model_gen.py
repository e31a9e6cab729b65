"""Model generator (proj/include/ocm/model_gen.hpp) against the reference.

CPU: the library's generate_model reproduces the reference's composite state
spaces bit for bit (golden digests of the unmodified reference,
tests/golden/make_model_golden.py) and its error contract. GPU: the device
lane solves the generated models to the reference's optimal cycle means.
"""
import hashlib
import json
import os

import numpy as np
import pytest

import oracle as O
import paper_1111_0627_b200 as P

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "model_golden.json")))


def scenario(kind):
    if kind == "worker":
        return P.worker_scenario()
    if kind == "server":
        return P.server_scenario()
    return P.loop_scenario(GOLD["loop_costs"])


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("case", GOLD["cases"], ids=[f"{c['kind']}-{c['clients']}" for c in GOLD["cases"]])
def test_model_matches_reference(case):
    g = P.generate_model(scenario(case["kind"]), case["clients"])
    assert (g.n, g.m) == (case["n"], case["m"])
    s, d, w = g.edges()
    assert (digest(s), digest(d), digest(w)) == (case["src"], case["dst"], case["w"])
    assert g.integer_exact


def test_model_errors():
    with pytest.raises(P.StructuralError, match=GOLD["too_large_message"]):
        P.generate_model(P.server_scenario(), 19)
    with pytest.raises(ValueError, match="at least one state and one client"):
        P.generate_model(P.server_scenario(), 0)
    bad = P.Scenario("bad", 2, [P.Transition(0, 5, 1)])
    with pytest.raises(ValueError, match="missing state"):
        P.generate_model(bad, 2)
    srv = P.Scenario("srv", 2, [P.Transition(0, 1, 1, acquires=True)])
    with pytest.raises(ValueError, match="server-free"):
        P.generate_model(srv, 2)
    with pytest.raises(ValueError, match="64 bits"):
        P.generate_model(P.loop_scenario([1] * 5), 30)
    with pytest.raises(ValueError, match="at least one transition"):
        P.loop_scenario([])


def test_model_beyond_reference_bound():
    # the library's own bound is a parameter; growth is monotone in clients
    a = P.generate_model(P.worker_scenario(), 6)
    b = P.generate_model(P.worker_scenario(), 7, max_states=10_000)
    assert b.n == 3 * a.n == 2187


@pytest.mark.gpu
@pytest.mark.parametrize("case", [c for c in GOLD["cases"] if "min" in c],
                         ids=[f"{c['kind']}-{c['clients']}" for c in GOLD["cases"] if "min" in c])
def test_model_solve_matches_reference(case):
    g = P.generate_model(scenario(case["kind"]), case["clients"])
    for obj in ("min", "max"):
        sol = P.solve(g, P.SolveOptions(objective=obj))
        num, den, cyc, clen = case[obj]
        assert sol.has_cycle
        assert (sol.mu_exact.numerator, sol.mu_exact.denominator) == (num, den), obj
        assert len(sol.cycle_vertices) == clen and sol.cycle_vertices[:64] == cyc, obj


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("scenario,clients", [("server", 3), ("server", 9), ("worker", 7)])
def test_oracle_model_generator_matches_reference(scenario, clients):
    """oracle/ocm_oracle.c oc_generate_model (the restatement used for graphs
    beyond the reference's 5*10^6-state bound) equals the reference's
    generate_model edge for edge."""
    n, s, d, w = O.generate_model(scenario, clients)
    nr, sr, dr, wr = O.ref_generate_model(scenario, clients)
    assert n == nr and np.array_equal(s, sr) and np.array_equal(d, dr) and np.array_equal(w, wr)


@pytest.mark.parametrize("kind", ["powerlaw", "powerlaw-hubs", "powerlaw-web"])
def test_oracle_powerlaw_generators_match_product(kind):
    q = {"powerlaw": 0, "powerlaw-hubs": 1, "powerlaw-web": 3}[kind]
    s, d, w = O.generate_powerlaw(50_000, 4, 5_000, 1, 100, 9, hubs=q)
    g = P.generate(P.Generator(kind, n=50_000, deg=4, dmax=5_000, seed=9))
    s2, d2, w2 = g.edges()
    assert np.array_equal(s, s2) and np.array_equal(d, d2) and np.array_equal(w, w2)
    indeg = np.bincount(d, minlength=50_000)
    if q:  # hub targets: in-degree tail exponent 3 (hubs) / ~2.14 (web)
        assert indeg.max() > (50 if q == 1 else 5000) * indeg.mean()
    else:
        assert indeg.max() < 10 * indeg.mean()
