"""CPU: pin the C oracle (oracle/ocm_oracle.c) against the reference's own
outputs (golden vectors from tests/golden/make_golden.py) and against the
independent walk-length DP oracle (oracle.hpp:137 restated)."""
import numpy as np
import pytest

import oracle as O
from helpers import case_arrays, golden_cases, random_graph

CASES = golden_cases()


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_oracle_matches_reference_golden(case):
    n = case["n"]
    src, dst, w = case_arrays(case)
    for key, ref in case["results"].items():
        objective, scc = key.split("/")
        got = O.oracle_solve(n, src, dst, w, objective, scc, values=(scc == "tarjan"))
        assert got.has_cycle == ref["has_cycle"], key
        if not ref["has_cycle"]:
            continue
        assert got.exact == ref["exact"]
        if ref["exact"]:
            assert (got.mu_num, got.mu_den) == (ref["mu_num"], ref["mu_den"]), key
        assert got.mu == ref["mu"], key
        assert got.cycle == ref["cycle"], key
        # howard-par lane stats (howard_par.hpp:566/606) and howard lane stats
        assert (got.outer_iters, got.spf_passes) == (ref["outer_iters"], ref["spf_passes"]), key
        assert (got.extra["outer_iters_seq"], got.extra["spf_passes_seq"]) == \
            (ref["seq_outer_iters"], ref["seq_spf_passes"]), key
        assert (got.regions, got.trivial_regions) == (ref["regions"], ref["trivial_regions"])
        if scc == "tarjan":
            assert got.succ_vertex.tolist() == ref["succ_vertex"], key
            if "value_key" in ref:
                k = got.wsum * got.lam_den - got.steps * got.lam_num
                assert k.tolist() == ref["value_key"], key
                assert got.lam_num.tolist() == ref["lam_num"]
                assert got.lam_den.tolist() == ref["lam_den"]
            else:
                np.testing.assert_array_equal(got.fval, np.array(ref["fval"]))


def test_golden_covers_reference_fixture_answers():
    """Answers the reference's own unit tests assert (test_howard.cpp,
    test_howard_par.cpp:428-455)."""
    by = {c["name"]: c for c in CASES}
    r = by["two_cycle"]["results"]["min/tarjan"]
    assert (r["mu_num"], r["mu_den"], r["cycle"]) == (3, 1, [0, 1])
    assert by["self_loop"]["results"]["min/tarjan"]["mu_num"] == 5
    assert by["unit_cycle_graph"]["results"]["min/tarjan"]["mu_num"] == 1
    r = by["two_component_graph"]["results"]["min/tarjan"]
    assert (r["mu_num"], r["mu_den"]) == (3, 2)
    assert not by["diamond_dag"]["results"]["min/tarjan"]["has_cycle"]
    r = by["four_component_graph"]["results"]["min/tarjan"]
    assert (r["mu_num"], r["mu_den"]) == (3, 2)


def test_oracle_agrees_with_dp_oracle():
    rng = np.random.default_rng(7)
    for _ in range(400):
        n, s, d, w = random_graph(rng, 10)
        hc, ex, num, den, mean = O.oracle_dp(n, s, d, w)
        got = O.oracle_solve(n, s, d, w)
        assert got.has_cycle == hc
        if hc:
            assert (got.mu_num, got.mu_den) == (num, den)


@pytest.mark.skipif(not O.ref_available(), reason="reference library not built here")
def test_oracle_matches_live_reference_medium():
    """When the reference library is present (build container), compare on
    larger generated graphs too."""
    for n, deg, seed in ((2000, 4, 3), (5000, 8, 4)):
        s, d, w = O.generate_uniform(n, deg, 1, 100, seed)
        a = O.oracle_solve(n, s, d, w, values=True)
        b = O.ref_solve(n, s, d, w, "howard")
        assert (a.mu_num, a.mu_den, a.cycle) == (b.mu_num, b.mu_den, b.cycle)
        v = O.ref_values(n, s, d, w)
        assert ((a.wsum * a.lam_den - a.steps * a.lam_num) ==
                (v.wsum * v.lam_den - v.steps * v.lam_num)).all()
