"""GPU parity: the device lane (through the C-ABI) against the reference's
golden vectors and the C oracle, plus size-independent optimality
certificates at benchmark sizes. Bar: bit-exact rationals, cycles, policies
and scalar values on integer graphs; float graphs compare means and values
exactly too (same summation order as the reference) with a 1e-9 relative
fallback tolerance noted where used."""
from fractions import Fraction

import numpy as np
import pytest

import oracle as O
import paper_1111_0627_b200 as P
from helpers import case_arrays, cycle_mean_exact, golden_cases, is_closed_walk, random_graph

pytestmark = pytest.mark.gpu
CASES = golden_cases()
NONE = 0xFFFFFFFF


def run(n, src, dst, w, objective="min", scc="tarjan"):
    g = P.build_graph(n, (src, dst, w))
    s = P.Session(g, P.SolveOptions(objective=objective, scc=scc))
    sol = s.solve()
    return sol, s.values()


def check_against(sol, vals, ref, key_field="value_key"):
    assert sol.has_cycle == ref["has_cycle"]
    if not ref["has_cycle"]:
        return
    if ref["exact"]:
        assert sol.exact
        assert (sol.mu_exact.numerator, sol.mu_exact.denominator) == (ref["mu_num"], ref["mu_den"])
    assert sol.mu == ref["mu"]
    assert sol.cycle_vertices == ref["cycle"]
    assert (sol.stats.outer_iters, sol.stats.spf_passes) == (ref["outer_iters"], ref["spf_passes"])
    assert (sol.stats.regions, sol.stats.trivial_regions) == (ref["regions"], ref["trivial_regions"])
    if vals is not None and "succ_vertex" in ref:
        assert vals["succ_vertex"].tolist() == ref["succ_vertex"]
        if key_field in ref:
            assert vals["key_num"].tolist() == ref[key_field]
            assert vals["lam_num"].tolist() == ref["lam_num"]
            assert vals["lam_den"].tolist() == ref["lam_den"]
        elif "fval" in ref:
            np.testing.assert_array_equal(vals["fval"], np.array(ref["fval"]))


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_golden_howard_lane_stats(case):
    """algo=howard: the reference's sequential lane sums every region's outer
    iterations and improvement passes (src/solve.cpp:71-72); mu and the
    cycle are the same as howard-par's."""
    n = case["n"]
    src, dst, w = case_arrays(case)
    g = P.build_graph(n, (src, dst, w))
    for key, ref in case["results"].items():
        objective, scc = key.split("/")
        if "seq_outer_iters" not in ref:
            continue
        sol = P.solve(g, P.SolveOptions(algo="howard", objective=objective, scc=scc))
        assert sol.has_cycle == ref["has_cycle"]
        if ref["has_cycle"]:
            assert sol.cycle_vertices == ref["cycle"]
            assert sol.mu == ref["mu"]
        assert (sol.stats.outer_iters, sol.stats.spf_passes) == \
            (ref["seq_outer_iters"], ref["seq_spf_passes"]), key


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_golden(case):
    n = case["n"]
    src, dst, w = case_arrays(case)
    for key, ref in case["results"].items():
        objective, scc = key.split("/")
        sol, vals = run(n, src, dst, w, objective, scc)
        check_against(sol, vals if scc == "tarjan" else None, ref)


def oracle_record(n, src, dst, w, objective, scc):
    o = O.oracle_solve(n, src, dst, w, objective, scc, values=True)
    r = {"has_cycle": o.has_cycle, "exact": o.exact, "mu_num": o.mu_num, "mu_den": o.mu_den,
         "mu": o.mu, "cycle": o.cycle, "outer_iters": o.outer_iters, "spf_passes": o.spf_passes,
         "regions": o.regions, "trivial_regions": o.trivial_regions}
    if scc == "tarjan":
        r["succ_vertex"] = o.succ_vertex.tolist()
        if o.exact or (len(w) and np.all(np.floor(w) == w)):
            r["value_key"] = (o.wsum * o.lam_den - o.steps * o.lam_num).tolist()
            r["lam_num"] = o.lam_num.tolist()
            r["lam_den"] = o.lam_den.tolist()
        else:
            r["fval"] = o.fval.tolist()
    return r


def test_random_small_graphs_vs_oracle():
    rng = np.random.default_rng(1234)
    for it in range(250):
        n, s, d, w = random_graph(rng, 12)
        if it % 4 == 0:
            w = w / 8 + 0.125
        for objective in ("min", "max"):
            scc = "off" if it % 5 == 0 else "tarjan"
            sol, vals = run(n, s, d, w, objective, scc)
            check_against(sol, vals if scc == "tarjan" else None,
                          oracle_record(n, s, d, w, objective, scc))


@pytest.mark.parametrize("n,deg,seed", [(1000, 2, 1), (10000, 4, 2), (20000, 1, 5),
                                        (100000, 8, 3)])
def test_generated_graphs_vs_oracle(n, deg, seed):
    g = P.generate_uniform(n, deg, 1, 100, seed)
    s, d, w = g.edges()
    for objective in ("min", "max"):
        sess = P.Session(g, P.SolveOptions(objective=objective))
        sol = sess.solve()
        check_against(sol, sess.values(), oracle_record(n, s, d, w, objective, "tarjan"))


@pytest.mark.parametrize("kind,n,deg,seed", [("uniform", 20000, 4, 7), ("powerlaw", 20000, 3, 8),
                                             ("uniform", 3000, 2, 9)])
def test_blocked_improvement_vs_oracle(kind, n, deg, seed, monkeypatch):
    """The propagation-blocked improvement pass (OCM_PB=1, forced here with
    tiny target bins so every vertex block spans many bins) must choose the
    same policy as the direct pass: identical results and iteration counts."""
    gen = P.Generator(kind, n=n, deg=deg, dmax=256 if kind == "powerlaw" else 0, wlo=1, whi=100,
                      seed=seed)
    g = P.generate(gen)
    s, d, w = g.edges()
    for objective in ("min", "max"):
        monkeypatch.setenv("OCM_PB", "0")
        direct = P.Session(g, P.SolveOptions(objective=objective)).solve()
        monkeypatch.setenv("OCM_PB", "1")
        monkeypatch.setenv("OCM_PB_BIN", "64")
        sess = P.Session(g, P.SolveOptions(objective=objective))
        sol = sess.solve()
        check_against(sol, sess.values(), oracle_record(n, s, d, w, objective, "tarjan"))
        assert sol.stats.spf_passes == direct.stats.spf_passes
        assert sol.cycle_vertices == direct.cycle_vertices


@pytest.mark.parametrize("n", [60, 200, 300, 3000, 9000])
def test_long_winning_cycle(n):
    """Winning cycles of every size class of the vote tail: shared-memory
    values (one block), global-memory values (one block) and the grid-wide
    rounds (longer than small_wc)."""
    rng = np.random.default_rng(n)
    ring_s = np.arange(n, dtype=np.uint32)
    ring_d = ((ring_s + 1) % n).astype(np.uint32)
    ring_w = rng.integers(1, 4, n).astype(np.float64)  # mean < 4
    chord_s = rng.integers(0, n, 2 * n).astype(np.uint32)
    chord_d = rng.integers(0, n, 2 * n).astype(np.uint32)
    chord_w = np.full(2 * n, 1e6)  # any cycle through a chord is worse
    s = np.concatenate([ring_s, chord_s])
    d = np.concatenate([ring_d, chord_d])
    w = np.concatenate([ring_w, chord_w])
    sol, vals = run(n, s, d, w, "min")
    ref = oracle_record(n, s, d, w, "min", "tarjan")
    check_against(sol, vals, ref)
    assert len(sol.cycle_vertices) == n


@pytest.mark.parametrize("n,deg,objective,scc", [(5000, 3, "min", "tarjan"), (100000, 4, "min", "tarjan"),
                                                  (100000, 4, "max", "tarjan"), (20000, 3, "min", "off")])
def test_float_weights_generated(n, deg, objective, scc):
    """Float lane (non-integer weights): same summation order as the
    reference, so means and values compare exactly, up to 10^5 vertices."""
    g = P.generate_uniform(n, deg, -400, 400, 9)
    s, d, w = g.edges()
    w = w / 16.0 + 0.03125
    sol, vals = run(n, s, d, w, objective, scc)
    ref = oracle_record(n, s, d, w, objective, scc)
    assert not sol.exact
    check_against(sol, vals, ref)


def test_no_cycle_and_empty():
    sol, _ = run(4, np.array([0, 0, 1, 2], np.uint32), np.array([1, 2, 3, 3], np.uint32),
                 np.array([1, 2, 3, -1.0]))
    assert not sol.has_cycle and sol.stats.spf_passes == 0
    g = P.build_graph(0, [])
    assert not P.solve(g).has_cycle
    # edgeless graph (scc.cpp: every vertex its own trivial region)
    e = np.array([], np.uint32)
    sol, _ = run(5, e, e, np.array([], np.float64))
    assert not sol.has_cycle and sol.stats.trivial_regions == 5
    # a lone self-loop is a non-trivial singleton region: mu = its weight
    sol, _ = run(3, np.array([1], np.uint32), np.array([1], np.uint32), np.array([-7.0]))
    assert sol.has_cycle and sol.mu_exact == -7 and sol.cycle_vertices == [1]
    sol, _ = run(4, np.array([0, 0, 1, 2], np.uint32), np.array([1, 2, 3, 3], np.uint32),
                 np.array([1, 2, 3, -1.0]), scc="off")
    assert not sol.has_cycle


def test_session_resolve_is_deterministic():
    g = P.generate_uniform(50000, 8, 1, 100, 21)
    s = P.Session(g)
    a = s.solve()
    va = s.values()
    b = s.solve()
    vb = s.values()
    assert (a.mu_exact, a.cycle_vertices, a.stats.spf_passes) == \
        (b.mu_exact, b.cycle_vertices, b.stats.spf_passes)
    assert (va["key_num"] == vb["key_num"]).all()


def bellman_certificate(g, sol, vals, objective):
    """Size-independent optimality certificate. With K = value*den per vertex,
    every intra-component edge (v,t) satisfies K[v] <= K[t] + w*den - num with
    equality attained by some edge of every vertex (the Bellman equation of
    the final policy), so no cycle has mean below lambda in its component;
    the returned cycle is a closed walk of mean mu; mu = min over components."""
    from scipy.sparse import csr_matrix
    from scipy.sparse.csgraph import connected_components
    s, d, w = g.edges()
    if objective == "max":
        w = -w
    n = g.n
    ncomp, lab = connected_components(csr_matrix((np.ones(len(s)), (s, d)), shape=(n, n)),
                                      directed=True, connection="strong")
    intra = lab[s] == lab[d]
    K = vals["key_num"]
    num = vals["lam_num"]
    den = vals["lam_den"]
    s_, d_, w_ = s[intra], d[intra], w[intra].astype(np.int64)
    rhs = K[d_] + w_ * den[s_] - num[s_]
    assert (K[s_] <= rhs).all()
    best = np.full(n, np.iinfo(np.int64).max)
    np.minimum.at(best, s_, rhs)
    solved = best != np.iinfo(np.int64).max
    assert (best[solved] == K[solved]).all()
    cyc = sol.cycle_vertices
    assert is_closed_walk(n, s, d, cyc)
    mean = cycle_mean_exact(s, d, w, cyc, "min")
    assert mean == (sol.mu_exact if objective == "min" else -sol.mu_exact)
    lam = [Fraction(int(a), int(b)) for a, b in zip(num[solved][:1000], den[solved][:1000])]
    assert min(lam) >= (sol.mu_exact if objective == "min" else -sol.mu_exact)


@pytest.mark.parametrize("objective", ["min", "max"])
def test_benchmark_size_certificate(objective):
    g = P.generate_uniform(1_000_000, 8, 1, 100, 1111_0627)
    sess = P.Session(g, P.SolveOptions(objective=objective))
    sol = sess.solve()
    assert sol.has_cycle and sol.exact
    bellman_certificate(g, sol, sess.values(), objective)


def test_scc_parallel_matches_tarjan():
    # --scc parallel (the reference's trim + pivoted reachability, scc.cpp:105)
    # decomposes into the same regions: identical solver output
    g = P.generate(P.Generator("powerlaw", n=30_000, deg=2, dmax=3000, seed=31))
    for objective in ("min", "max"):
        a = P.Session(g, P.SolveOptions(objective=objective, scc="tarjan"))
        b = P.Session(g, P.SolveOptions(objective=objective, scc="parallel"))
        sa, sb = a.solve(), b.solve()
        assert (sa.mu_exact, sa.cycle_vertices, sa.stats.spf_passes, sa.stats.regions) == \
            (sb.mu_exact, sb.cycle_vertices, sb.stats.spf_passes, sb.stats.regions)
        assert np.array_equal(a.values()["key_num"], b.values()["key_num"])


def test_limits_fail_loudly():
    # 2^40 weights run (wide lane); the remaining limit -- doubling sums of
    # the largest region at |w| near 2^53 could leave 64 bits -- is refused
    # loudly (OverflowError) instead of silently changing arithmetic
    src = np.array([0, 1], np.uint32)
    dst = np.array([1, 0], np.uint32)
    g = P.build_graph(2, (src, dst, np.array([2.0 ** 40, 1.0])))
    s = P.solve(g)
    assert s.exact and s.mu_exact == Fraction(2 ** 40 + 1, 2)
    n = 1024
    ring = np.arange(n, dtype=np.uint32)
    big = np.ones(n)
    big[0] = 2.0 ** 52 + 2.0 ** 51
    with pytest.raises(OverflowError, match="62 bits"):
        P.solve(P.build_graph(n, (ring, (ring + 1) % n, big)))
    # a device ordinal that does not exist
    with pytest.raises(ValueError, match="device"):
        P.solve(P.build_graph(2, (src, dst, np.array([1.0, 2.0]))), P.SolveOptions(device=99))


def test_float_session_resolve_and_sessions_interleave():
    g = P.generate_uniform(20_000, 4, -50, 50, 41)
    s, d, w = g.edges()
    gf = P.build_graph(g.n, (s, d, w / 8.0 + 0.0625))
    fs = P.Session(gf)
    es = P.Session(g, P.SolveOptions(objective="max"))
    a = fs.solve()
    e1 = es.solve()
    b = fs.solve()
    e2 = es.solve()
    assert (a.mu, a.cycle_vertices, a.stats.spf_passes) == (b.mu, b.cycle_vertices, b.stats.spf_passes)
    assert (e1.mu_exact, e1.cycle_vertices) == (e2.mu_exact, e2.cycle_vertices)
    ref = oracle_record(g.n, s, d, w / 8.0 + 0.0625, "min", "tarjan")
    check_against(a, fs.values(), ref)


def _csr(g):
    s, d, w = g.edges()
    idx = np.zeros(g.n + 1, np.uint32)
    np.cumsum(np.bincount(s, minlength=g.n), out=idx[1:])
    return idx, d, w


@pytest.mark.parametrize("case", CASES[::3], ids=[c["name"] for c in CASES[::3]])
def test_solve_csr_matches_solve(case):
    """ocm_solve_csr (the reference's CSR arrays, staged from pageable
    memory, validated and exactness-derived on the device) == ocm_solve."""
    g = P.build_graph(case["n"], case_arrays(case))
    idx, d, w = _csr(g)
    for objective in ("min", "max"):
        for scc in ("tarjan", "off"):
            for algo in ("howard", "howard-par"):
                o = P.SolveOptions(algo=algo, objective=objective, scc=scc)
                a, b = P.solve(g, o), P.solve_csr(g.n, idx, d, w, o)
                assert (a.has_cycle, a.exact, a.mu_exact, a.mu, a.cycle_vertices) == \
                    (b.has_cycle, b.exact, b.mu_exact, b.mu, b.cycle_vertices)
                assert (a.stats.outer_iters, a.stats.spf_passes, a.stats.regions) == \
                    (b.stats.outer_iters, b.stats.spf_passes, b.stats.regions)


def test_solve_csr_large_pageable_graph():
    """A 10^6 x 8 graph (100 MB through the staging ring) equals the session."""
    g = P.generate(P.Generator("uniform", n=1_000_000, deg=8, seed=5))
    idx, d, w = _csr(g)
    a = P.Session(g, P.SolveOptions()).solve()
    b = P.solve_csr(g.n, idx, d, w)
    assert (a.mu_exact, a.cycle_vertices, a.stats.spf_passes) == \
        (b.mu_exact, b.cycle_vertices, b.stats.spf_passes)
    # integral weights in int32 range cross PCIe as int32 (widened on the device)
    assert b.stats.h2d_bytes == (g.n + 1) * 4 + g.m * 8


@pytest.mark.parametrize("last", [2.5, 2.0**31, -2.0**31 - 1, -0.0, np.nan])
def test_solve_csr_weight_narrowing_falls_back(last):
    """The int32 upload of pageable weights gives up at the first chunk
    holding any other value -- here the very last edge of a 10^6 x 8 graph,
    after ~3 chunks went up as int32 -- and copies the doubles instead: the
    result equals the pinned ocm_solve path (float lane, wide lane, the
    non-finite error of build_graph)."""
    g = P.generate(P.Generator("uniform", n=1_000_000, deg=8, seed=6))
    idx, d, w = _csr(g)
    w = w.copy()
    w[-1] = last
    if np.isnan(last):
        with pytest.raises(ValueError, match=f"edge {g.m - 1} has non-finite weight"):
            P.solve_csr(g.n, idx, d, w)
        return
    src = np.repeat(np.arange(g.n, dtype=np.uint32), np.diff(idx).astype(np.int64))
    a = P.solve(P.build_graph(g.n, (src, d, w)))
    b = P.solve_csr(g.n, idx, d, w)
    assert (a.exact, a.mu_exact, a.mu, a.cycle_vertices, a.stats.spf_passes) == \
        (b.exact, b.mu_exact, b.mu, b.cycle_vertices, b.stats.spf_passes)
    narrow = last == 0.0  # -0.0 is the integer 0
    assert b.stats.h2d_bytes == (g.n + 1) * 4 + g.m * (8 if narrow else 12)


def test_solve_csr_validates_like_build_graph():
    idx = np.array([0, 1, 2], np.uint32)
    with pytest.raises(ValueError, match="edge 1 endpoint out of range"):
        P.solve_csr(2, idx, np.array([1, 2], np.uint32), np.array([1.0, 2.0]))
    with pytest.raises(ValueError, match="edge 0 has non-finite weight"):
        P.solve_csr(2, idx, np.array([1, 0], np.uint32), np.array([np.nan, 2.0]))
    with pytest.raises(ValueError, match="offsets"):
        P.solve_csr(2, np.array([0, 2, 1], np.uint32), np.array([1, 0], np.uint32),
                    np.array([1.0, 2.0]))
    # the first bad edge in id order wins, as in build_graph's loop
    with pytest.raises(ValueError, match="edge 0 has non-finite weight"):
        P.solve_csr(2, idx, np.array([1, 5], np.uint32), np.array([np.inf, 2.0]))
    with pytest.raises(ValueError, match="edge 0 endpoint out of range"):
        P.solve_csr(2, idx, np.array([7, 1], np.uint32), np.array([1.0, np.nan]))
    # exactness is derived on the device: 2.5 makes the graph a float graph
    s = P.solve_csr(2, idx, np.array([1, 0], np.uint32), np.array([2.5, 2.0]))
    assert s.has_cycle and not s.exact and s.mu == 2.25
    s = P.solve_csr(2, idx, np.array([1, 0], np.uint32), np.array([3.0, 2.0]))
    assert s.exact and s.mu_exact == Fraction(5, 2)


WIDE_CASES = [c for c in CASES if c["name"].startswith("wide")]


@pytest.mark.parametrize("case", WIDE_CASES, ids=[c["name"] for c in WIDE_CASES])
def test_wide_weights_run_the_wide_lane(case):
    """Weights of 2^40-2^48 (the reference accepts integral |w| < 2^53,
    graph.cpp:15): the device packs 64-bit weights and runs 128-bit keys --
    same mean, cycle, policy, value keys and statistics as the reference."""
    n = case["n"]
    src, dst, w = case_arrays(case)
    g = P.build_graph(n, (src, dst, w))
    for key, ref in case["results"].items():
        objective, scc = key.split("/")
        s = P.Session(g, P.SolveOptions(objective=objective, scc=scc))
        sol = s.solve()
        check_against(sol, s.values() if scc == "tarjan" else None, ref)
        if ref["has_cycle"]:
            assert s.wide


@pytest.mark.parametrize("case", CASES[::2], ids=[c["name"] for c in CASES[::2]])
def test_forced_wide_lane_matches_reference(case, monkeypatch):
    """OCM_WIDE=1: the 128-bit lane on ordinary graphs reproduces the
    reference bit for bit as well (keys read at full width)."""
    monkeypatch.setenv("OCM_WIDE", "1")
    n = case["n"]
    src, dst, w = case_arrays(case)
    for key, ref in case["results"].items():
        objective, scc = key.split("/")
        sol, vals = run(n, src, dst, w, objective, scc)
        check_against(sol, vals if scc == "tarjan" else None, ref)


def test_keys_beyond_62_bits_promote_to_the_wide_lane():
    """A 2^17-vertex ring, weights +(2^31-1) on one half and -(2^31-1) on the
    other with a net sum of 1: mean 1/2^17 (den = 2^17) and path sums near
    2^47, so keys K = value*den reach ~2^64. The fast lane proves at adoption
    that a key could leave +-2^62 and the session re-solves with 128-bit keys;
    mean, cycle and every value key (exact integers; the reference's own
    (wsum, steps) pairs still fit int64) equal the oracle. A second graph,
    with chords, promotes on the provable bound as well."""
    n = 1 << 17
    ring = np.arange(n, dtype=np.uint32)
    w = np.where(ring < n // 2, 2.0 ** 31 - 1, -(2.0 ** 31 - 1))
    w[-1] += 1
    rng = np.random.default_rng(7)
    graphs = [(ring, (ring + 1) % n, w, True)]
    m = 1 << 16
    r2 = np.arange(m, dtype=np.uint32)
    graphs.append((np.concatenate([r2, rng.integers(0, m, 64).astype(np.uint32)]),
                   np.concatenate([(r2 + 1) % m, rng.integers(0, m, 64).astype(np.uint32)]),
                   np.concatenate([rng.integers(-(1 << 30), 1 << 30, m),
                                   np.full(64, 1 << 30)]).astype(np.float64), False))
    for src, dst, ww, huge in graphs:
        nn = int(max(src.max(), dst.max())) + 1
        g = P.build_graph(nn, (src, dst, ww))
        for objective in ("min", "max"):
            s = P.Session(g, P.SolveOptions(objective=objective))
            sol = s.solve()
            ref = oracle_record(nn, src, dst, ww, objective, "tarjan")
            o = O.oracle_solve(nn, src, dst, ww, objective, "tarjan", values=True)
            ref["value_key"] = [int(a) * int(b) - int(c) * int(d)
                                for a, b, c, d in zip(o.wsum, o.lam_den, o.steps, o.lam_num)]
            check_against(sol, s.values(), ref)
            if huge:
                assert s.wide and sol.mu_exact.denominator == n
                assert max(abs(int(k)) for k in s.keys_wide()) > 1 << 62
            elif objective == "min":  # the whole ring wins: den = 65536
                assert s.wide
            cert = s.certify()
            assert cert["key_violations"] == cert["policy_violations"] == cert["cycle_violations"] == 0


def test_wide_lane_certificate_and_generated_graph(monkeypatch):
    monkeypatch.setenv("OCM_WIDE", "1")
    spec = P.Generator("powerlaw", n=20_000, deg=4, dmax=2_000, wlo=-50, whi=50, seed=9)
    a = P.Session.generated(spec, P.SolveOptions())
    sa = a.solve()
    assert a.wide
    cert = a.certify()
    assert cert["key_violations"] == cert["policy_violations"] == cert["cycle_violations"] == 0
    monkeypatch.setenv("OCM_WIDE", "0")
    b = P.Session.generated(spec, P.SolveOptions())
    sb = b.solve()
    assert not b.wide
    assert (sa.mu_exact, sa.cycle_vertices, sa.stats.spf_passes) == \
        (sb.mu_exact, sb.cycle_vertices, sb.stats.spf_passes)
    assert a.keys_wide().tolist() == [int(x) for x in b.values()["key_num"]]


def test_session_from_reference_csr():
    """ocm_session_create_csr: a resident session on the reference's CSR
    arrays solves, re-solves and certifies like a session on the graph."""
    g = P.generate(P.Generator("powerlaw", n=40_000, deg=4, dmax=4_000, seed=13))
    idx, d, w = _csr(g)
    for objective in ("min", "max"):
        a = P.Session(g, P.SolveOptions(objective=objective))
        b = P.Session.from_csr(g.n, idx, d, w, P.SolveOptions(objective=objective))
        for _ in range(2):
            sa, sb = a.solve(), b.solve()
            assert (sa.mu_exact, sa.cycle_vertices, sa.stats.spf_passes) == \
                (sb.mu_exact, sb.cycle_vertices, sb.stats.spf_passes)
        assert np.array_equal(a.values()["key_num"], b.values()["key_num"])
        c = b.certify()
        assert c["key_violations"] == c["policy_violations"] == c["cycle_violations"] == 0
    with pytest.raises(ValueError, match="endpoint out of range"):
        P.Session.from_csr(2, np.array([0, 1, 2], np.uint32), np.array([1, 9], np.uint32),
                           np.array([1.0, 1.0]))


def test_scc_off_hamiltonian_overflow_matches_reference():
    """--scc off with weights near 2^52: the Hamiltonian weight 2n(max|w|+1)+1
    leaves the exact doubles; the reference throws std::overflow_error
    (graph.cpp:116), the device reports the same (OverflowError)."""
    src = np.array([0, 1, 2], np.uint32)
    dst = np.array([1, 2, 0], np.uint32)
    w = np.array([2.0 ** 52 - 1, -(2.0 ** 52 - 1), 3.0])
    if O.ref_available():
        with pytest.raises(RuntimeError, match="hamiltonian weight too large to stay exact"):
            O.ref_solve(3, src, dst, w, "howard", "min", "off")
    g = P.build_graph(3, (src, dst, w))
    with pytest.raises(OverflowError, match="hamiltonian weight too large to stay exact"):
        P.solve(g, P.SolveOptions(scc="off"))
    # with tarjan regions the same graph solves (wide lane): mean 1
    s = P.solve(g)
    assert s.exact and s.mu_exact == Fraction(1, 1)


def _sc_graph(rng, n, extra, float_w=False):
    perm = rng.permutation(n)
    s = np.concatenate([perm, rng.integers(0, n, extra * n)]).astype(np.uint32)
    d = np.concatenate([np.roll(perm, -1), rng.integers(0, n, extra * n)]).astype(np.uint32)
    w = rng.integers(-50, 51, len(s)).astype(np.float64)
    return n, s, d, (w / 8 + 0.1 if float_w else w)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("seed,n,extra,float_w", [(1, 50, 2, False), (2, 2000, 4, False),
                                                  (3, 20000, 7, False), (4, 2000, 4, True),
                                                  (5, 20000, 3, True)])
@pytest.mark.parametrize("objective", ["min", "max"])
def test_lambda_trace_lockstep_with_reference(seed, n, extra, float_w, objective):
    """Lockstep with the reference iteration by iteration (its acceptance
    criterion 6 compares the parallel and sequential lanes the same way,
    acceptance_main.cpp:260): on strongly connected graphs the device's
    lambda after every policy iteration equals the reference HowardPar's
    trace (howard_par.hpp:588) -- exact rationals, or the same doubles in the
    float lane."""
    n, s, d, w = _sc_graph(np.random.default_rng(seed), n, extra, float_w)
    ref = O.ref_lambda_trace(n, s, d, w, objective)
    assert ref is not None and len(ref) > 0
    sess = P.Session(P.build_graph(n, (s, d, w)), P.SolveOptions(objective=objective))
    sess.solve()
    assert sess.lambda_trace() == ref


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("seed,n,extra,float_w", [(11, 40, 2, False), (12, 1500, 4, False),
                                                  (13, 1500, 3, True), (14, 300, 6, True)])
@pytest.mark.parametrize("objective", ["min", "max"])
def test_policy_and_values_lockstep_with_reference(seed, n, extra, float_w, objective, monkeypatch):
    """Move for move: after EVERY policy iteration the device's policy (edge
    ids) and value plane equal the reference HowardPar's trace entry
    (howard_par.hpp:588: lambda, succ_edge, the plane just written) -- exact
    keys K = wsum*den - steps*num, or the same doubles in the float lane."""
    monkeypatch.setenv("OCM_TRACE_ITERS", "64")
    n, s, d, w = _sc_graph(np.random.default_rng(seed), n, extra, float_w)
    ref = O.ref_iter_trace(n, s, d, w, objective, cap_iters=64)
    lam = O.ref_lambda_trace(n, s, d, w, objective)
    assert ref and len(ref) == len(lam)
    sess = P.Session(P.build_graph(n, (s, d, w)), P.SolveOptions(objective=objective))
    sess.solve()
    assert sess.lambda_trace() == lam
    for i, (r, l) in enumerate(zip(ref, lam)):
        got = sess.iteration_trace(i)
        assert np.array_equal(got["succ_edge"], r["succ_edge"]), i
        if float_w:
            assert np.array_equal(got["fval"], r["fval"]), i
        else:
            key = [int(a) * l.denominator - int(b) * l.numerator for a, b in zip(r["wsum"], r["steps"])]
            assert got["key_num"].tolist() == key, i
