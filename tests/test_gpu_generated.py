"""GPU parity of the generated workloads (BASELINE.json configs 2-5 shapes).

* graphs generated directly in HBM are the host generator's graphs: the two
  sessions agree bit for bit (policy, keys, iteration counts);
* power-law graphs exercise the block-cooperative path for heavy vertices,
  checked against the C oracle (forced low heavy threshold included);
* the reference's client/server state space is solved to the oracle's result;
* at larger sizes a size-independent optimality certificate is checked.
"""
import os

import numpy as np
import pytest

import oracle as O
import paper_1111_0627_b200 as P
from test_gpu_parity import check_against, oracle_record

pytestmark = pytest.mark.gpu


def solve_both(sess_a, sess_b):
    a, b = sess_a.solve(), sess_b.solve()
    va, vb = sess_a.values(), sess_b.values()
    assert (a.mu_exact, a.cycle_vertices) == (b.mu_exact, b.cycle_vertices)
    assert (a.stats.outer_iters, a.stats.spf_passes, a.stats.m_solved) == \
        (b.stats.outer_iters, b.stats.spf_passes, b.stats.m_solved)
    for k in ("key_num", "lam_num", "lam_den", "succ_vertex"):
        assert np.array_equal(va[k], vb[k]), k
    return a


@pytest.mark.parametrize("spec", [
    P.Generator("uniform", n=100_000, deg=8, seed=3),
    P.Generator("powerlaw", n=100_000, deg=8, dmax=1 << 20, seed=4),
    P.Generator("powerlaw", n=50_000, deg=2, dmax=5000, wlo=-50, whi=50, seed=6),
], ids=["uniform", "powerlaw", "powerlaw-signed"])
@pytest.mark.parametrize("objective", ["min", "max"])
def test_device_generator_matches_host(spec, objective):
    opt = P.SolveOptions(objective=objective)
    g = P.generate(spec)
    solve_both(P.Session.generated(spec, opt), P.Session(g, opt))


@pytest.mark.parametrize("heavy", [None, "16"])
@pytest.mark.parametrize("objective", ["min", "max"])
def test_powerlaw_vs_oracle(heavy, objective, monkeypatch):
    if heavy:
        monkeypatch.setenv("OCM_HEAVY_DEG", heavy)
    spec = P.Generator("powerlaw", n=20_000, deg=4, dmax=20_000, seed=11)
    g = P.generate(spec)
    s, d, w = g.edges()
    sess = P.Session(g, P.SolveOptions(objective=objective))
    sol = sess.solve()
    check_against(sol, sess.values(), oracle_record(g.n, s, d, w, objective, "tarjan"))


@pytest.mark.parametrize("objective", ["min", "max"])
def test_server_model_vs_oracle(objective):
    g = P.generate_model(P.server_scenario(), 12)
    s, d, w = g.edges()
    sess = P.Session(g, P.SolveOptions(objective=objective))
    sol = sess.solve()
    check_against(sol, sess.values(), oracle_record(g.n, s, d, w, objective, "tarjan"))


def certificate(g, sol, vals, objective):
    """Vectorised optimality certificate (see test_gpu_parity.bellman_certificate):
    K[v] <= K[t] + w*den - num on every intra-component edge with equality on
    the policy edge, the cycle is a closed walk of mean mu, mu = min lambda."""
    from fractions import Fraction

    from scipy.sparse import csr_matrix
    from scipy.sparse.csgraph import connected_components
    s, d, w = g.edges()
    if objective == "max":
        w = -w
    n = g.n
    _, lab = connected_components(csr_matrix((np.ones(len(s), np.int8), (s, d)), shape=(n, n)),
                                  directed=True, connection="strong")
    intra = lab[s] == lab[d]
    K, num, den = vals["key_num"], vals["lam_num"], vals["lam_den"]
    s_, d_, w_ = s[intra], d[intra], w[intra].astype(np.int64)
    rhs = K[d_] + w_ * den[s_] - num[s_]
    assert (K[s_] <= rhs).all()
    best = np.full(n, np.iinfo(np.int64).max)
    np.minimum.at(best, s_, rhs)
    solved = best != np.iinfo(np.int64).max
    assert (best[solved] == K[solved]).all()
    cyc = np.array(sol.cycle_vertices, np.int64)
    nxt = np.roll(cyc, -1)
    keys = s.astype(np.int64) * n + d.astype(np.int64)
    order = np.argsort(keys, kind="stable")
    sk = keys[order]
    q = cyc * n + nxt
    pos = np.searchsorted(sk, q)
    assert (pos < len(sk)).all() and (sk[pos] == q).all()  # closed walk
    # cheapest parallel edge per cycle step (weights already signed for max)
    wk = w[order]
    tot = Fraction(0)
    for i, qq in enumerate(q.tolist()):
        lo, hi = np.searchsorted(sk, qq), np.searchsorted(sk, qq, side="right")
        tot += Fraction(float(wk[lo:hi].min()))
    mu = sol.mu_exact if objective == "min" else -sol.mu_exact
    assert tot / len(cyc) == mu
    lam = {Fraction(int(a), int(b)) for a, b in zip(num[solved], den[solved])} if solved.sum() < 10 ** 6 \
        else {Fraction(int(a), int(b)) for a, b in zip(num[solved][::97], den[solved][::97])}
    assert min(lam) >= mu


@pytest.mark.parametrize("objective", ["min", "max"])
def test_powerlaw_certificate(objective):
    spec = P.Generator("powerlaw", n=2_000_000, deg=8, dmax=1 << 20, seed=1111_0627)
    sess = P.Session.generated(spec, P.SolveOptions(objective=objective))
    sol = sess.solve()
    assert sol.has_cycle and sol.exact
    certificate(P.generate(spec), sol, sess.values(), objective)


@pytest.mark.parametrize("hot", ["0", "1", None])
@pytest.mark.parametrize("slots", ["64", "2048"])
@pytest.mark.parametrize("objective", ["min", "max"])
def test_hub_graph_staged_keys_vs_oracle(hot, slots, objective, monkeypatch):
    """In-degree-skewed power-law graph ("powerlaw-hubs"): the improvement
    pass reading hub keys from the per-CTA shared-memory table (OCM_HOT=1
    forces it on, None = the automatic choice, 0 = off; 64 slots make hubs
    collide and fall back to gathers) equals the oracle bit for bit."""
    if hot is not None:
        monkeypatch.setenv("OCM_HOT", hot)
    monkeypatch.setenv("OCM_HOT_SLOTS", slots)
    spec = P.Generator("powerlaw-hubs", n=30_000, deg=4, dmax=20_000, seed=12)
    g = P.generate(spec)
    s, d, w = g.edges()
    sess = P.Session(g, P.SolveOptions(objective=objective))
    sol = sess.solve()
    check_against(sol, sess.values(), oracle_record(g.n, s, d, w, objective, "tarjan"))


@pytest.mark.parametrize("objective", ["min", "max"])
def test_staged_keys_on_uniform_graph(objective, monkeypatch):
    """The table forced on for a graph without hubs (every probe misses or
    hits a vertex of ordinary degree) changes nothing."""
    spec = P.Generator("uniform", n=100_000, deg=8, seed=3)
    monkeypatch.setenv("OCM_HOT", "0")
    a = P.Session.generated(spec, P.SolveOptions(objective=objective))
    monkeypatch.setenv("OCM_HOT", "1")
    b = P.Session.generated(spec, P.SolveOptions(objective=objective))
    solve_both(a, b)


@pytest.mark.parametrize("spec", [
    P.Generator("uniform", n=100_000, deg=8, seed=3),
    P.Generator("powerlaw", n=60_000, deg=8, dmax=1 << 20, seed=4),
    P.Generator("powerlaw-web", n=60_000, deg=4, dmax=5000, wlo=-50, whi=50, seed=6),
], ids=["uniform", "powerlaw", "web-signed"])
@pytest.mark.parametrize("objective", ["min", "max"])
def test_tma_staged_pass_matches_direct(spec, objective, monkeypatch):
    """The improvement pass fed by bulk-TMA copies of each chunk's offsets
    and edges into shared memory (OCM_STAGED=1; on by default only for key
    arrays beyond 64 MB) equals the direct pass bit for bit, including chunks
    too large for a stage (heavy vertices) that fall back to global loads."""
    monkeypatch.setenv("OCM_STAGED", "0")
    a = P.Session.generated(spec, P.SolveOptions(objective=objective))
    monkeypatch.setenv("OCM_STAGED", "1")
    b = P.Session.generated(spec, P.SolveOptions(objective=objective))
    solve_both(a, b)
    solve_both(a, b)  # re-solves: mbarrier phases carried across launches


@pytest.mark.parametrize("objective", ["min", "max"])
def test_tma_staged_pass_vs_oracle(objective, monkeypatch):
    monkeypatch.setenv("OCM_STAGED", "1")
    spec = P.Generator("powerlaw-hubs", n=20_000, deg=4, dmax=20_000, seed=11)
    g = P.generate(spec)
    s, d, w = g.edges()
    sess = P.Session(g, P.SolveOptions(objective=objective))
    sol = sess.solve()
    check_against(sol, sess.values(), oracle_record(g.n, s, d, w, objective, "tarjan"))


@pytest.mark.parametrize("spec", [
    P.Generator("uniform", n=100_000, deg=8, seed=3),
    P.Generator("powerlaw-hubs", n=100_000, deg=8, dmax=1 << 20, seed=4),
    P.Generator("powerlaw", n=50_000, deg=2, dmax=5000, wlo=-50, whi=50, seed=6),
], ids=["uniform", "powerlaw-hubs", "powerlaw-signed"])
@pytest.mark.parametrize("objective", ["min", "max"])
def test_connected_bitmap_attach_matches_gathers(spec, objective, monkeypatch):
    """Attach testing heads with the connected-vertex bitmap (on by default
    from 2^24 vertices; OCM_CBITS_MIN_N=0 forces it) equals the conn[]
    gathers bit for bit: same policy, values, statistics."""
    monkeypatch.setenv("OCM_CBITS_MIN_N", "2147483647")
    a = P.Session.generated(spec, P.SolveOptions(objective=objective))
    monkeypatch.setenv("OCM_CBITS_MIN_N", "0")
    b = P.Session.generated(spec, P.SolveOptions(objective=objective))
    solve_both(a, b)
    solve_both(a, b)


@pytest.mark.parametrize("objective", ["min", "max"])
def test_connected_bitmap_attach_vs_oracle(objective, monkeypatch):
    """Forced bitmap on a multi-region graph, exact (64- and 128-bit keys)
    and float lanes, against the pinned oracle."""
    monkeypatch.setenv("OCM_CBITS_MIN_N", "0")
    g = P.generate(P.Generator("powerlaw", n=20_000, deg=2, dmax=2000, seed=12))
    s, d, w = g.edges()
    for ww, wide in ((w, "0"), (w / 8 + 0.125, "0"), (w * 2.0**33, "1")):
        monkeypatch.setenv("OCM_WIDE", wide)
        gg = P.build_graph(g.n, (s, d, ww))
        sess = P.Session(gg, P.SolveOptions(objective=objective))
        sol = sess.solve()
        assert sess.wide == (wide == "1")
        check_against(sol, sess.values(), oracle_record(g.n, s, d, ww, objective, "tarjan"))


@pytest.mark.parametrize("objective", ["min", "max"])
@pytest.mark.parametrize("cbits", ["0", "2147483647"])
def test_block_cooperative_attach_vs_oracle(objective, cbits, monkeypatch):
    """Pending vertices of out-degree >= 256 attach by a block-wide scan of
    their row (first hit in CSR order = least hit edge id): a dense
    power-law graph where ~6% of the vertices are that heavy, exact and
    float lanes, with and without the connected bitmap, against the oracle."""
    monkeypatch.setenv("OCM_CBITS_MIN_N", cbits)
    g = P.generate(P.Generator("powerlaw", n=4000, deg=64, dmax=4000, seed=23))
    s, d, w = g.edges()
    assert (np.bincount(s, minlength=g.n) >= 256).mean() > 0.03
    for ww in (w, w / 8 + 0.125):
        gg = P.build_graph(g.n, (s, d, ww))
        sess = P.Session(gg, P.SolveOptions(objective=objective))
        sol = sess.solve()
        assert sol.stats.fixpoint_iters > 0
        check_against(sol, sess.values(), oracle_record(g.n, s, d, ww, objective, "tarjan"))


@pytest.mark.parametrize("spec", [
    P.Generator("uniform", n=100_000, deg=8, seed=3),
    P.Generator("powerlaw", n=50_000, deg=2, dmax=5000, wlo=-50, whi=50, seed=6),
], ids=["uniform", "powerlaw-signed"])
@pytest.mark.parametrize("objective", ["min", "max"])
def test_doubling_steps_per_pass_agree(spec, objective, monkeypatch):
    """Two doubling steps per pass (the k_solve instantiation graphs beyond
    2^21 vertices use) and three (the default below) give bit-identical
    solves: same policy, values and statistics."""
    monkeypatch.setenv("OCM_ROUND_S", "2")
    a = P.Session.generated(spec, P.SolveOptions(objective=objective))
    monkeypatch.setenv("OCM_ROUND_S", "3")
    b = P.Session.generated(spec, P.SolveOptions(objective=objective))
    solve_both(a, b)
    solve_both(a, b)
