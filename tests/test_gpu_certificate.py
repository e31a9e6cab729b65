"""GPU: the device optimality certificate (ocm_session_certify) at the
BASELINE.json configurations' full sizes -- the size-independent parity
property for sizes the CPU oracle cannot solve: Bellman optimality of every
key on every intra-region edge, the policy edge attaining it, and each
region's anchor cycle closed, least-anchored and of mean exactly lambda
(together: lambda is the region's minimum cycle mean). Smaller cases pin
the certificate itself against the oracle's mu."""
import pytest

import oracle as O
import paper_1111_0627_b200 as P
from helpers import case_arrays, golden_cases

pytestmark = pytest.mark.gpu

SEED = 1111_0627


def clean(c):
    return c["key_violations"] == 0 and c["policy_violations"] == 0 and c["cycle_violations"] == 0


@pytest.mark.parametrize("case", golden_cases()[:60], ids=lambda c: c["name"])
def test_certificate_on_golden_cases(case):
    g = P.build_graph(case["n"], case_arrays(case))
    for objective in ("min", "max"):
        sess = P.Session(g, P.SolveOptions(objective=objective))
        sol = sess.solve()
        if not sol.has_cycle or not sol.exact:
            continue
        c = sess.certify()
        assert clean(c), c
        assert c["vertices"] > 0 and c["regions"] > 0


@pytest.mark.parametrize("objective", ["min", "max"])
def test_certificate_agrees_with_oracle(objective):
    g = P.generate_uniform(20000, 3, -50, 100, 77)
    s, d, w = g.edges()
    sess = P.Session(g, P.SolveOptions(objective=objective))
    sol = sess.solve()
    c = sess.certify()
    assert clean(c) and c["edges"] > 0, c
    ref = O.oracle_solve(g.n, s, d, w, objective)
    assert (ref.mu_num, ref.mu_den) == (sol.mu_exact.numerator, sol.mu_exact.denominator)


def test_certificate_float_lane_is_unsupported():
    import numpy as np
    g = P.build_graph(3, (np.array([0, 1, 2], np.uint32), np.array([1, 2, 0], np.uint32),
                          np.array([0.5, 1.25, 2.0])))
    sess = P.Session(g)
    sess.solve()
    with pytest.raises(P.UnsupportedError):
        sess.certify()


FULL = {
    "config2-uniform-1e6": P.Generator("uniform", n=1_000_000, deg=8, seed=SEED),
    "config4-powerlaw-6.4e7": P.Generator("powerlaw", n=64_000_000, deg=8, dmax=1 << 20, seed=SEED),
    "config5-uniform-2.5e8": P.Generator("uniform", n=250_000_000, deg=8, seed=SEED),
}


@pytest.mark.parametrize("name", sorted(FULL))
@pytest.mark.parametrize("objective", ["min", "max"])
def test_full_size_certificate(name, objective):
    sess = P.Session.generated(FULL[name], P.SolveOptions(objective=objective))
    sol = sess.solve()
    assert sol.has_cycle and sol.exact
    c = sess.certify()
    assert clean(c), c
    assert c["vertices"] > 0.9 * FULL[name].n and c["regions"] >= 1


def test_certificate_detects_a_corrupted_policy():
    """The certificate is not vacuous: after a solve, overwrite one policy
    weight and one policy head in device memory (through the sharded lane's
    zero-copy buffer views, world 1) and the check must flag them."""
    import ctypes as C

    import torch
    from paper_1111_0627_b200.sharded import LocalComm, ShardSession, solve_sharded
    g = P.generate_uniform(5000, 4, 1, 100, 3)
    sh = ShardSession(g, P.SolveOptions(), 0, 1)
    (sol,) = solve_sharded([sh], LocalComm())
    assert sol.has_cycle

    def certify():
        c = P._Certificate()
        P._check(P._lib.ocm_session_certify(sh._h, C.byref(c)))
        return {f: int(getattr(c, f)) for f, _ in P._Certificate._fields_}

    assert clean(certify())
    (succ_e, succ_v, succ_w), _ = sh.tensors()
    v = int(sol.cycle_vertices[0])
    succ_w[v] += 1  # the policy weight no longer matches its edge
    torch.cuda.synchronize()
    c = certify()
    assert c["policy_violations"] >= 1 and c["cycle_violations"] >= 1, c
    succ_w[v] -= 1
    succ_v[v] = (int(succ_v[v]) + 1) % 5000  # the policy head no longer matches its edge
    torch.cuda.synchronize()
    assert certify()["policy_violations"] >= 1


def test_repeated_solves_are_identical_and_certified():
    """A hundred back-to-back solves on resident sessions (the persistent
    kernel's counters, stamps and rings persist across launches) give the
    same mu, cycle and iteration counts every time, and stay certified."""
    spec = P.Generator("uniform", n=200_000, deg=8, seed=SEED)
    for objective in ("min", "max"):
        sess = P.Session.generated(spec, P.SolveOptions(objective=objective))
        first = sess.solve()
        key = (first.mu_exact, first.cycle_vertices, first.stats.spf_passes, first.stats.outer_iters)
        for _ in range(100):
            s = sess.solve()
            assert (s.mu_exact, s.cycle_vertices, s.stats.spf_passes, s.stats.outer_iters) == key
        assert clean(sess.certify())
