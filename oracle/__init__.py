"""TEST INFRASTRUCTURE ONLY — ctypes bindings for the CPU checkers.

Two checkers live under ``oracle/``:

* ``lib/liboracle.so`` — ``ocm_oracle.c``, the plain-C restatement of the
  reference's sequential policy iteration (each function cites the reference
  file:line it follows).
* ``_ref/libocm_ref.so`` — the UNMODIFIED reference library compiled in place
  from ``/root/reference/proj/src`` by ``oracle/Makefile`` plus a C-ABI shim.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference`` arm) may import this package,
and only as the checker / baseline. The product package
``paper_1111_0627_b200`` never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "lib", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libocm_ref.so")

ALGOS = {"howard": 0, "howard-par": 1, "lawler": 2, "tree": 3, "oracle-enum": 4, "oracle-dp": 5}
SCCS = {"tarjan": 0, "parallel": 1, "off": 2}
SCHEDULES = {"seq": 0, "par": 1, "shuffle": 2}


class _OcResult(C.Structure):
    _fields_ = [
        ("has_cycle", C.c_int32), ("exact", C.c_int32),
        ("mu_num", C.c_int64), ("mu_den", C.c_int64), ("mu", C.c_double),
        ("cycle_len", C.c_uint32),
        ("outer_iters_seq", C.c_uint32), ("spf_passes_seq", C.c_uint32),
        ("outer_iters_par", C.c_uint32), ("spf_passes_par", C.c_uint32),
        ("regions", C.c_uint32), ("trivial_regions", C.c_uint32),
    ]


class _RefResult(C.Structure):
    _fields_ = [
        ("has_cycle", C.c_int32), ("exact", C.c_int32),
        ("mu_num", C.c_int64), ("mu_den", C.c_int64), ("mu", C.c_double),
        ("cycle_len", C.c_uint32), ("outer_iters", C.c_uint32), ("spf_passes", C.c_uint32),
        ("regions", C.c_uint32), ("trivial_regions", C.c_uint32),
        ("launches", C.c_uint64), ("fixpoint_iters", C.c_uint64),
        ("solve_ms", C.c_double), ("build_ms", C.c_double),
    ]


@dataclass
class CheckerResult:
    has_cycle: bool
    exact: bool
    mu_num: int
    mu_den: int
    mu: float
    cycle: List[int]
    outer_iters: int = 0
    spf_passes: int = 0
    regions: int = 0
    trivial_regions: int = 0
    solve_ms: float = 0.0
    build_ms: float = 0.0
    # final value plane (exact: wsum/steps, float: fval) + per-vertex lambda
    wsum: Optional[np.ndarray] = None
    steps: Optional[np.ndarray] = None
    fval: Optional[np.ndarray] = None
    lam_num: Optional[np.ndarray] = None
    lam_den: Optional[np.ndarray] = None
    lam_f: Optional[np.ndarray] = None
    succ_vertex: Optional[np.ndarray] = None
    extra: dict = field(default_factory=dict)


_oracle = None
_ref = None


def _ptr(a, t):
    return a.ctypes.data_as(C.POINTER(t)) if a is not None else None


def _edges(src, dst, w):
    src = np.ascontiguousarray(src, dtype=np.uint32)
    dst = np.ascontiguousarray(dst, dtype=np.uint32)
    w = np.ascontiguousarray(w, dtype=np.float64)
    assert src.shape == dst.shape == w.shape
    return src, dst, w


def oracle_lib():
    global _oracle
    if _oracle is None:
        if not os.path.exists(ORACLE_SO):
            raise RuntimeError(f"oracle not built: {ORACLE_SO} (run make -C oracle oracle)")
        lib = C.CDLL(ORACLE_SO)
        lib.oc_solve_howard.restype = C.c_int
        lib.oc_solve_howard.argtypes = [
            C.c_uint32, C.c_uint64, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
            C.POINTER(C.c_double), C.c_int, C.c_int, C.POINTER(_OcResult),
            C.POINTER(C.c_uint32), C.c_uint32, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
            C.POINTER(C.c_double), C.POINTER(C.c_int64), C.POINTER(C.c_int64),
            C.POINTER(C.c_double), C.POINTER(C.c_uint32)]
        lib.oc_dp_min_cycle_mean.restype = C.c_int
        lib.oc_dp_min_cycle_mean.argtypes = [
            C.c_uint32, C.c_uint64, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
            C.POINTER(C.c_double), C.POINTER(C.c_int32), C.POINTER(C.c_int32),
            C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_double)]
        lib.oc_generate_uniform.restype = None
        lib.oc_generate_uniform.argtypes = [
            C.c_uint32, C.c_uint32, C.c_int32, C.c_int32, C.c_uint64,
            C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), C.POINTER(C.c_double)]
        _oracle = lib
    return _oracle


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise RuntimeError(f"reference not built: {REF_SO} (run make -C oracle ref)")
        lib = C.CDLL(REF_SO)
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_solve.restype = C.c_int
        lib.ref_solve.argtypes = [
            C.c_uint32, C.c_uint64, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
            C.POINTER(C.c_double), C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint, C.c_uint64,
            C.c_double, C.POINTER(_RefResult), C.POINTER(C.c_uint32), C.c_uint32]
        lib.ref_howard_values.restype = C.c_int
        lib.ref_howard_values.argtypes = [
            C.c_uint32, C.c_uint64, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
            C.POINTER(C.c_double), C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
            C.POINTER(C.c_double), C.POINTER(C.c_int64), C.POINTER(C.c_int64),
            C.POINTER(C.c_double), C.POINTER(C.c_uint32)]
        _ref = lib
    return _ref


def oracle_solve(n, src, dst, w, objective="min", scc="tarjan", values=False) -> CheckerResult:
    """ocm_oracle.c: oc_solve_howard (restates src/solve.cpp run_howard_seq)."""
    lib = oracle_lib()
    src, dst, w = _edges(src, dst, w)
    m = src.shape[0]
    res = _OcResult()
    cap = max(int(n), 1)
    cyc = np.zeros(cap, dtype=np.uint32)
    arrs = {}
    if values:
        for k, t in (("wsum", np.int64), ("steps", np.int64), ("fval", np.float64),
                     ("lam_num", np.int64), ("lam_den", np.int64), ("lam_f", np.float64),
                     ("succ_vertex", np.uint32)):
            arrs[k] = np.zeros(max(int(n), 1), dtype=t)
    rc = lib.oc_solve_howard(
        n, m, _ptr(src, C.c_uint32), _ptr(dst, C.c_uint32), _ptr(w, C.c_double),
        1 if objective == "max" else 0, 1 if scc == "off" else 0, C.byref(res),
        _ptr(cyc, C.c_uint32), cap,
        _ptr(arrs.get("wsum"), C.c_int64), _ptr(arrs.get("steps"), C.c_int64),
        _ptr(arrs.get("fval"), C.c_double), _ptr(arrs.get("lam_num"), C.c_int64),
        _ptr(arrs.get("lam_den"), C.c_int64), _ptr(arrs.get("lam_f"), C.c_double),
        _ptr(arrs.get("succ_vertex"), C.c_uint32))
    if rc == 1:
        raise ValueError("oracle: bad input (endpoint out of range or non-finite weight)")
    if rc != 0:
        raise RuntimeError(f"oracle: structural error {rc}")
    out = CheckerResult(bool(res.has_cycle), bool(res.exact), res.mu_num, res.mu_den, res.mu,
                        cyc[: res.cycle_len].tolist(), res.outer_iters_par, res.spf_passes_par,
                        res.regions, res.trivial_regions)
    out.extra = {"outer_iters_seq": res.outer_iters_seq, "spf_passes_seq": res.spf_passes_seq}
    for k, a in arrs.items():
        setattr(out, k, a[: int(n)])
    return out


def oracle_dp(n, src, dst, w):
    """ocm_oracle.c: oc_dp_min_cycle_mean (restates include/ocm/oracle.hpp:137)."""
    lib = oracle_lib()
    src, dst, w = _edges(src, dst, w)
    hc, ex, num, den, mean = C.c_int32(), C.c_int32(), C.c_int64(), C.c_int64(), C.c_double()
    rc = lib.oc_dp_min_cycle_mean(n, src.shape[0], _ptr(src, C.c_uint32), _ptr(dst, C.c_uint32),
                                  _ptr(w, C.c_double), C.byref(hc), C.byref(ex), C.byref(num),
                                  C.byref(den), C.byref(mean))
    if rc:
        raise ValueError("dp oracle refused the graph")
    return bool(hc.value), bool(ex.value), num.value, den.value, mean.value


def generate_uniform(n, deg, wlo, whi, seed):
    """The seeded uniform generator shared bit-for-bit with the CUDA library."""
    lib = oracle_lib()
    m = int(n) * int(deg)
    src = np.empty(m, np.uint32)
    dst = np.empty(m, np.uint32)
    w = np.empty(m, np.float64)
    lib.oc_generate_uniform(n, deg, wlo, whi, seed, _ptr(src, C.c_uint32), _ptr(dst, C.c_uint32),
                            _ptr(w, C.c_double))
    return src, dst, w


def ref_solve(n, src, dst, w, algo="howard-par", objective="min", scc="tarjan", schedule="seq",
              workers=1, seed=1, epsilon=1e-9) -> CheckerResult:
    """The reference's ocm::solve (proj/src/solve.cpp:198) through oracle/_ref."""
    lib = ref_lib()
    src, dst, w = _edges(src, dst, w)
    res = _RefResult()
    cap = max(int(n), 1)
    cyc = np.zeros(cap, dtype=np.uint32)
    rc = lib.ref_solve(n, src.shape[0], _ptr(src, C.c_uint32), _ptr(dst, C.c_uint32),
                       _ptr(w, C.c_double), ALGOS[algo], 1 if objective == "max" else 0,
                       SCCS[scc], SCHEDULES[schedule], workers, seed, epsilon, C.byref(res),
                       _ptr(cyc, C.c_uint32), cap)
    if rc:
        raise RuntimeError("reference: " + lib.ref_last_error().decode())
    out = CheckerResult(bool(res.has_cycle), bool(res.exact), res.mu_num, res.mu_den, res.mu,
                        cyc[: res.cycle_len].tolist(), res.outer_iters, res.spf_passes,
                        res.regions, res.trivial_regions, res.solve_ms, res.build_ms)
    out.extra = {"launches": res.launches, "fixpoint_iters": res.fixpoint_iters}
    return out


def ref_values(n, src, dst, w, objective="min") -> CheckerResult:
    """Final value plane of the reference's HowardPar (howard_par.hpp:544 run())."""
    lib = ref_lib()
    src, dst, w = _edges(src, dst, w)
    nn = max(int(n), 1)
    a = {k: np.zeros(nn, dtype=t) for k, t in (
        ("wsum", np.int64), ("steps", np.int64), ("fval", np.float64), ("lam_num", np.int64),
        ("lam_den", np.int64), ("lam_f", np.float64), ("succ_vertex", np.uint32))}
    rc = lib.ref_howard_values(n, src.shape[0], _ptr(src, C.c_uint32), _ptr(dst, C.c_uint32),
                               _ptr(w, C.c_double), 1 if objective == "max" else 0,
                               _ptr(a["wsum"], C.c_int64), _ptr(a["steps"], C.c_int64),
                               _ptr(a["fval"], C.c_double), _ptr(a["lam_num"], C.c_int64),
                               _ptr(a["lam_den"], C.c_int64), _ptr(a["lam_f"], C.c_double),
                               _ptr(a["succ_vertex"], C.c_uint32))
    if rc:
        raise RuntimeError("reference: " + lib.ref_last_error().decode())
    out = CheckerResult(False, False, 0, 1, 0.0, [])
    for k, v in a.items():
        setattr(out, k, v[: int(n)])
    return out


def ref_generate_model(kind, clients, costs=()):
    """The reference's ocm::generate_model (src/model_gen.cpp:90) through
    oracle/_ref. kind: "worker" | "server" | "loop" (with costs)."""
    lib = ref_lib()
    fn = lib.ref_generate_model
    fn.restype = C.c_int
    fn.argtypes = [C.c_int, C.POINTER(C.c_int64), C.c_uint32, C.c_uint32, C.POINTER(C.c_uint32),
                   C.POINTER(C.c_uint64), C.c_uint64, C.POINTER(C.c_uint32),
                   C.POINTER(C.c_uint32), C.POINTER(C.c_double)]
    k = {"worker": 0, "server": 1, "loop": 2}[kind]
    cs = np.asarray(costs, dtype=np.int64)
    n, m = C.c_uint32(), C.c_uint64()
    if fn(k, _ptr(cs, C.c_int64), len(cs), clients, C.byref(n), C.byref(m), 0, None, None, None):
        raise RuntimeError("reference: " + lib.ref_last_error().decode())
    src = np.empty(m.value, np.uint32)
    dst = np.empty(m.value, np.uint32)
    w = np.empty(m.value, np.float64)
    if fn(k, _ptr(cs, C.c_int64), len(cs), clients, C.byref(n), C.byref(m), m.value,
          _ptr(src, C.c_uint32), _ptr(dst, C.c_uint32), _ptr(w, C.c_double)):
        raise RuntimeError("reference: " + lib.ref_last_error().decode())
    return n.value, src, dst, w


def ref_parse_graph_text(text: str, source: str = "<text>"):
    """The reference's ocm::parse_graph_text (src/graph_io.cpp) through
    oracle/_ref. Returns ("ok", n, src, dst, w, integer_exact) or
    ("parse", message, line) / ("error", message)."""
    lib = ref_lib()
    fn = lib.ref_parse_graph_text
    fn.restype = C.c_int
    fn.argtypes = [C.c_char_p, C.c_uint64, C.c_char_p, C.POINTER(C.c_uint32),
                   C.POINTER(C.c_uint64), C.POINTER(C.c_int32), C.c_uint64,
                   C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), C.POINTER(C.c_double),
                   C.POINTER(C.c_int32)]
    b = text.encode() if isinstance(text, str) else bytes(text)
    n, m, ex, line = C.c_uint32(), C.c_uint64(), C.c_int32(), C.c_int32()
    rc = fn(b, len(b), source.encode(), C.byref(n), C.byref(m), C.byref(ex), 0, None, None, None,
            C.byref(line))
    if rc == 1:
        return ("parse", lib.ref_last_error().decode(), line.value)
    if rc:
        return ("error", lib.ref_last_error().decode())
    src = np.empty(m.value, np.uint32)
    dst = np.empty(m.value, np.uint32)
    w = np.empty(m.value, np.float64)
    fn(b, len(b), source.encode(), C.byref(n), C.byref(m), C.byref(ex), m.value,
       _ptr(src, C.c_uint32), _ptr(dst, C.c_uint32), _ptr(w, C.c_double), C.byref(line))
    return ("ok", n.value, src, dst, w, bool(ex.value))


def generate_powerlaw(n, dmin, dmax, wlo, whi, seed, hubs=False):
    """Power-law out-degree generator ("powerlaw" / "powerlaw-hubs" with
    hubs=True or 1 / "powerlaw-web" with hubs=3), shared bit-for-bit with the
    CUDA library's host and device generators."""
    lib = oracle_lib()
    fn = lib.oc_generate_powerlaw
    fn.restype = C.c_uint64
    fn.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_int32, C.c_int32, C.c_uint64, C.c_int,
                   C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), C.POINTER(C.c_double)]
    m = int(fn(n, dmin, dmax, wlo, whi, seed, int(hubs), None, None, None))
    src = np.empty(m, np.uint32)
    dst = np.empty(m, np.uint32)
    w = np.empty(m, np.float64)
    fn(n, dmin, dmax, wlo, whi, seed, int(hubs), _ptr(src, C.c_uint32), _ptr(dst, C.c_uint32),
       _ptr(w, C.c_double))
    return src, dst, w


# proj/src/model_gen.cpp:23 worker_scenario / :36 server_scenario, restated as
# (states, [(from, to, cost, acquires, releases)], uses_server)
SCENARIOS = {
    "worker": (3, [(0, 1, 1, 0, 0), (1, 0, 0, 0, 0), (1, 2, 2, 0, 0), (2, 0, 3, 0, 0)], False),
    "server": (4, [(0, 1, 1, 0, 0), (1, 0, 0, 0, 0), (1, 2, 2, 1, 0), (2, 3, 5, 0, 0),
                   (3, 0, 1, 0, 1)], True),
}


def generate_model(scenario, clients, max_states=1 << 31):
    """oc_generate_model: the restated reference model generator
    (model_gen.cpp:88) without the reference's 5*10^6-state bound.
    Returns (n, src, dst, w) in edge-id order."""
    lib = oracle_lib()
    fn = lib.oc_generate_model
    fn.restype = C.c_int
    P = C.POINTER
    fn.argtypes = [C.c_uint32, C.c_uint32, P(C.c_uint32), P(C.c_uint32), P(C.c_int64),
                   P(C.c_int32), P(C.c_int32), C.c_int, C.c_uint32, C.c_uint64, P(C.c_uint32),
                   P(C.c_uint64), P(P(C.c_uint32)), P(P(C.c_uint32)), P(P(C.c_double))]
    lib.oc_free.restype = None
    lib.oc_free.argtypes = [C.c_void_p]
    states, trs, uses_server = SCENARIOS[scenario] if isinstance(scenario, str) else scenario
    cols = list(zip(*trs)) if trs else [(), (), (), (), ()]
    f, t, c, a, r = (np.ascontiguousarray(x, dt) for x, dt in zip(
        cols, (np.uint32, np.uint32, np.int64, np.int32, np.int32)))
    n, m = C.c_uint32(), C.c_uint64()
    ps, pd, pw = P(C.c_uint32)(), P(C.c_uint32)(), P(C.c_double)()
    rc = fn(states, len(trs), _ptr(f, C.c_uint32), _ptr(t, C.c_uint32), _ptr(c, C.c_int64),
            _ptr(a, C.c_int32), _ptr(r, C.c_int32), int(uses_server), clients, max_states,
            C.byref(n), C.byref(m), C.byref(ps), C.byref(pd), C.byref(pw))
    if rc:
        raise {1: ValueError, 2: OverflowError}.get(rc, MemoryError)(f"oc_generate_model rc={rc}")
    mm = m.value
    try:
        src = np.ctypeslib.as_array(ps, (mm,)).copy() if mm else np.empty(0, np.uint32)
        dst = np.ctypeslib.as_array(pd, (mm,)).copy() if mm else np.empty(0, np.uint32)
        w = np.ctypeslib.as_array(pw, (mm,)).copy() if mm else np.empty(0, np.float64)
    finally:
        for p in (ps, pd, pw):
            lib.oc_free(C.cast(p, C.c_void_p))
    return n.value, src, dst, w


class RefGraph:
    """A reference ocm::Graph built once (oracle/_ref ref_graph_create) and
    solved repeatedly -- also from several threads at once (ctypes releases
    the GIL; ocm::solve only reads the graph)."""

    def __init__(self, n, src, dst, w):
        lib = ref_lib()
        lib.ref_graph_create.restype = C.c_void_p
        lib.ref_graph_create.argtypes = [C.c_uint32, C.c_uint64, C.POINTER(C.c_uint32),
                                         C.POINTER(C.c_uint32), C.POINTER(C.c_double)]
        lib.ref_graph_free.restype = None
        lib.ref_graph_free.argtypes = [C.c_void_p]
        lib.ref_graph_solve.restype = C.c_int
        lib.ref_graph_solve.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int,
                                        C.POINTER(_RefResult), C.POINTER(C.c_uint32), C.c_uint32]
        src, dst, w = _edges(src, dst, w)
        self.n = int(n)
        self._lib = lib
        self._h = lib.ref_graph_create(n, src.shape[0], _ptr(src, C.c_uint32),
                                       _ptr(dst, C.c_uint32), _ptr(w, C.c_double))
        if not self._h:
            raise RuntimeError("reference: " + lib.ref_last_error().decode())

    def solve(self, algo="howard", objective="min", scc="tarjan") -> CheckerResult:
        res = _RefResult()
        cap = max(self.n, 1)
        cyc = np.zeros(cap, dtype=np.uint32)
        if self._lib.ref_graph_solve(self._h, ALGOS[algo], 1 if objective == "max" else 0,
                                     SCCS[scc], C.byref(res), _ptr(cyc, C.c_uint32), cap):
            raise RuntimeError("reference: " + self._lib.ref_last_error().decode())
        out = CheckerResult(bool(res.has_cycle), bool(res.exact), res.mu_num, res.mu_den, res.mu,
                            cyc[: res.cycle_len].tolist(), res.outer_iters, res.spf_passes,
                            res.regions, res.trivial_regions, res.solve_ms, 0.0)
        return out

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self._lib.ref_graph_free(h)
            self._h = None


def ref_lambda_trace(n, src, dst, w, objective="min", scc="tarjan"):
    """The reference's lambda after each policy iteration (HowardPar::run
    trace, howard_par.hpp:588) of a single-region graph (or, scc="off", of
    the Hamiltonian-augmented graph): Fractions (exact) or floats; None when
    the graph is not strongly connected."""
    lib = ref_lib()
    fn = lib.ref_lambda_trace2
    fn.restype = C.c_int
    fn.argtypes = [C.c_uint32, C.c_uint64, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                   C.POINTER(C.c_double), C.c_int, C.c_int, C.POINTER(C.c_int64),
                   C.POINTER(C.c_int64), C.POINTER(C.c_double), C.c_uint32, C.POINTER(C.c_uint32)]
    src, dst, w = _edges(src, dst, w)
    cap = 1 << 16
    num = np.zeros(cap, np.int64)
    den = np.zeros(cap, np.int64)
    f = np.zeros(cap, np.float64)
    ln = C.c_uint32()
    rc = fn(n, src.shape[0], _ptr(src, C.c_uint32), _ptr(dst, C.c_uint32), _ptr(w, C.c_double),
            1 if objective == "max" else 0, 1 if scc == "off" else 0, _ptr(num, C.c_int64),
            _ptr(den, C.c_int64), _ptr(f, C.c_double), cap, C.byref(ln))
    if rc == 2:
        return None
    if rc:
        raise RuntimeError("reference: " + lib.ref_last_error().decode())
    k = min(int(ln.value), cap)
    from fractions import Fraction
    if den[:k].any():
        return [Fraction(int(a), int(b)) for a, b in zip(num[:k], den[:k])]
    return f[:k].tolist()


def ref_iter_trace(n, src, dst, w, objective="min", cap_iters=64):
    """The reference HowardPar trace of a single-region graph, per iteration:
    list of dicts {succ_edge, wsum, steps} (exact) or {succ_edge, fval}."""
    lib = ref_lib()
    fn = lib.ref_iter_trace
    fn.restype = C.c_int
    P = C.POINTER
    fn.argtypes = [C.c_uint32, C.c_uint64, P(C.c_uint32), P(C.c_uint32), P(C.c_double), C.c_int,
                   C.c_uint32, P(C.c_uint32), P(C.c_int64), P(C.c_int64), P(C.c_double),
                   P(C.c_uint32)]
    src, dst, w = _edges(src, dst, w)
    cells = cap_iters * int(n)
    se = np.zeros(cells, np.uint32)
    ws = np.zeros(cells, np.int64)
    st = np.zeros(cells, np.int64)
    fv = np.zeros(cells, np.float64)
    ln = C.c_uint32()
    rc = fn(n, src.shape[0], _ptr(src, C.c_uint32), _ptr(dst, C.c_uint32), _ptr(w, C.c_double),
            1 if objective == "max" else 0, cap_iters, _ptr(se, C.c_uint32), _ptr(ws, C.c_int64),
            _ptr(st, C.c_int64), _ptr(fv, C.c_double), C.byref(ln))
    if rc == 2:
        return None
    if rc:
        raise RuntimeError("reference: " + lib.ref_last_error().decode())
    out = []
    for i in range(min(int(ln.value), cap_iters)):
        sl = slice(i * n, (i + 1) * n)
        out.append({"succ_edge": se[sl].copy(), "wsum": ws[sl].copy(), "steps": st[sl].copy(),
                    "fval": fv[sl].copy()})
    return out
