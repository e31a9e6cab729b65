"""paper_1111_0627_b200 — B200-native optimal cycle mean (policy iteration).

Python mirror of the reference's public interface (proj/include/ocm):

=========================  ==========================================
reference                  here
=========================  ==========================================
ocm::build_graph           :func:`build_graph`        (graph.hpp:76)
ocm::parse_graph_text      :func:`parse_graph_text`   (graph_io.hpp:41)
ocm::read_graph_file       :func:`read_graph_file`    (graph_io.hpp:45)
ocm::SolveOptions          :class:`SolveOptions`      (solve.hpp:36)
ocm::Solution / SolveStats :class:`Solution`          (solve.hpp:45/54)
ocm::solve                 :func:`solve`              (solve.hpp:64)
ocm::ParseError            :class:`ParseError`        (graph_io.hpp:27)
=========================  ==========================================

Everything computes through ``lib/libocm_b200.so`` (the C-ABI declared in
``include/ocm_b200.h``; CUDA kernels for sm_100a). There is no CPU fallback:
importing works without a GPU (graph building and parsing are host code), but
:func:`solve` raises :class:`DeviceError` when no sm_100 device is present, and
the module refuses to import when the native library has not been built.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from fractions import Fraction
from typing import Iterable, List, Optional, Sequence, Tuple

import numpy as np

__all__ = [
    "Graph", "build_graph", "parse_graph_text", "read_graph_file", "generate_uniform",
    "Scenario", "Transition", "loop_scenario", "worker_scenario", "server_scenario",
    "generate_model", "K_MAX_MODEL_STATES", "Generator", "generate",
    "SolveOptions", "SolveStats", "Solution", "solve", "solve_csr", "Session",
    "ParseError", "StructuralError", "DeviceError", "UnsupportedError", "LIB_PATH",
]

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("OCM_LIB") or os.path.join(HERE, "lib", "libocm_b200.so")

OK, E_INVALID, E_PARSE, E_LOGIC, E_CUDA, E_UNSUPPORTED, E_RANGE, E_IO = range(8)
ALGOS = {"howard": 0, "howard-par": 1, "lawler": 2, "tree": 3, "oracle-enum": 4, "oracle-dp": 5}
OBJECTIVES = {"min": 0, "max": 1}
SCCS = {"tarjan": 0, "parallel": 1, "off": 2}


class ParseError(ValueError):
    """Malformed graph text; message is ``<source>:<line>: <what>``."""

    def __init__(self, msg: str, line: int):
        super().__init__(msg)
        self.line = line


class StructuralError(RuntimeError):
    """The reference's std::logic_error (e.g. a region that is not strongly connected)."""


class DeviceError(RuntimeError):
    """No usable sm_100a device or a CUDA failure (there is no CPU fallback)."""


class UnsupportedError(NotImplementedError):
    """Lane or option the device library does not provide."""


class _Transition(C.Structure):
    _fields_ = [("from_", C.c_uint32), ("to", C.c_uint32), ("cost", C.c_int64),
                ("acquires", C.c_int32), ("releases", C.c_int32)]


class _Gen(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n", C.c_uint32), ("deg", C.c_uint32), ("dmax", C.c_uint32),
                ("wlo", C.c_int32), ("whi", C.c_int32), ("seed", C.c_uint64)]


class _Certificate(C.Structure):
    _fields_ = [("vertices", C.c_uint64), ("edges", C.c_uint64), ("regions", C.c_uint64),
                ("key_violations", C.c_uint64), ("policy_violations", C.c_uint64),
                ("cycle_violations", C.c_uint64)]


class _ShardBuffers(C.Structure):
    _fields_ = [("rank", C.c_uint32), ("world", C.c_uint32), ("chunk", C.c_uint32),
                ("own_lo", C.c_uint32), ("own_hi", C.c_uint32), ("n", C.c_uint32),
                ("succ_e", C.c_void_p), ("succ_v", C.c_void_p), ("succ_w", C.c_void_p),
                ("succ_w_bytes", C.c_uint32), ("regions", C.c_uint32),
                ("changed0", C.c_void_p), ("changed1", C.c_void_p), ("stream", C.c_void_p)]


class _ShardPeer(C.Structure):
    _fields_ = [("ptr", C.c_uint64 * 6), ("ipc", (C.c_ubyte * 64) * 6), ("device", C.c_int32),
                ("rank", C.c_uint32)]


class _Opts(C.Structure):
    _fields_ = [("algo", C.c_int32), ("objective", C.c_int32), ("scc", C.c_int32),
                ("device", C.c_int32), ("epsilon", C.c_double)]


class _Sol(C.Structure):
    _fields_ = [
        ("has_cycle", C.c_int32), ("exact", C.c_int32), ("mu_num", C.c_int64),
        ("mu_den", C.c_int64), ("mu", C.c_double), ("cycle_len", C.c_uint32),
        ("outer_iters", C.c_uint32), ("spf_passes", C.c_uint32), ("regions", C.c_uint32),
        ("trivial_regions", C.c_uint32), ("n_solved", C.c_uint32), ("m_solved", C.c_uint64),
        ("launches", C.c_uint64), ("fixpoint_iters", C.c_uint64), ("device_ms", C.c_double),
        ("improve_ms", C.c_double), ("host_prep_ms", C.c_double),
        ("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64),
    ]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"native library missing: {LIB_PATH}; build it with `make -C {HERE}` "
            "(or __graft_entry__.build())")
    lib = C.CDLL(LIB_PATH)
    P = C.POINTER
    sig = {
        "ocm_last_error": (C.c_char_p, []),
        "ocm_last_error_line": (C.c_int, []),
        "ocm_version": (C.c_char_p, []),
        "ocm_device_count": (C.c_int, []),
        "ocm_build_graph": (C.c_int, [C.c_uint32, C.c_uint64, P(C.c_uint32), P(C.c_uint32),
                                      P(C.c_double), P(C.c_void_p)]),
        "ocm_parse_graph_text": (C.c_int, [C.c_char_p, C.c_size_t, C.c_char_p, P(C.c_void_p)]),
        "ocm_read_graph_file": (C.c_int, [C.c_char_p, P(C.c_void_p)]),
        "ocm_generate_uniform": (C.c_int, [C.c_uint32, C.c_uint32, C.c_int32, C.c_int32,
                                           C.c_uint64, P(C.c_void_p)]),
        "ocm_generate_model": (C.c_int, [C.c_uint32, P(_Transition), C.c_uint32, C.c_int32,
                                         C.c_uint32, C.c_uint64, P(C.c_void_p)]),
        "ocm_generate": (C.c_int, [P(_Gen), P(C.c_void_p)]),
        "ocm_session_create_generated": (C.c_int, [P(_Gen), P(_Opts), P(C.c_void_p)]),
        "ocm_session_n": (C.c_uint32, [C.c_void_p]),
        "ocm_session_create_shard": (C.c_int, [C.c_void_p, P(_Gen), P(_Opts), C.c_uint32,
                                               C.c_uint32, P(C.c_void_p)]),
        "ocm_session_shard_buffers": (C.c_int, [C.c_void_p, P(_ShardBuffers)]),
        "ocm_session_shard_step": (C.c_int, [C.c_void_p, P(C.c_int32)]),
        "ocm_session_shard_finish": (C.c_int, [C.c_void_p, P(_Sol), P(C.c_uint32), C.c_uint32]),
        "ocm_session_shard_peer_info": (C.c_int, [C.c_void_p, P(_ShardPeer)]),
        "ocm_session_shard_connect": (C.c_int, [C.c_void_p, P(_ShardPeer), C.c_uint32, C.c_int32]),
        "ocm_session_shard_fused_launch": (C.c_int, [C.c_void_p]),
        "ocm_session_shard_fused_finish": (C.c_int, [C.c_void_p, P(_Sol), P(C.c_uint32),
                                                     C.c_uint32]),
        "ocm_graph_free": (None, [C.c_void_p]),
        "ocm_graph_n": (C.c_uint32, [C.c_void_p]),
        "ocm_graph_m": (C.c_uint64, [C.c_void_p]),
        "ocm_graph_integer_exact": (C.c_int, [C.c_void_p]),
        "ocm_graph_edges": (C.c_int, [C.c_void_p, P(C.c_uint32), P(C.c_uint32), P(C.c_double)]),
        "ocm_graph_csr": (C.c_int, [C.c_void_p, P(P(C.c_uint64)), P(P(C.c_uint32)),
                                    P(P(C.c_double))]),
        "ocm_solve": (C.c_int, [C.c_void_p, P(_Opts), P(_Sol), P(C.c_uint32), C.c_uint32]),
        "ocm_solve_csr": (C.c_int, [C.c_uint32, C.c_uint32, P(C.c_uint32), P(C.c_uint32),
                                    P(C.c_double), P(_Opts), P(_Sol), P(C.c_uint32), C.c_uint32]),
        "ocm_session_create_csr": (C.c_int, [C.c_uint32, C.c_uint32, P(C.c_uint32), P(C.c_uint32),
                                             P(C.c_double), P(_Opts), P(C.c_void_p)]),
        "ocm_session_create": (C.c_int, [C.c_void_p, P(_Opts), P(C.c_void_p)]),
        "ocm_session_solve": (C.c_int, [C.c_void_p, P(_Sol), P(C.c_uint32), C.c_uint32]),
        "ocm_session_values": (C.c_int, [C.c_void_p, P(C.c_int64), P(C.c_int64), P(C.c_int64),
                                         P(C.c_double), P(C.c_uint32)]),
        "ocm_session_certify": (C.c_int, [C.c_void_p, P(_Certificate)]),
        "ocm_session_keys_wide": (C.c_int, [C.c_void_p, P(C.c_int64), P(C.c_uint64)]),
        "ocm_session_is_wide": (C.c_int, [C.c_void_p]),
        "ocm_session_lambda_trace": (C.c_int, [C.c_void_p, P(C.c_int64), P(C.c_int64), P(C.c_double),
                                               C.c_uint32, P(C.c_uint32)]),
        "ocm_session_iter_trace": (C.c_int, [C.c_void_p, C.c_uint32, P(C.c_uint32), P(C.c_int64),
                                             P(C.c_double)]),
        "ocm_session_stream": (C.c_void_p, [C.c_void_p]),
        "ocm_session_free": (None, [C.c_void_p]),
    }
    for name, (res, args) in sig.items():
        if os.environ.get("OCM_LIB") and not hasattr(lib, name):
            continue  # experimental library override (scripts/build_variant.sh) may be older
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_lib = _load()
EXPORTED_SYMBOLS = (
    "ocm_last_error", "ocm_last_error_line", "ocm_version", "ocm_device_count",
    "ocm_build_graph", "ocm_parse_graph_text", "ocm_read_graph_file", "ocm_generate_uniform",
    "ocm_generate_model", "ocm_generate", "ocm_session_create_generated", "ocm_session_n",
    "ocm_session_create_shard", "ocm_session_shard_buffers", "ocm_session_shard_step",
    "ocm_session_shard_finish", "ocm_session_shard_peer_info", "ocm_session_shard_connect",
    "ocm_session_shard_fused_launch", "ocm_session_shard_fused_finish",
    "ocm_graph_free", "ocm_graph_n", "ocm_graph_m", "ocm_graph_integer_exact", "ocm_graph_edges",
    "ocm_graph_csr",
    "ocm_solve", "ocm_solve_csr", "ocm_session_create_csr", "ocm_session_create", "ocm_session_solve", "ocm_session_values",
    "ocm_session_stream", "ocm_session_free", "ocm_session_certify", "ocm_session_keys_wide",
    "ocm_session_is_wide", "ocm_session_lambda_trace", "ocm_session_iter_trace",
)


def _check(rc: int) -> None:
    if rc == OK:
        return
    msg = (_lib.ocm_last_error() or b"").decode()
    if rc == E_PARSE:
        raise ParseError(msg, _lib.ocm_last_error_line())
    if rc == E_INVALID:
        raise ValueError(msg)
    if rc == E_LOGIC:
        raise StructuralError(msg)
    if rc == E_CUDA:
        raise DeviceError(msg)
    if rc == E_UNSUPPORTED:
        raise UnsupportedError(msg)
    if rc == E_RANGE:
        raise OverflowError(msg)
    raise OSError(msg)


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t)) if a is not None else None


class Graph:
    """Handle on a host CSR graph (ocm::Graph, graph.hpp:34): edge ids are CSR
    positions grouped by source, input order preserved within a source."""

    def __init__(self, handle):
        self._h = C.c_void_p(handle)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and h.value and _lib is not None:
            _lib.ocm_graph_free(h)
            self._h = C.c_void_p(None)

    @property
    def n(self) -> int:
        return int(_lib.ocm_graph_n(self._h))

    @property
    def m(self) -> int:
        return int(_lib.ocm_graph_m(self._h))

    @property
    def integer_exact(self) -> bool:
        return bool(_lib.ocm_graph_integer_exact(self._h))

    def csr(self) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
        """(fwd_index, fwd_target, fwd_weight) as read-only zero-copy views of
        the graph's own CSR (graph.hpp:38-41; offsets 64-bit here). The views
        keep the graph alive."""
        pi, pt, pw = C.POINTER(C.c_uint64)(), C.POINTER(C.c_uint32)(), C.POINTER(C.c_double)()
        _check(_lib.ocm_graph_csr(self._h, C.byref(pi), C.byref(pt), C.byref(pw)))
        n, m = self.n, self.m
        out = []
        for ptr, cnt in ((pi, n + 1), (pt, m), (pw, m)):
            if cnt:
                buf = (ptr._type_ * cnt).from_address(C.addressof(ptr.contents))
                buf._graph = self  # the array's base owns a reference to the graph
                a = np.ctypeslib.as_array(buf)
            else:
                a = np.empty(0, ptr._type_)
            a.flags.writeable = False
            out.append(a)
        return tuple(out)

    def edges(self) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
        """(source, target, weight) arrays in edge-id order (Graph::edges())."""
        m = self.m
        s = np.empty(m, np.uint32)
        d = np.empty(m, np.uint32)
        w = np.empty(m, np.float64)
        _check(_lib.ocm_graph_edges(self._h, _p(s, C.c_uint32), _p(d, C.c_uint32),
                                    _p(w, C.c_double)))
        return s, d, w


def _as_arrays(edges) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
    if isinstance(edges, tuple) and len(edges) == 3 and hasattr(edges[0], "__len__") and \
            not isinstance(edges[0], (int, float)):
        s, d, w = edges
    else:
        lst = list(edges)
        s = [e[0] for e in lst]
        d = [e[1] for e in lst]
        w = [e[2] for e in lst]
    s = np.asarray(s).reshape(-1)
    d = np.asarray(d).reshape(-1)
    w = np.asarray(w, dtype=np.float64).reshape(-1)
    if not (s.shape[0] == d.shape[0] == w.shape[0]):
        raise ValueError(f"edge arrays differ in length (src {s.shape[0]}, dst {d.shape[0]}, "
                         f"weight {w.shape[0]})")
    for name, a in (("source", s), ("target", d)):
        if a.size == 0:
            continue
        if a.dtype.kind not in "iu":
            if not np.all(np.floor(a) == a):
                raise ValueError(f"non-integral {name} vertex id")
        lo, hi = a.min(), a.max()
        if lo < 0 or hi >= 2**32:
            # the reference's Vertex is uint32 (graph.hpp:20); never wrap silently
            raise ValueError(f"{name} vertex id {int(lo if lo < 0 else hi)} out of range")
    return (np.ascontiguousarray(s, np.uint32), np.ascontiguousarray(d, np.uint32),
            np.ascontiguousarray(w))


def build_graph(n: int, edges) -> Graph:
    """ocm::build_graph (graph.hpp:76). ``edges``: iterable of (u, v, w) or a
    (src, dst, w) tuple of arrays. Raises ValueError like std::invalid_argument:
    on ``n`` outside [0, 2^32), arrays of unequal length, and (in the native
    builder, with the reference's message) endpoints outside [0, n)."""
    if int(n) != n or not 0 <= int(n) < 2**32:
        raise ValueError(f"vertex count {n} out of range")
    s, d, w = _as_arrays(edges)
    h = C.c_void_p()
    _check(_lib.ocm_build_graph(int(n), s.shape[0], _p(s, C.c_uint32), _p(d, C.c_uint32),
                                _p(w, C.c_double), C.byref(h)))
    return Graph(h.value)


def parse_graph_text(text: str, source: str = "<text>") -> Graph:
    """ocm::parse_graph_text (graph_io.hpp:41): 'p ocm n m' / 'a u v w' (1-based) or
    plain '<u> <v> <w>' edge lists (0-based)."""
    b = text.encode()
    h = C.c_void_p()
    _check(_lib.ocm_parse_graph_text(b, len(b), source.encode(), C.byref(h)))
    return Graph(h.value)


def read_graph_file(path: str) -> Graph:
    """ocm::read_graph_file (graph_io.hpp:45)."""
    h = C.c_void_p()
    _check(_lib.ocm_read_graph_file(os.fsencode(path), C.byref(h)))
    return Graph(h.value)


def generate_uniform(n: int, deg: int, wlo: int = 1, whi: int = 100, seed: int = 1) -> Graph:
    """Seeded random digraph with out-degree exactly ``deg`` and integer weights."""
    h = C.c_void_p()
    _check(_lib.ocm_generate_uniform(int(n), int(deg), int(wlo), int(whi), int(seed), C.byref(h)))
    return Graph(h.value)


@dataclass
class Generator:
    """Synthetic benchmark graph (include/ocm_b200.h ocm_generator): kind
    "uniform" (out-degree exactly ``deg``), "powerlaw" (out-degree
    min(dmax, floor(deg / sqrt(u))), tail exponent 3, uniform targets) or
    "powerlaw-hubs" (the same out-degrees, targets floor(n*u^2) scattered by
    a bijection: in-degrees with tail exponent 3, i.e. hub vertices) or
    "powerlaw-web" (targets floor(n*u^8): in-degree density exponent ~2.14,
    the web graphs' law); integer weights
    uniform in [wlo, whi]. :func:`generate` builds it on the host,
    :meth:`Session.generated` directly in HBM -- bit-identical graphs."""
    kind: str = "uniform"
    n: int = 1000
    deg: int = 8
    dmax: int = 0
    wlo: int = 1
    whi: int = 100
    seed: int = 1

    def _c(self) -> "_Gen":
        kinds = {"uniform": 0, "powerlaw": 1, "powerlaw-hubs": 2, "powerlaw-web": 3}
        if self.kind not in kinds:
            raise ValueError(f"unknown generator kind {self.kind!r}")
        return _Gen(kinds[self.kind], int(self.n), int(self.deg), int(self.dmax), int(self.wlo),
                    int(self.whi), int(self.seed))


def generate(spec: Generator) -> Graph:
    """Host graph of a generator description."""
    h = C.c_void_p()
    _check(_lib.ocm_generate(C.byref(spec._c()), C.byref(h)))
    return Graph(h.value)


K_MAX_MODEL_STATES = 5_000_000  # proj/include/ocm/model_gen.hpp:70 kMaxModelStates


@dataclass
class Transition:
    """proj/include/ocm/model_gen.hpp:31 Scenario::Transition."""
    from_: int
    to: int
    cost: int
    acquires: bool = False
    releases: bool = False


@dataclass
class Scenario:
    """proj/include/ocm/model_gen.hpp:29 Scenario."""
    name: str
    states: int
    transitions: List[Transition]
    uses_server: bool = False


def loop_scenario(costs) -> Scenario:
    """model_gen.cpp:10 loop_scenario: 0 -> 1 -> ... -> 0 with the given costs."""
    costs = [int(c) for c in costs]
    if not costs:
        raise ValueError("loop scenario needs at least one transition")
    k = len(costs)
    return Scenario(f"loop{k}", k, [Transition(i, (i + 1) % k, costs[i]) for i in range(k)])


def worker_scenario() -> Scenario:
    """model_gen.cpp:21 worker_scenario (template "server-free")."""
    return Scenario("worker", 3, [Transition(0, 1, 1), Transition(1, 0, 0), Transition(1, 2, 2),
                                  Transition(2, 0, 3)])


def server_scenario() -> Scenario:
    """model_gen.cpp:34 server_scenario (template "server")."""
    return Scenario("server", 4, [Transition(0, 1, 1), Transition(1, 0, 0),
                                  Transition(1, 2, 2, acquires=True), Transition(2, 3, 5),
                                  Transition(3, 0, 1, releases=True)], uses_server=True)


def generate_model(sc: Scenario, clients: int, max_states: int = K_MAX_MODEL_STATES) -> Graph:
    """model_gen.hpp:67 generate_model: composite state space of `clients`
    interleaved copies of `sc`, vertices in breadth-first discovery order.
    Raises ValueError on malformed scenarios and StructuralError (the
    reference's std::length_error) past max_states."""
    arr = (_Transition * max(1, len(sc.transitions)))()
    for i, t in enumerate(sc.transitions):
        arr[i] = _Transition(int(t.from_), int(t.to), int(t.cost), int(bool(t.acquires)),
                             int(bool(t.releases)))
    h = C.c_void_p()
    _check(_lib.ocm_generate_model(int(sc.states), arr, len(sc.transitions), int(sc.uses_server),
                                   int(clients), int(max_states), C.byref(h)))
    return Graph(h.value)


@dataclass
class SolveOptions:
    """ocm::SolveOptions (solve.hpp:36). The reference's CPU-engine schedule,
    workers and seed have no device meaning and are accepted but ignored."""
    algo: str = "howard-par"
    objective: str = "min"
    scc: str = "tarjan"
    epsilon: float = 1e-9
    device: int = 0
    schedule: str = "seq"
    workers: int = 0
    seed: int = 1

    def _c(self) -> _Opts:
        if self.algo not in ALGOS:
            raise ValueError(f"unknown algorithm '{self.algo}'")
        return _Opts(ALGOS[self.algo], OBJECTIVES[self.objective], SCCS[self.scc],
                     int(self.device), float(self.epsilon))


@dataclass
class SolveStats:
    """ocm::SolveStats (solve.hpp:45) plus device timing."""
    outer_iters: int = 0
    spf_passes: int = 0
    launches: int = 0
    fixpoint_iters: int = 0
    regions: int = 0
    trivial_regions: int = 0
    n_solved: int = 0
    m_solved: int = 0
    device_ms: float = 0.0
    improve_ms: float = 0.0
    host_prep_ms: float = 0.0
    h2d_bytes: int = 0
    d2h_bytes: int = 0


@dataclass
class Solution:
    """ocm::Solution (solve.hpp:54)."""
    has_cycle: bool = False
    exact: bool = False
    mu_exact: Fraction = Fraction(0)
    mu: float = 0.0
    cycle_vertices: List[int] = field(default_factory=list)
    stats: SolveStats = field(default_factory=SolveStats)


def _solution(sol: _Sol, cyc: np.ndarray) -> Solution:
    st = SolveStats(sol.outer_iters, sol.spf_passes, sol.launches, sol.fixpoint_iters,
                    sol.regions, sol.trivial_regions, sol.n_solved, sol.m_solved,
                    sol.device_ms, sol.improve_ms, sol.host_prep_ms, sol.h2d_bytes,
                    sol.d2h_bytes)
    mu_exact = Fraction(sol.mu_num, sol.mu_den) if sol.exact else Fraction(0)
    return Solution(bool(sol.has_cycle), bool(sol.exact), mu_exact, float(sol.mu),
                    cyc[: min(sol.cycle_len, cyc.shape[0])].astype(np.int64).tolist(), st)


def solve(g: Graph, opt: Optional[SolveOptions] = None) -> Solution:
    """ocm::solve (solve.hpp:64) on the B200: policy iteration (lane howard-par)."""
    opt = opt or SolveOptions()
    sol = _Sol()
    cyc = np.empty(max(g.n, 1), np.uint32)  # only the first cycle_len entries are read
    _check(_lib.ocm_solve(g._h, C.byref(opt._c()), C.byref(sol), _p(cyc, C.c_uint32),
                          cyc.shape[0]))
    return _solution(sol, cyc)


def solve_csr(n: int, fwd_index, fwd_target, fwd_weight,
              opt: Optional[SolveOptions] = None) -> Solution:
    """ocm::solve on the reference's own CSR arrays (ocm::Graph fwd_index /
    fwd_target / fwd_weight, graph.hpp:38-41) through ``ocm_solve_csr``: read
    in place (pageable memory is staged through the library's pinned ring),
    checked on the device like build_graph (ValueError), exactness derived
    on the device."""
    opt = opt or SolveOptions()
    idx = np.ascontiguousarray(fwd_index, np.uint32)
    tgt = np.ascontiguousarray(fwd_target, np.uint32)
    w = np.ascontiguousarray(fwd_weight, np.float64)
    n = int(n)
    if idx.shape[0] != n + 1 or tgt.shape[0] != w.shape[0] or tgt.shape[0] >= 2**32:
        raise ValueError("CSR arrays: fwd_index needs n+1 entries, fwd_target and fwd_weight m each")
    sol = _Sol()
    cyc = np.empty(max(n, 1), np.uint32)
    _check(_lib.ocm_solve_csr(n, tgt.shape[0], _p(idx, C.c_uint32), _p(tgt, C.c_uint32),
                              _p(w, C.c_double), C.byref(opt._c()), C.byref(sol),
                              _p(cyc, C.c_uint32), cyc.shape[0]))
    return _solution(sol, cyc)


class Session:
    """A graph resident in HBM (region-compacted CSR uploaded once); each
    :meth:`solve` re-runs policy iteration from the initial policy."""

    def __init__(self, g: Graph, opt: Optional[SolveOptions] = None):
        self.opt = opt or SolveOptions()
        self.n = g.n
        h = C.c_void_p()
        _check(_lib.ocm_session_create(g._h, C.byref(self.opt._c()), C.byref(h)))
        self._h = h

    @classmethod
    def from_csr(cls, n: int, fwd_index, fwd_target, fwd_weight,
                 opt: Optional[SolveOptions] = None) -> "Session":
        """Session on the reference's CSR arrays (ocm::Graph fwd_index /
        fwd_target / fwd_weight), checked on the device like build_graph."""
        self = cls.__new__(cls)
        self.opt = opt or SolveOptions()
        idx = np.ascontiguousarray(fwd_index, np.uint32)
        tgt = np.ascontiguousarray(fwd_target, np.uint32)
        w = np.ascontiguousarray(fwd_weight, np.float64)
        if idx.shape[0] != int(n) + 1 or tgt.shape[0] != w.shape[0]:
            raise ValueError("CSR arrays: fwd_index needs n+1 entries, fwd_target and fwd_weight m each")
        h = C.c_void_p()
        _check(_lib.ocm_session_create_csr(int(n), tgt.shape[0], _p(idx, C.c_uint32),
                                           _p(tgt, C.c_uint32), _p(w, C.c_double),
                                           C.byref(self.opt._c()), C.byref(h)))
        self._h = h
        self.n = int(n)
        return self

    @classmethod
    def generated(cls, spec: Generator, opt: Optional[SolveOptions] = None) -> "Session":
        """Session over a generated graph written directly into HBM."""
        self = cls.__new__(cls)
        self.opt = opt or SolveOptions()
        h = C.c_void_p()
        _check(_lib.ocm_session_create_generated(C.byref(spec._c()), C.byref(self.opt._c()),
                                                 C.byref(h)))
        self._h = h
        self.n = int(_lib.ocm_session_n(h))
        return self

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and h.value and _lib is not None:
            _lib.ocm_session_free(h)
            self._h = C.c_void_p(None)

    @property
    def stream(self) -> int:
        return int(_lib.ocm_session_stream(self._h) or 0)

    def solve(self) -> Solution:
        sol = _Sol()
        cyc = np.empty(max(self.n, 1), np.uint32)
        _check(_lib.ocm_session_solve(self._h, C.byref(sol), _p(cyc, C.c_uint32), cyc.shape[0]))
        return _solution(sol, cyc)

    def certify(self) -> dict:
        """Device-side optimality certificate of the last solve (exact lane;
        include/ocm_b200.h ocm_certificate): checked counts and violation
        counts -- all violations 0 proves every region's lambda optimal."""
        c = _Certificate()
        _check(_lib.ocm_session_certify(self._h, C.byref(c)))
        return {f: int(getattr(c, f)) for f, _ in _Certificate._fields_}

    @property
    def wide(self) -> bool:
        """True when the last solve ran the wide exact lane (128-bit keys)."""
        return bool(_lib.ocm_session_is_wide(self._h))

    def lambda_trace(self) -> list:
        """Lambda of the non-trivial region after each policy iteration of the
        last solve (Fractions in the exact lanes, floats in the float lane):
        the reference's HowardTrace (howard_par.hpp:588)."""
        cap = 4096
        num = np.zeros(cap, np.int64)
        den = np.zeros(cap, np.int64)
        f = np.zeros(cap, np.float64)
        ln = C.c_uint32()
        _check(_lib.ocm_session_lambda_trace(self._h, _p(num, C.c_int64), _p(den, C.c_int64),
                                             _p(f, C.c_double), cap, C.byref(ln)))
        k = min(int(ln.value), cap)
        if den[:k].any():
            return [Fraction(int(a), int(b)) for a, b in zip(num[:k], den[:k])]
        return f[:k].tolist()

    def iteration_trace(self, it: int) -> dict:
        """Debug (session created with OCM_TRACE_ITERS=k in the environment):
        policy edge ids, value keys (exact) / values (float) after iteration
        `it` of the last solve."""
        n = max(self.n, 1)
        out = {"succ_edge": np.zeros(n, np.uint32), "key_num": np.zeros(n, np.int64),
               "fval": np.zeros(n, np.float64)}
        _check(_lib.ocm_session_iter_trace(self._h, int(it), _p(out["succ_edge"], C.c_uint32),
                                           _p(out["key_num"], C.c_int64), _p(out["fval"], C.c_double)))
        return {k: v[: self.n] for k, v in out.items()}

    def keys_wide(self) -> np.ndarray:
        """Exact value keys at full width as Python ints (object array):
        value(v) = key[v] / lam_den[v]."""
        n = max(self.n, 1)
        hi = np.zeros(n, np.int64)
        lo = np.zeros(n, np.uint64)
        _check(_lib.ocm_session_keys_wide(self._h, _p(hi, C.c_int64), _p(lo, C.c_uint64)))
        return np.array([(int(h) << 64) | int(l) for h, l in zip(hi[: self.n], lo[: self.n])],
                        dtype=object)

    def values(self):
        """Final value plane: dict with key_num/lam_num/lam_den (exact: value =
        key_num/lam_den), fval (float graphs) and succ_vertex, in original order.
        After a wide-lane solve key_num holds Python ints (object array)."""
        n = max(self.n, 1)
        out = {k: np.zeros(n, t) for k, t in (("key_num", np.int64), ("lam_num", np.int64),
                                              ("lam_den", np.int64), ("fval", np.float64),
                                              ("succ_vertex", np.uint32))}
        wide = bool(_lib.ocm_session_is_wide(self._h))
        _check(_lib.ocm_session_values(self._h, None if wide else _p(out["key_num"], C.c_int64),
                                       _p(out["lam_num"], C.c_int64),
                                       _p(out["lam_den"], C.c_int64),
                                       _p(out["fval"], C.c_double),
                                       _p(out["succ_vertex"], C.c_uint32)))
        res = {k: v[: self.n] for k, v in out.items()}
        if wide:
            res["key_num"] = Session.keys_wide(self)
        return res
