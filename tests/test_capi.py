"""CPU: the C-ABI library loads, exports every symbol include/ocm_b200.h
declares, and its host-side entry points behave like the reference's
(build_graph, parse_graph_text/read_graph_file error contract)."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import paper_1111_0627_b200 as P
from conftest import HAS_GPU, ROOT

HEADER = os.path.join(ROOT, "include", "ocm_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(ocm_[a-z_]+)\s*\(", text)))


def test_header_symbols_exported():
    syms = declared_symbols()
    assert len(syms) >= 15
    lib = ctypes.CDLL(P.LIB_PATH)
    for s in syms:
        assert hasattr(lib, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", P.LIB_PATH], capture_output=True,
                         text=True).stdout
    for s in syms:
        assert re.search(rf"\bT {s}$", out, re.M), s
    assert set(P.EXPORTED_SYMBOLS) == set(syms)


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", P.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_build_graph_layout_matches_reference():
    # proj/tests/test_graph.cpp:17: grouped by source, input order kept
    g = P.build_graph(3, [(1, 0, 10), (0, 2, 1), (1, 2, 20), (0, 1, 2), (1, 0, 30)])
    s, d, w = g.edges()
    assert s.tolist() == [0, 0, 1, 1, 1]
    assert d.tolist() == [2, 1, 0, 2, 0]
    assert w.tolist() == [1, 2, 10, 20, 30]
    assert g.integer_exact
    assert not P.build_graph(2, [(0, 1, 0.5)]).integer_exact


def test_build_graph_rejects_bad_input():
    with pytest.raises(ValueError, match="endpoint out of range"):
        P.build_graph(2, [(0, 2, 1)])
    with pytest.raises(ValueError, match="non-finite"):
        P.build_graph(2, [(0, 1, float("inf"))])


def test_parse_formats_and_errors(tmp_path):
    g = P.parse_graph_text("c x\np ocm 3 2\na 1 2 5\na 3 1 -2\n")
    assert (g.n, g.m) == (3, 2)
    assert g.edges()[1].tolist() == [1, 0]
    g = P.parse_graph_text("# c\n0 1 2\n1 0 4\n")
    assert (g.n, g.m) == (2, 2)
    for text, line, what in [
        ("p ocm 2 1\na 1 3 1\n", 2, "out of range"),
        ("p ocm 2 2\na 1 2 1\n", 2, "arc count mismatch"),
        ("c x\na 1 2 1\n", 2, "arc before problem line"),
        ("c x\nq 1\n", 2, "unknown line kind"),
        ("a 1 2 1\n", 1, "expected"),
        ("0 1\n", 1, "expected"),
        ("0 1 x\n", 1, "bad weight"),
        ("", 0, "empty input"),
        ("p ocm 2 0\np ocm 2 0\n", 2, "duplicate problem line"),
    ]:
        with pytest.raises(P.ParseError, match=what) as ei:
            P.parse_graph_text(text, "f.txt")
        assert ei.value.line == line
        assert str(ei.value).startswith(f"f.txt:{line}:")
    p = tmp_path / "g.txt"
    p.write_text("0 1 2\n1 0 4\n")
    assert P.read_graph_file(str(p)).m == 2
    with pytest.raises(OSError):
        P.read_graph_file(str(tmp_path / "missing.txt"))


def test_generator_matches_oracle_generator():
    import oracle as O
    g = P.generate_uniform(3000, 8, 1, 100, 11)
    s, d, w = g.edges()
    s2, d2, w2 = O.generate_uniform(3000, 8, 1, 100, 11)
    assert (s == s2).all() and (d == d2).all() and (w == w2).all()


@pytest.mark.skipif(HAS_GPU, reason="checks the no-device contract")
def test_no_cpu_fallback_without_device():
    g = P.build_graph(2, [(0, 1, 2), (1, 0, 4)])
    with pytest.raises(P.DeviceError):
        P.solve(g)


def test_unsupported_lanes_fail_loudly():
    g = P.build_graph(2, [(0, 1, 2), (1, 0, 4)])
    with pytest.raises((P.UnsupportedError, P.DeviceError)):
        P.solve(g, P.SolveOptions(algo="lawler"))


def test_build_graph_rejects_unequal_arrays():
    # the native builder would read past the shorter arrays
    with pytest.raises(ValueError, match="differ in length"):
        P.build_graph(4, (np.arange(4), [1], [1.0]))
    with pytest.raises(ValueError, match="differ in length"):
        P.build_graph(4, (np.arange(2), np.arange(2), [1.0]))


def test_build_graph_rejects_ids_that_would_wrap():
    # ids >= 2^32 wrapped to uint32 and a negative n became 2^32-1
    with pytest.raises(ValueError, match="out of range"):
        P.build_graph(2, [(0, 2**32, 1.0)])
    with pytest.raises(ValueError, match="out of range"):
        P.build_graph(-1, [(0, 0, 1.0)])
    with pytest.raises(ValueError, match="out of range"):
        P.build_graph(2**32, [(0, 0, 1.0)])
    with pytest.raises(ValueError):
        P.build_graph(3, (np.array([0.5]), np.array([1]), np.array([1.0])))
    g = P.build_graph(0, (np.array([], np.int64), np.array([], np.int64), np.array([])))
    assert (g.n, g.m) == (0, 0)
