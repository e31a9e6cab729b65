"""The drop-in boundary in C++ (INTEGRATION.md §1): oracle/_ref/ocm_integration
is the reference compiled in place with integration/howard_b200_lane.hpp --
the lane a maintainer adds to proj/src/solve.cpp -- linked to
libocm_b200.so. It reads each graph with the reference's read_graph_file and
compares ocm::solve (lanes howard and howard-par) with the same solve()
front end dispatching to the B200 lane through ocm_solve_csr, for min/max x
tarjan/off."""
import os
import subprocess

import numpy as np
import pytest

import paper_1111_0627_b200 as P
from conftest import HAS_GPU, ROOT
from helpers import case_arrays, golden_cases

BIN = os.path.join(ROOT, "oracle", "_ref", "ocm_integration")
pytestmark = pytest.mark.skipif(not os.path.exists(BIN), reason="oracle/_ref/ocm_integration not built")


def write_problem_file(path, n, src, dst, w):
    """The reference's problem-line format (graph_io.hpp:7-10; keeps n)."""
    with open(path, "w") as f:
        f.write(f"c written by tests/test_integration_cpp.py\np ocm {n} {len(src)}\n")
        for u, v, x in zip(src.tolist(), dst.tolist(), w.tolist()):
            f.write(f"a {u + 1} {v + 1} {int(x) if float(x).is_integer() else repr(float(x))}\n")


def test_binary_links_the_product_library():
    out = subprocess.run(["ldd", BIN], capture_output=True, text=True)
    assert "libocm_b200.so" in out.stdout and "not found" not in out.stdout


@pytest.mark.skipif(HAS_GPU, reason="checks the no-device contract")
def test_binary_fails_loudly_without_device(tmp_path):
    p = tmp_path / "g.txt"
    write_problem_file(p, 2, np.array([0, 1]), np.array([1, 0]), np.array([2.0, 4.0]))
    out = subprocess.run([BIN, str(p)], capture_output=True, text=True, timeout=120)
    assert out.returncode != 0 and "FAIL" in out.stdout and "OK" not in out.stdout.split()


@pytest.mark.gpu
def test_golden_cases_through_the_cpp_lane(tmp_path):
    files = []
    for c in golden_cases():
        p = tmp_path / f"{c['name']}.txt"
        write_problem_file(p, c["n"], *case_arrays(c))
        files.append(str(p))
    out = subprocess.run([BIN] + files, capture_output=True, text=True, timeout=1200)
    lines = out.stdout.splitlines()
    assert len(lines) == 12 * len(files)
    bad = [l for l in lines if not l.startswith("OK")]
    assert out.returncode == 0 and not bad, bad[:10]


@pytest.mark.gpu
def test_generated_graphs_through_the_cpp_lane(tmp_path):
    files = []
    for spec in (P.Generator("uniform", n=100_000, deg=8, seed=3),
                 P.Generator("powerlaw-hubs", n=50_000, deg=4, dmax=5_000, seed=4)):
        g = P.generate(spec)
        p = tmp_path / f"{spec.kind}.txt"
        write_problem_file(p, g.n, *g.edges())
        files.append(str(p))
    out = subprocess.run([BIN] + files, capture_output=True, text=True, timeout=1800)
    bad = [l for l in out.stdout.splitlines() if not l.startswith("OK")]
    assert out.returncode == 0 and not bad, bad[:10]
