"""Graph text parsing against the UNMODIFIED reference parser (oracle/_ref,
proj/src/graph_io.cpp): the same graph (n, edges in edge-id order, exactness)
or the same ParseError message and line, case by case. The corpus holds the
reference's own tests (proj/tests/test_graph_io.cpp:40-112) and a seeded
fuzz corpus of mutated lines."""
import random

import numpy as np
import pytest

import oracle as O
import paper_1111_0627_b200 as P

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")

REFERENCE_CASES = [
    # test_graph_io.cpp:40 problem line format, 1-based arcs
    "c comment\np ocm 3 3\na 1 2 5\na 2 3 7\na 3 1 0\n",
    # :57 plain edge list, inferred size, float weight
    "# plain\n0 1 2.5\n1 0 -1\n",
    # :65 errors carry the line number, and the other error cases there
    "p ocm 2 1\nx 1 2 3\n",
    "p ocm 2 2\na 1 2 0\n",
    "p ocm 2 0\na 1 2 0\n",
    "p wrong 2 1\na 1 2 0\n",
    "a 1 2 0\n",
    "0 1 zero\n",
    "0 1\n",
    "",
    "p ocm 2 1\na 1 2 inf\n",
]

EXTRA_CASES = [
    "\n\n   \n", "c only\n", "p ocm 0 0\n", "p ocm -1 0\n", "p ocm 2 -1\n", "p ocm 2\n",
    "p ocm x 1\n", "p ocm 2 y\n", "p ocm 2 1\np ocm 2 1\n", "p ocm 2 1\na 0 1 3\n",
    "p ocm 2 1\na 1 3 3\n", "p ocm 2 1\na 1 2\n", "p ocm 2 1\na 1 2 3 4\n",
    "p ocm 2 1\na 1 2 0x10\n", "p ocm 2 1\na 1 2 nan\n", "p ocm 2 1\na 1 2 1e400\n",
    "p ocm 2 1\na 1 2 +3\n", "p ocm 2 1\na +1 2 3\n", "p ocm 2 1\n# hash\n",
    "p ocm 2 1\r\na 1 2 3\r\n", "c\tx\np\tocm\t2\t1\na 1 2 -7.25", "0 0 1", "0 1 1\n#x\n1 0 2",
    "#only comment\n", "0 -1 2\n", "5 3 2\n", "0 1 2 3\n", "0 1 2\n1\n",
    "0 1 99999999999999999999\n", "0 1 1e-310\n", "1 0 3\n0 1 4\n1 0 5\n",
    "0 1 2\nc 1 2\n", "p ocm 3 2\nc between\na 3 1 1\n\na 1 3 2\n",
    "0 1 9007199254740993\n", "0 1 4.5e15\n", "0 1 12345678901234567\n",
    "p ocm 3 1\na 1 99999999999999999999 2\n", "0 1 2\x00\n",
]


def _fuzz_cases(seed=1234, count=300):
    rnd = random.Random(seed)
    atoms = ["p", "ocm", "a", "c", "#", "0", "1", "2", "3", "-1", "7", "2.5", "x", "1e3",
             "inf", "", "\t", "  ", "-0", "0x1p3", "4294967295"]
    out = []
    for _ in range(count):
        lines = []
        if rnd.random() < 0.5:
            lines.append(f"p ocm {rnd.randint(0, 4)} {rnd.randint(0, 4)}")
        for _ in range(rnd.randint(0, 5)):
            if rnd.random() < 0.6:
                kind = rnd.choice(["a", "", "c", "#"])
                lines.append(" ".join([kind] + [rnd.choice(atoms) for _ in range(rnd.randint(0, 4))]).strip())
            else:
                lines.append(" ".join(rnd.choice(atoms) for _ in range(rnd.randint(0, 5))))
        out.append("\n".join(lines) + ("\n" if rnd.random() < 0.7 else ""))
    return out


def _ours(text):
    try:
        g = P.parse_graph_text(text, "mem")
    except P.ParseError as e:
        return ("parse", str(e), e.line)
    except ValueError as e:  # std::invalid_argument from build_graph
        return ("error", str(e))
    s, d, w = g.edges()
    return ("ok", g.n, s, d, w, g.integer_exact)


def _same(a, b):
    if a[0] != b[0]:
        return False
    if a[0] != "ok":
        return tuple(a) == tuple(b)
    return (a[1] == b[1] and np.array_equal(a[2], b[2]) and np.array_equal(a[3], b[3])
            and np.array_equal(a[4].view(np.uint64), b[4].view(np.uint64)) and a[5] == b[5])


@pytest.mark.parametrize("text", REFERENCE_CASES + EXTRA_CASES)
def test_parser_matches_reference(text):
    ref = O.ref_parse_graph_text(text, "mem")
    assert _same(_ours(text), ref), (text, _ours(text)[:3], ref[:3])


def test_parser_fuzz_matches_reference():
    bad = []
    for text in _fuzz_cases():
        ours, ref = _ours(text), O.ref_parse_graph_text(text, "mem")
        if not _same(ours, ref):
            bad.append((text, ours[:3], ref[:3]))
    assert not bad, bad[:5]


def test_read_graph_file_matches_reference(tmp_path):
    p = tmp_path / "g.txt"
    text = "# two components\n0 1 3\n1 0 5\n2 3 1.5\n3 2 -2\n"
    p.write_text(text)
    g = P.read_graph_file(str(p))
    ref = O.ref_parse_graph_text(text, str(p))
    assert _same(("ok", g.n, *g.edges(), g.integer_exact), ref)
