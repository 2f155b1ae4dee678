"""Graph file readers (ref: graphio.cpp:72-176) against the reference's own
readers (oracle/_ref) on the same text: node counts, edges in order, weight
columns and every error message identical.  Cases: the reference CLI tests'
files (test_cli.cpp:91-163) plus edge cases of the grammar and random files."""
import os

import numpy as np
import pytest

import pyoracle as po

import paper_2305_02522_b200 as bg

pytestmark = pytest.mark.skipif(not po.ref_available(), reason="oracle/_ref (reference library) not built")

EDGE_LISTS = [
    "# a comment\n1 2\n0 5\n", "0 1\n", "0 1\nfoo bar\n", "# nothing here\n", "", "\n\n  \t\n",
    "0 1 x\n", "0 1 2.5\n1 2\n3 4 -7e-1\n", "0 -1\n", "-3 1\n", "1 2 3 4\n", "1 2\r\n3 4\r\n", "% mm-style comment\n2 2\n",
    "1\n", "1 2 -\n", "1 2 -x\n", "1 2 .\n", "1 2 1e\n", "1 2 +5\n", "+1 +2\n", "1.5 2\n", "3abc 4\n",
    "99999999999999999999 1\n", "9223372036854775807 1\n", "0x10 2\n", "   7    8   \n", "1 2 #tail\n",
    "5 5\n5 6\n6 5\n", "1 2 1e400\n", "4 3", "\t1\t2\t0.25", "1 2 nan\n", "1 2 inf\n",
]

MATRIX_MARKET = [
    "%%MatrixMarket matrix coordinate real symmetric\n3 3 2\n2 1 0.5\n3 3 1.0\n",
    "%%MatrixMarket matrix coordinate real general\n3 3 3\n1 1 1.0\n2 2 1.0\n",
    "%%MatrixMarket matrix coordinate pattern general\n% comment\n\n4 4 3\n1 2\n2 3\n4 1\n",
    "%%MatrixMarket matrix coordinate integer symmetric\n2 2 1\n1 2 7\n",
    "%%MatrixMarket matrix array real general\n2 2\n", "%%MatrixMarket matrix coordinate complex general\n",
    "%%MatrixMarket matrix coordinate real hermitian\n", "%%MatrixMarket matrix coordinate real general\n",
    "%%MatrixMarket matrix coordinate real general\n% only comments\n",
    "%%MatrixMarket matrix coordinate real general\n2 3 1\n1 1 1\n",
    "%%MatrixMarket matrix coordinate real general\n0 0 0\n", "%%MatrixMarket matrix coordinate real general\nx y z\n",
    "%%MatrixMarket matrix coordinate real general\n3 3 1\n1 4 1.0\n",
    "%%MatrixMarket matrix coordinate real general\n3 3 1\n1 2\n", "%%MatrixMarket matrix coordinate real general\n3 3 1\nfoo\n",
    "%%MatrixMarket matrix coordinate pattern general\n3 3 2\n1 2\n", "", "\n", "garbage\n",
    "%%MatrixMarket matrix coordinate pattern general\n3 3 1\n1 2 extra\n",
]


def _both(kind, text, *args):
    try:
        want = po.ref_read_graph(kind, text, *args)
    except ValueError as e:
        want = ("error", str(e))
    try:
        if kind == 0:
            e = bg.read_edge_list(text, *args)
        elif kind == 1:
            e = bg.read_matrix_market(text, args[0], *args[2:])
        else:
            e = bg.load_graph(text, *args[1:])
        got = (e.node_count, e.src, e.dst, e.weights)
    except bg.RuntimeFailure as ex:
        got = ("error", str(ex))
    return got, want


def _same(got, want):
    if want[0] == "error" or got[0] == "error":
        assert got == want
        return
    assert got[0] == want[0]
    for a, b in zip(got[1:], want[1:]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("undirected", [False, True])
@pytest.mark.parametrize("forced", [-1, 10])
@pytest.mark.parametrize("text", EDGE_LISTS)
def test_edge_list_matches_reference(text, forced, undirected):
    _same(*_both(0, text, "edges.txt", forced, undirected))


@pytest.mark.parametrize("undirected", [False, True])
@pytest.mark.parametrize("text", MATRIX_MARKET)
def test_matrix_market_matches_reference(text, undirected):
    _same(*_both(1, text, "g.mtx", -1, undirected))


def test_random_edge_files_match_reference():
    rng = np.random.default_rng(5)
    for it in range(40):
        n = int(rng.integers(1, 60))
        lines = []
        for _ in range(int(rng.integers(0, 200))):
            s, d = rng.integers(0, n, 2)
            r = rng.random()
            if r < 0.1:
                lines.append("# c")
            elif r < 0.4:
                lines.append(f"{s} {d} {rng.normal():.6g}")
            else:
                lines.append(f"{s}\t{d}")
        text = "\n".join(lines) + ("\n" if it % 2 else "")
        _same(*_both(0, text, "r.txt", -1 if it % 3 else 64, bool(it % 4 == 1)))


def test_load_graph_sniffs_text_formats(tmp_path):
    files = {"a.txt": "# c\n0 3\n2 1 0.5\n", "b.mtx": "%%MatrixMarket matrix coordinate pattern symmetric\n4 4 2\n1 2\n3 3\n",
             "c.txt": "0 1\nbad\n"}
    for name, text in files.items():
        p = tmp_path / name
        p.write_text(text)
        for forced, und in ((-1, False), (8, True)):
            _same(*_both(2, str(p), "", forced, und))
    _same(*_both(2, str(tmp_path / "missing.txt"), "", -1, False))


def test_load_graph_on_a_large_edge_file(tmp_path):
    # 200k lines: same edges as the reference, parsed without per-line streams
    rng = np.random.default_rng(11)
    s, d = rng.integers(0, 50000, (2, 200000))
    p = tmp_path / "big.txt"
    p.write_text("".join(f"{a} {b}\n" for a, b in zip(s, d)))
    e = bg.load_graph(str(p))
    assert e.node_count == max(s.max(), d.max()) + 1
    assert np.array_equal(e.src, s) and np.array_equal(e.dst, d)
    _same((e.node_count, e.src, e.dst, e.weights), po.ref_read_graph(2, str(p)))
