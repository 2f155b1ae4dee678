"""FRDC container I/O (ref: write_frdc / read_frdc, bitsparse.cpp:171-222),
mirroring proj/tests/test_bitsparse.cpp:199-290: the declared little-endian
byte layout, rejection of foreign and damaged headers, and round trips."""
import struct

import numpy as np
import pytest
import torch

import pyoracle as po
from helpers import bits_equal

import paper_2305_02522_b200 as bg

pytestmark = pytest.mark.gpu


def _expected_bytes(n_rows, n_cols, rp, ci, ti, word_bits):
    """The layout of bitsparse.hpp:92-96, written independently of the library."""
    head = b"FRDC" + struct.pack("<IBBHQQQ", 1, 4, word_bits, 0, n_rows, n_cols, len(ci))
    return (head + np.asarray(rp, "<u8").tobytes() + np.asarray(ci, "<u4").tobytes() +
            np.asarray(ti, "<u2").tobytes())


def test_serialized_bytes_follow_the_declared_layout():
    # ref: test_bitsparse.cpp:199-236 (the reference's own golden bytes)
    m = bg.frdc_from_edges(8, [1, 0], [2, 5], False)
    want = b"FRDC" + struct.pack("<I", 1) + bytes([4, 32]) + struct.pack("<H", 0)
    want += struct.pack("<QQQ", 8, 8, 2) + struct.pack("<QQQ", 0, 2, 2)
    want += struct.pack("<II", 0, 1) + struct.pack("<HH", 0x0200, 0x4000)
    got = m.to_bytes(32)
    assert len(got) == len(want) == 36 + 24 + 8 + 4
    assert got == want


def test_reader_rejects_foreign_and_damaged_headers():
    # ref: test_bitsparse.cpp:237-267 (+ the messages of bitsparse.cpp:30-36, :197-205)
    good = bg.frdc_from_edges(4, [0], [1], False).to_bytes()
    cases = [(b"X" + good[1:], "FRDC: bad magic"),
             (good[:4] + bytes([2]) + good[5:], "FRDC: unsupported version"),
             (good[:8] + bytes([3]) + good[9:], "FRDC: unsupported tile_dim"),
             (good[:9] + bytes([16]) + good[10:], "FRDC: bad word_bits"),
             (good[:10] + bytes([1]) + good[11:], "FRDC: nonzero reserved field"),
             (good[:-1], "FRDC: truncated file"),
             (good[:2], "FRDC: bad magic"),
             (good[:20], "FRDC: truncated file")]
    for data, msg in cases:
        with pytest.raises(bg.RuntimeFailure, match=msg):
            bg.FrdcMatrix.from_bytes(data)


@pytest.mark.parametrize("rows,nnz", [(8, 1 << 63), (8, (1 << 64) - 1), (8, 1 << 40),
                                      ((1 << 62), 0), (8, 3)])
def test_reader_rejects_untrusted_sizes_before_allocating(rows, nnz, tmp_path):
    # crafted headers whose declared arrays overflow size arithmetic or exceed
    # the bytes present: "truncated", never a wrapped size or a huge allocation
    body = struct.pack("<QQQ", 0, 0, 1 << 63) + struct.pack("<I", 0) + struct.pack("<H", 0x8000)
    data = b"FRDC" + struct.pack("<IBBHQQQ", 1, 4, 32, 0, rows, 8, nnz) + body
    with pytest.raises(bg.RuntimeFailure, match="FRDC: truncated file"):
        bg.FrdcMatrix.from_bytes(data)
    p = tmp_path / "crafted.frdc"
    p.write_bytes(data)
    with pytest.raises(bg.RuntimeFailure, match="FRDC: truncated file"):
        bg.FrdcMatrix.read(str(p))


def test_reader_rejects_payload_that_fails_validation():
    # a container whose tiles break the FrdcMatrix invariants (all-zero tile)
    m = bg.frdc_from_edges(8, [1, 0], [2, 5], False)
    data = bytearray(m.to_bytes())
    data[-2:] = b"\x00\x00"
    with pytest.raises(bg.InvalidArgument, match="FRDC: stored all-zero tile"):
        bg.FrdcMatrix.from_bytes(bytes(data))


def test_writer_rejects_bad_word_bits():
    m = bg.frdc_from_edges(4, [0], [1], False)
    with pytest.raises(bg.InvalidArgument, match="word_bits must be 32 or 64"):
        m.to_bytes(16)


@pytest.mark.parametrize("it", range(24))
def test_random_edge_lists_round_trip_through_bytes(it):
    # ref: test_bitsparse.cpp:269-286
    rng = po.Rng(41 + it)
    n = 1 + (it * 389) % 2048
    s, d = rng.random_edges(n, (it * 977) % (3 * n + 1), True)
    loops = bool(it % 2)
    word_bits = 32 if it % 3 else 64
    m = bg.frdc_from_edges(n, s, d, loops)
    data = m.to_bytes(word_bits)
    ref = po.frdc_from_edges(n, s, d, loops)
    assert data == _expected_bytes(n, n, ref.row_ptr, ref.col_ind, ref.tiles, word_bits)
    back, wb = bg.FrdcMatrix.from_bytes(data)
    assert wb == word_bits
    for a, b in zip(back.download(), m.download()):
        assert np.array_equal(a, b)
    assert back.nnz_bits == m.nnz_bits


def test_file_round_trip_and_aggregation_from_a_loaded_graph(tmp_path):
    n, e = 3000, 90000
    rng = po.Rng(77)
    s, d = rng.random_edges(n, e, False)
    m = bg.frdc_from_edges(n, s, d, True)
    path = tmp_path / "g.frdc"
    m.write(path, 64)
    assert path.stat().st_size == len(m.to_bytes())
    back, wb = bg.FrdcMatrix.read(path)
    assert wb == 64
    X = rng.random_dense(n, 128)
    b = po.binarize(X, 32)
    dx = bg.BitOperand(bg.BitDenseMatrix.from_numpy(b, n, 128, 32))
    got = bg.bspmm("BSpMM.BBB", bg.AdjacencyOperand(back), dx)
    want = po.bspmm("BSpMM.BBB", po.frdc_from_edges(n, s, d, True), po.Mat.binary(b, n, 128, 32), None, None, 32)
    assert bits_equal(got.bits.numpy(), want.bits)


def test_missing_file_names_the_path(tmp_path):
    p = tmp_path / "nope.frdc"
    with pytest.raises(bg.RuntimeFailure, match="read_frdc: cannot open .*nope.frdc"):
        bg.FrdcMatrix.read(p)
    m = bg.frdc_from_edges(4, [0], [1], False)
    with pytest.raises(bg.RuntimeFailure, match="write_frdc: cannot open"):
        m.write(tmp_path / "no_dir" / "x.frdc")


@pytest.mark.skipif(not po.ref_available(), reason="oracle/_ref (reference library) not built")
@pytest.mark.parametrize("forced,undirected", [(-1, False), (-1, True), (5000, False), (10, False)])
def test_load_graph_decodes_a_container_like_the_reference(tmp_path, forced, undirected):
    # graphio.cpp:46-70: tiles -> edges in storage order, node count from the
    # header (trailing isolated nodes kept), the forced count checked
    n = 3001  # not a multiple of 4; node 3000 is isolated
    s, d = po.Rng(78).random_edges(3000, 20000, False)
    m = bg.frdc_from_edges(n, s, d, False)
    path = tmp_path / "g.frdc"
    m.write(path)
    try:
        want = po.ref_read_graph(2, str(path), "", forced, undirected)
    except ValueError as e:
        with pytest.raises(bg.RuntimeFailure) as got:
            bg.load_graph(str(path), forced, undirected)
        assert str(got.value) == str(e)
        return
    e = bg.load_graph(str(path), forced, undirected)
    assert e.node_count == want[0]
    assert np.array_equal(e.src, want[1]) and np.array_equal(e.dst, want[2])
    # and the edges rebuild the same adjacency on the device
    back = bg.frdc_from_edges(e.node_count, e.src, e.dst, False)
    if not undirected and forced < 0:
        for a, b in zip(back.download(), m.download()):
            assert np.array_equal(a, b)
