"""Tile sets, dense expansion and FRDC statistics on the device against the
reference's known answers (proj/tests/test_bitsparse.cpp:131-197) and the C
oracle (bitsparse.cpp:114-169): gather_tileset / tileset_count one set at a
time, gather_tilesets for every set of the matrix at once, frdc_to_dense,
frdc_stats."""
import ctypes as C

import numpy as np
import pytest

import pyoracle as po

import paper_2305_02522_b200 as bg

pytestmark = pytest.mark.gpu


def _ten_tile_row():
    # ref: test_bitsparse.cpp:131-135
    return bg.frdc_from_edges(40, np.zeros(10, np.int64), 4 * np.arange(10, dtype=np.int64), False)


def test_ten_tile_row_gathers_into_two_sets_with_six_padded_slots():
    # ref: test_bitsparse.cpp:131-161
    m = _ten_tile_row()
    assert m.nnz_tiles == 10
    assert bg.tileset_count(m, 0, 32) == 2 and bg.tileset_count(m, 0, 64) == 1
    assert bg.tileset_count(m, 1, 32) == 0
    s0, s1 = bg.gather_tileset(m, 0, 0, 32), bg.gather_tileset(m, 0, 1, 32)
    assert s0.ts == 8 and list(s0.cols[:8]) == list(range(8))
    assert s1.cols[0] == 8 and s1.cols[1] == 9
    assert sum(c == bg.bitgnn.PAD_COL for c in s1.cols[2:8]) == 6
    assert s0.rows[0] == 0x88888888 and s1.rows[0] == 0x88000000 and s1.rows[1] == 0
    w = bg.gather_tileset(m, 0, 0, 64)
    assert w.ts == 16 and w.rows[0] == 0x8888888888000000 and w.cols[10] == bg.bitgnn.PAD_COL


@pytest.mark.parametrize("args,msg", [((0, 0, 16), "gather_tileset: word_bits must be 32 or 64"),
                                      ((10, 0, 32), "gather_tileset: tile_row out of range"),
                                      ((-1, 0, 32), "gather_tileset: tile_row out of range"),
                                      ((0, 2, 32), "gather_tileset: set_index out of range"),
                                      ((1, 0, 32), "gather_tileset: set_index out of range")])
def test_gather_tileset_errors_are_the_references(args, msg):
    # ref: bitsparse.cpp:137-143 (std::invalid_argument, same text)
    with pytest.raises(bg.InvalidArgument, match=msg):
        bg.gather_tileset(_ten_tile_row(), *args)


def _sets_of(sets, i):
    rec = sets[i].cpu().numpy().tobytes()
    ts = int(np.frombuffer(rec[:4], np.int32)[0])
    rows = [int(v) for v in np.frombuffer(rec[8:40], np.uint64)]
    cols = [int(v) for v in np.frombuffer(rec[40:104], np.uint32)]
    return ts, rows, cols


@pytest.mark.parametrize("word_bits", [32, 64])
@pytest.mark.parametrize("it", range(6))
def test_tilesets_match_the_oracle_one_by_one_and_batched(word_bits, it):
    rng = po.Rng(70 + it)
    n = 1 + rng.index(160)
    src, dst = rng.random_edges(n, rng.index(10 * n + 1), True)
    mine = bg.frdc_from_edges(n, src, dst, it % 2 == 0)
    ref = po.frdc_from_edges(n, src, dst, it % 2 == 0)
    set_ptr, sets = bg.gather_tilesets(mine, word_bits)
    sp = set_ptr.cpu().numpy()
    for tr in range((n + 3) // 4):
        k = po.tileset_count(ref, tr, word_bits)
        assert bg.tileset_count(mine, tr, word_bits) == k
        assert sp[tr + 1] - sp[tr] == k
        for s in range(k):
            want = po.gather_tileset(ref, tr, s, word_bits)
            got = bg.gather_tileset(mine, tr, s, word_bits)
            assert (got.ts, list(got.rows), list(got.cols)) == want
            assert _sets_of(sets, int(sp[tr]) + s) == want


def test_tilesets_of_a_full_size_tile_row_spread():
    # a graph with long and empty tile rows: the batched gather's row search
    rng = po.Rng(5)
    n = 4096
    src, dst = rng.random_edges(n, 60_000, False)
    src = np.concatenate([src, np.zeros(600, np.int64)])
    dst = np.concatenate([dst, np.arange(600, dtype=np.int64) * 6])
    mine = bg.frdc_from_edges(n, src, dst, True)
    ref = po.frdc_from_edges(n, src, dst, True)
    set_ptr, sets = bg.gather_tilesets(mine, 32)
    sp = set_ptr.cpu().numpy()
    assert int(sp[-1]) == sum(po.tileset_count(ref, tr, 32) for tr in range(n // 4))
    for g in list(range(0, int(sp[-1]), 97)) + [int(sp[-1]) - 1]:
        tr = int(np.searchsorted(sp, g, side="right")) - 1
        assert _sets_of(sets, g) == po.gather_tileset(ref, tr, g - int(sp[tr]), 32)


@pytest.mark.parametrize("word_bits", [32, 64])
@pytest.mark.parametrize("n", [1, 5, 33, 130, 1000])
def test_frdc_to_dense_matches_the_oracle(n, word_bits):
    rng = po.Rng(n)
    src, dst = rng.random_edges(n, 4 * n, True)
    mine = bg.frdc_from_edges(n, src, dst, True)
    ref = po.frdc_from_edges(n, src, dst, True)
    d = bg.frdc_to_dense(mine, word_bits)
    assert d.semantics == bg.bitgnn.ZERO_ONE and (d.rows, d.cols) == (n, n)
    assert np.array_equal(d.numpy(), po.frdc_to_dense(ref, word_bits))


def test_frdc_stats_are_the_references():
    # ref: bitsparse.cpp:162-169
    rng = po.Rng(9)
    n = 500
    src, dst = rng.random_edges(n, 3000, True)
    m = bg.frdc_from_edges(n, src, dst, True)
    ref = po.frdc_from_edges(n, src, dst, True)
    st = bg.frdc_stats(m)
    bits = ref.nnz_bits()
    assert st.nnz_tiles == ref.nnz and st.nnz_bits == bits
    assert st.bytes == (n // 4 + 1) * 8 + ref.nnz * 6
    assert st.fill_ratio == bits / (16.0 * ref.nnz)
    empty = bg.frdc_from_edges(8, np.zeros(0, np.int64), np.zeros(0, np.int64), False)
    e = bg.frdc_stats(empty)
    assert (e.nnz_tiles, e.nnz_bits, e.fill_ratio) == (0, 0, 0.0)
