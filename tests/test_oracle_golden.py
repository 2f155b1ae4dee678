"""CPU: pin the C oracle (oracle/bitgnn_oracle.c) before trusting it.

1. The reference's own known-answer tests (proj/tests/*.cpp), restated.
2. Fixtures produced by the REAL reference (tests/golden/make_golden.py via
   oracle/_ref): inputs, FRDC arrays, every trace point and the logits must
   hash identically.
3. Where oracle/_ref is present (dev container), direct oracle-vs-reference
   runs on more seeds.
"""
import hashlib
import json
import math
import os

import numpy as np
import pytest

import pyoracle as po

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "reference_fixtures.json")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# ---------------------------------------------------------------- KATs -------
def test_binarize_kat():
    # ref: test_bitdense.cpp:54-68
    b = po.binarize(np.array([[0.5, -2.0, -0.1, 0.0]], np.float32))
    assert b[0, 0] == 0x90000000


def test_scale_kats():
    # ref: test_bitdense.cpp:70-101
    assert po.l1_scales(np.array([[1, -3, 2, -2]], np.float32), po.ROW)[0] == 2.0
    s = po.l1_scales(np.array([[1, -4, 0], [3, 2, 0]], np.float32), po.COL)
    assert list(s[:2]) == [2.0, 3.0] and s[2] == np.float32(1e-12)


def test_transpose_kat_and_involution():
    # ref: test_bitdense.cpp:172-199
    rng = po.Rng(5)
    for (r, c, wb) in [(32, 32, 32), (70, 45, 32), (33, 100, 64)]:
        x = rng.random_dense(r, c)
        b = po.binarize(x, wb)
        t = po.transpose_bits(b, r, c, wb)
        assert np.array_equal(po.transpose_bits(t, c, r, wb), b)
        assert np.array_equal(t, po.binarize(np.ascontiguousarray(x.T), wb))


def test_payload_sizes():
    # ref: test_bitdense.cpp:201-213 -- Cora 2708 x 1433: 487,440 B @32, 498,272 B @64
    assert 2708 * po.spw(1433, 32) * 4 == 487440
    assert 2708 * po.spw(1433, 64) * 4 == 498272


def test_frdc_kats():
    # ref: test_bitsparse.cpp:31-67
    m = po.frdc_from_edges(8, [1, 0], [2, 5], False)
    assert list(m.row_ptr) == [0, 2, 2] and list(m.col_ind) == [0, 1]
    assert list(m.tiles) == [0x0200, 0x4000]
    m = po.frdc_from_edges(4, [0, 1, 1, 2, 2, 3], [1, 0, 2, 1, 3, 2], True)
    assert list(m.tiles) == [0xCE73]
    m = po.frdc_from_edges(6, [0, 0, 0, 5, 2], [3, 3, 3, 5, 4], False)
    assert m.nnz_bits() == 3
    m = po.frdc_from_edges(10, [], [], False)
    assert m.nnz == 0 and list(m.row_ptr) == [0, 0, 0, 0]
    with pytest.raises(ValueError):
        po.frdc_from_edges(4, [0, 2], [1, 9], False)


def test_frdc_matches_dense_definition():
    # ref: test_bitsparse.cpp:83-115 (random graphs, tiles never empty, columns increase)
    rng = po.Rng(5)
    for it in range(30):
        n = rng.range(1, 200)
        s, d = rng.random_edges(n, rng.range(0, 4 * n), True)
        loops = bool(it % 2)
        m = po.frdc_from_edges(n, s, d, loops)
        dense = np.zeros((n, n), bool)
        dense[s, d] = True
        if loops:
            dense[np.arange(n), np.arange(n)] = True
        got = np.zeros((n, n), bool)
        for tr in range((n + 3) // 4):
            prev = -1
            for k in range(m.row_ptr[tr], m.row_ptr[tr + 1]):
                assert m.tiles[k] != 0 and m.col_ind[k] > prev
                prev = m.col_ind[k]
                for r in range(4):
                    for c in range(4):
                        if (m.tiles[k] >> (15 - (4 * r + c))) & 1:
                            got[4 * tr + r, 4 * m.col_ind[k] + c] = True
        assert np.array_equal(got, dense)


def test_normalized_two_node_kat():
    # ref: test_graphops.cpp:117-136
    g = po.Graph(2, np.array([0, 1]), np.array([1, 0]))
    assert list(g.structure.tiles) == [0xCC00]
    assert np.allclose(g.norm, 1 / math.sqrt(2.0))


def test_bundle_kat():
    # ref: test_graphops.cpp:138-153
    g = po.Graph(3, np.array([0, 1, 1, 2]), np.array([1, 0, 2, 2]))
    assert g.structure.nnz_bits() == 6 and g.raw.nnz_bits() == 3
    assert list(g.neighbor_count) == [1, 2, 0]
    assert list(g.mean_row) == [1.0, 0.5, 1.0]


def test_add_kats():
    # ref: test_kernels.cpp:350-377
    f = po.add("ADD.FFF", po.Mat.dense(np.array([[1.5, -2.0]])), po.Mat.dense(np.array([[0.25, 1.0]])))
    assert list(f.f[0]) == [1.75, -1.0]
    a = po.Mat.binary(po.binarize(np.array([[1, 1, -1]], np.float32)), 1, 3)
    b = po.Mat.binary(po.binarize(np.array([[1, -1, -1]], np.float32)), 1, 3)
    assert list(po.add("ADD.BBF", a, b).f[0]) == [2.0, 0.0, -2.0]
    o = po.add("ADD.BBB", a, b)
    assert o.bits[0, 0] >> 29 == 0b110


def test_isolated_node_kat():
    # ref: test_kernels.cpp:305-321
    A = po.frdc_from_edges(3, [1, 2], [2, 1], False)
    X = po.Rng(111).random_dense(3, 5)
    xb = po.Mat.binary(po.binarize(X), 3, 5)
    b = po.bspmm("BSpMM.BBB", A, xb)
    assert b.bits[0, 0] >> 27 == 0b11111
    f = po.bspmm("BSpMM.BBF", A, xb)
    assert np.all(f.f[0] == 0.0)


def test_model_kats_simulated_fc():
    # ref: test_oracle.cpp:222-246 -- FC MM.FBF: logits[1] = -2 * 1.25 * 1.75
    layers = [po.Layer(po.FC, ["MM.FBF"], np.array([[1, -3], [2, 0.5]], np.float32)), po.Layer(po.SOFTMAX)]
    _, lg, pts = po.run_model(layers, None, np.array([[0.5, -2]], np.float32))
    assert [p.label for p in pts] == ["layer0.mm.bin_in", "layer0.mm.bin_w"]
    assert lg[0, 0] == 0.0 and lg[0, 1] == np.float32(-2.0 * 1.25 * 1.75)


def test_model_kat_binary_chain():
    # ref: test_oracle.cpp:248-267
    layers = [po.Layer(po.FC, ["MM.FBB"], np.array([[1, -3], [2, 0.5]], np.float32)),
              po.Layer(po.FC, ["MM.BBF"], np.array([[2], [-4]], np.float32)), po.Layer(po.SOFTMAX)]
    _, lg, pts = po.run_model(layers, None, np.array([[0.5, -2]], np.float32))
    assert [p.label for p in pts] == ["layer0.mm.bin_in", "layer0.mm.bin_w", "layer0.mm.out", "layer1.mm.bin_w"]
    assert pts[2].bits[0, 0] >> 30 == 0b10  # dots [0, -2] -> signs [+1, -1]
    assert lg[0, 0] == 6.0


def test_rng_is_mt19937_64():
    # the C++ standard pins the 10000th output of a default-seeded mt19937_64
    r = po.Rng(5489)
    for _ in range(9999):
        r.next()
    assert r.next() == 9981545732273789042


# ------------------------------------------------------- reference fixtures ---
def _cases():
    with open(GOLDEN) as fh:
        return json.load(fh)["cases"]


@pytest.mark.parametrize("case", _cases(), ids=lambda c: c["name"])
def test_oracle_reproduces_reference_fixtures(case):
    n = case["nodes"]
    s, d = po.Rng(case["graph_seed"]).random_edges(n, case["edge_draws"], False)
    assert sha(s) == case["sha_src"] and sha(d) == case["sha_dst"]
    layers, X = po.build_model(case["model"], case["features"], case["hidden"], case["classes"],
                               case["model_seed"], n, case["plan"])
    assert sha(X) == case["sha_x"]
    for l, (h1, h2) in zip(layers, case["sha_w"]):
        assert (sha(l.w1) if l.w1 is not None else None) == h1
        assert (sha(l.w2) if l.w2 is not None else None) == h2
    g = po.Graph(n, s, d)
    for fr, key in ((g.structure, "frdc_loops"), (g.raw, "frdc_raw")):
        want = case[key]
        assert fr.nnz == want["nnz"]
        assert sha(fr.row_ptr) == want["sha_row_ptr"]
        assert sha(fr.col_ind) == want["sha_col_ind"]
        assert sha(fr.tiles) == want["sha_tiles"]
    assert sha(g.norm) == case["sha_norm"] and sha(g.mean_row) == case["sha_mean_row"]
    assert sha(g.neighbor_count) == case["sha_neighbor_count"]
    out, lg, pts = po.run_model(layers, g, X, word_bits=case["word_bits"])
    assert [p.label for p in pts] == [t["label"] for t in case["trace"]]
    for p, t in zip(pts, case["trace"]):
        assert (p.rows, p.cols, p.word_bits) == (t["rows"], t["cols"], t["word_bits"])
        assert sha(p.bits) == t["sha"], p.label
    assert sha(lg) == case["sha_logits"]
    assert sha(out) == case["sha_out"]


# ----------------------------------------- direct runs against oracle/_ref ---
ref_only = pytest.mark.skipif(not po.ref_available(), reason="oracle/_ref not built here")


@ref_only
@pytest.mark.parametrize("seed", [1, 2, 3])
@pytest.mark.parametrize("model", ["gcn", "sage", "saint"])
def test_oracle_matches_reference_random(model, seed):
    rng = po.Rng(seed)
    n = rng.range(50, 400)
    e = rng.range(n, 12 * n)
    f, h, c = rng.range(5, 80), 2 * rng.range(4, 40), rng.range(2, 9)
    s, d = po.ref_random_edges(seed, n, e, False)
    rg = po.RefGraph(n, s, d)
    rm = po.RefModel(rg, model, f, h, c, seed + 7, n)
    ro, rl, rp = rm.run(c)
    layers, X = po.build_model(model, f, h, c, seed + 7, n)
    o, l, p = po.run_model(layers, po.Graph(n, s, d), X)
    assert [a.label for a in p] == [b.label for b in rp]
    assert all(np.array_equal(a.bits, b.bits) for a, b in zip(p, rp))
    assert np.array_equal(l, rl) and np.array_equal(o, ro)


# ------------------------------------------------------------- tile sets -----
def _ten_tile_row():
    # ref: test_bitsparse.cpp:131-135 -- node 0 -> nodes 0, 4, ..., 36
    return po.frdc_from_edges(40, np.zeros(10, np.int64), 4 * np.arange(10, dtype=np.int64), False)


def test_tileset_kat_ten_tiles():
    # ref: test_bitsparse.cpp:131-161
    m = _ten_tile_row()
    assert m.nnz == 10
    assert po.tileset_count(m, 0, 32) == 2 and po.tileset_count(m, 0, 64) == 1
    assert po.tileset_count(m, 1, 32) == 0
    ts0, r0, c0 = po.gather_tileset(m, 0, 0, 32)
    ts1, r1, c1 = po.gather_tileset(m, 0, 1, 32)
    assert ts0 == 8 and c0[:8] == list(range(8))
    assert c1[0] == 8 and c1[1] == 9 and sum(c == po.PAD_COL for c in c1[2:8]) == 6
    assert r0[0] == 0x88888888 and r1[0] == 0x88000000 and r1[1] == 0
    tsw, rw, cw = po.gather_tileset(m, 0, 0, 64)
    assert tsw == 16 and rw[0] == 0x8888888888000000 and cw[10] == po.PAD_COL


@pytest.mark.parametrize("args,msg", [((0, 0, 16), "word_bits must be 32 or 64"),
                                      ((10, 0, 32), "tile_row out of range"),
                                      ((-1, 0, 32), "tile_row out of range"),
                                      ((0, 2, 32), "set_index out of range"),
                                      ((1, 0, 32), "set_index out of range")])
def test_gather_tileset_rejects_like_the_reference(args, msg):
    # ref: bitsparse.cpp:137-143
    with pytest.raises(ValueError, match=msg):
        po.gather_tileset(_ten_tile_row(), *args)


@pytest.mark.parametrize("word_bits", [32, 64])
def test_gather_reassembles_the_stored_tile_bits(word_bits):
    # ref: test_bitsparse.cpp:163-197 -- every assembled bit against frdc_to_dense
    rng = po.Rng(7)
    for it in range(25):
        n = 1 + rng.index(120)
        m_edges = rng.index(6 * n + 1)
        src, dst = rng.random_edges(n, m_edges, True)
        m = po.frdc_from_edges(n, src, dst, False)
        dense = po.frdc_to_dense(m)
        ts = word_bits // 4
        for tr in range((n + 3) // 4):
            for s in range(po.tileset_count(m, tr, word_bits)):
                g_ts, rows, cols = po.gather_tileset(m, tr, s, word_bits)
                assert g_ts == ts
                for slot in range(ts):
                    tc = cols[slot]
                    for r in range(4):
                        for c in range(4):
                            got = (rows[r] >> (word_bits - 1 - (4 * slot + c))) & 1
                            gi, gj = 4 * tr + r, (-1 if tc == po.PAD_COL else 4 * tc + c)
                            want = gj >= 0 and gi < n and gj < n and \
                                (int(dense[gi, gj // 32]) >> (31 - gj % 32)) & 1
                            assert got == int(bool(want))


def test_frdc_to_dense_matches_edge_set():
    rng = po.Rng(3)
    n = 77
    src, dst = rng.random_edges(n, 300, True)
    m = po.frdc_from_edges(n, src, dst, True)
    d = po.frdc_to_dense(m, 64)
    assert d.shape == (n, po.spw(n, 64))
    want = set(zip(src.tolist(), dst.tolist())) | {(i, i) for i in range(n)}
    got = {(i, j) for i in range(n) for j in range(n) if (int(d[i, j // 32]) >> (31 - j % 32)) & 1}
    assert got == want


@pytest.mark.skipif(not po.ref_available(), reason="oracle/_ref not built")
def test_tileset_oracle_matches_reference_library():
    # the real reference's gather_tileset / frdc_to_dense through oracle/_ref
    rng = po.Rng(11)
    for it in range(6):
        n = 5 + rng.index(200)
        src, dst = rng.random_edges(n, rng.index(8 * n + 1), True)
        m = po.frdc_from_edges(n, src, dst, False)
        for wb in (32, 64):
            assert np.array_equal(po.frdc_to_dense(m, wb), po.ref_frdc_to_dense(m, wb))
            for tr in range((n + 3) // 4):
                for s in range(po.tileset_count(m, tr, wb)):
                    assert po.gather_tileset(m, tr, s, wb) == po.ref_gather_tileset(m, tr, s, wb)
