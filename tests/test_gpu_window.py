"""Column-windowed bit-SpMM (window.cu) vs the oracle.  The windowed layout
must give bit-identical BBB / BBF results to the reference for every window
size, row range and degree profile (integer counting is order-free), and the
models that run through it must stay bit-exact end to end."""
import numpy as np
import pytest
import torch

import pyoracle as po
from helpers import bits_equal, to_layer_specs

import paper_2305_02522_b200 as bg
from paper_2305_02522_b200 import _lib as L

pytestmark = pytest.mark.gpu


@pytest.fixture
def window_mode():
    def set_mode(window_nodes=0):
        bg.set_aggregation(L.AGG_WINDOW, window_nodes)
    yield set_mode
    bg.set_aggregation(L.AGG_AUTO, 0)


def cuda(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()


def _bits_operand(X, wb):
    b = po.binarize(X, wb)
    dev = bg.BitOperand(bg.BitDenseMatrix.from_numpy(b, X.shape[0], X.shape[1], wb))
    return dev, po.Mat.binary(b, X.shape[0], X.shape[1], wb)


# (nodes, edge draws, features, word bits, window nodes): features always give
# 4 storage words per row (the windowed kernel's operand shape).
CASES = [
    (5, 9, 128, 32, 0), (37, 150, 97, 32, 3), (64, 900, 128, 32, 7), (300, 30000, 120, 32, 64),
    (1000, 60000, 128, 32, 100), (1000, 60000, 128, 64, 999), (2000, 8000, 70, 64, 128),
    (513, 120000, 128, 32, 33), (4096, 400000, 101, 32, 0), (777, 5000, 128, 32, 1),
    (3000, 600000, 128, 32, 256), (160, 2000, 128, 32, 160),
]


@pytest.mark.parametrize("v", ["BSpMM.BBB", "BSpMM.BBF"])
@pytest.mark.parametrize("case", CASES)
def test_window_bspmm_matches_oracle(window_mode, v, case):
    n, e, f, wb, wn = case
    window_mode(wn)
    rng = po.Rng(7000 + n + e + f + wn)
    s, d = rng.random_edges(n, e, True)
    A = po.frdc_from_edges(n, s, d, True)
    dA = bg.frdc_from_edges(n, s, d, True)
    X = rng.random_dense(n, f)
    dx, ox = _bits_operand(X, wb)
    got = bg.bspmm(v, bg.AdjacencyOperand(dA), dx, None, wb)
    want = po.bspmm(v, A, ox, None, None, wb)
    if want.prec == po.B:
        assert bits_equal(got.bits.numpy(), want.bits)
    else:
        assert np.array_equal(got.cpu().numpy(), want.f)


def test_window_hub_rows_and_isolated_nodes(window_mode):
    # one hub row adjacent to everything (degree > 2^10 -> 12-bit counters),
    # isolated nodes (degree 0 -> bit 1 / 0.0), a full 4x4 tile block
    window_mode(50)
    n = 1500
    src = [0] * n + list(range(8)) * 8 + [700, 701]
    dst = list(range(n)) + [j for j in range(8) for _ in range(8)] + [701, 700]
    rng = po.Rng(91)
    X = rng.random_dense(n, 128)
    A = po.frdc_from_edges(n, np.array(src), np.array(dst), False)
    dA = bg.frdc_from_edges(n, src, dst, False)
    dx, ox = _bits_operand(X, 32)
    for v in ("BSpMM.BBB", "BSpMM.BBF"):
        got = bg.bspmm(v, bg.AdjacencyOperand(dA), dx, None, 32)
        want = po.bspmm(v, A, ox, None, None, 32)
        if want.prec == po.B:
            assert bits_equal(got.bits.numpy(), want.bits)
        else:
            assert np.array_equal(got.cpu().numpy(), want.f)


def test_window_and_slivers_agree_across_window_sizes():
    n, e = 2500, 250000
    rng = po.Rng(93)
    s, d = rng.random_edges(n, e, False)
    dA = bg.frdc_from_edges(n, s, d, True)
    dx, _ = _bits_operand(rng.random_dense(n, 128), 32)
    bg.set_aggregation(L.AGG_SLIVERS, 0)
    try:
        ref = bg.bspmm("BSpMM.BBB", bg.AdjacencyOperand(dA), dx).bits.numpy()
        for wn in (1, 17, 512, 2500, 0):
            bg.set_aggregation(L.AGG_WINDOW, wn)
            got = bg.bspmm("BSpMM.BBB", bg.AdjacencyOperand(dA), dx).bits.numpy()
            assert np.array_equal(got, ref), wn
    finally:
        bg.set_aggregation(L.AGG_AUTO, 0)


def test_aggregation_setting_roundtrip_and_validation():
    bg.set_aggregation(L.AGG_WINDOW, 123)
    try:
        assert bg.get_aggregation() == (L.AGG_WINDOW, 123)
        with pytest.raises(bg.InvalidArgument):
            bg.set_aggregation(9, 0)
        with pytest.raises(bg.InvalidArgument):
            bg.set_aggregation(L.AGG_AUTO, 70000)
    finally:
        bg.set_aggregation(L.AGG_AUTO, 0)
    assert bg.get_aggregation() == (L.AGG_AUTO, 0)


@pytest.mark.parametrize("model,h", [("gcn", 128), ("saint", 128), ("sage", 128)])
def test_dense_graph_models_bit_exact_in_window_mode(window_mode, model, h):
    # a small dense graph (average degree ~120) through the whole engine with
    # the windowed aggregation forced; graph-captured replays agree
    window_mode(300)
    n, e, f, c = 3000, 360000, 300, 41
    s, d = po.Rng(100).random_edges(n, e, False)
    layers, X = po.build_model(model, f, h, c, 99, n)
    o_out, o_log, o_pts = po.run_model(layers, po.Graph(n, s, d), X)
    m = bg.Model(to_layer_specs(bg, layers), bg.prepare_graph(n, s, d))
    out, logits, pts = m.forward_traced(cuda(X))
    assert [p.label for p in pts] == [p.label for p in o_pts]
    for p, q in zip(pts, o_pts):
        assert bits_equal(p.bits.numpy(), q.bits), p.label
    assert np.array_equal(logits.cpu().numpy(), o_log)
    for _ in range(3):
        out2 = m.forward(cuda(X))
    torch.cuda.synchronize()
    assert torch.equal(out2, out)
    assert np.allclose(out.cpu().numpy(), o_out, rtol=1e-6, atol=1e-7)


# Every aggregation layout on the same operands: AUTO picks the row-group
# kernel for short rows and the window/sliver kernels otherwise; SLIVERS and
# TILES force the gather kernels.  All must agree with the oracle bit for bit.
@pytest.mark.parametrize("mode", [L.AGG_AUTO, L.AGG_SLIVERS, L.AGG_TILES, L.AGG_WINDOW])
@pytest.mark.parametrize("v", ["BSpMM.BBB", "BSpMM.BBF"])
@pytest.mark.parametrize("nef", [(2000, 9000, 128), (1500, 30000, 64), (700, 2000, 250), (96, 3000, 31),
                                 (5000, 20000, 100), (300, 60000, 128)])
def test_every_layout_matches_oracle(mode, v, nef):
    n, e, f = nef
    rng = po.Rng(9100 + n + e + f)
    s, d = rng.random_edges(n, e, True)
    A = po.frdc_from_edges(n, s, d, True)
    dA = bg.frdc_from_edges(n, s, d, True)
    X = rng.random_dense(n, f)
    dx, ox = _bits_operand(X, 32)
    bg.set_aggregation(mode, 0)
    try:
        got = bg.bspmm(v, bg.AdjacencyOperand(dA), dx, None, 32)
    finally:
        bg.set_aggregation(L.AGG_AUTO, 0)
    want = po.bspmm(v, A, ox, None, None, 32)
    if want.prec == po.B:
        assert bits_equal(got.bits.numpy(), want.bits)
    else:
        assert np.array_equal(got.cpu().numpy(), want.f)


@pytest.mark.parametrize("cols", [1, 7, 41, 47, 48, 64, 65, 130])
def test_softmax_rows_matches_oracle(cols):
    rng = po.Rng(9300 + cols)
    X = (rng.random_dense(1000, cols) * 30.0).astype(np.float32)
    X[3, :] = -np.inf if cols > 1 else X[3, :]
    X[5, 0] = 80.0
    X[7, cols // 2] = np.nan
    got = bg.softmax_rows(cuda(X)).cpu().numpy()
    want = po.softmax_rows(X)
    assert np.array_equal(np.isnan(got), np.isnan(want))
    ok = np.isfinite(want)
    assert np.allclose(got[ok], want[ok], rtol=1e-6, atol=1e-12)


@pytest.mark.parametrize("tpr", ["1", "2"])
@pytest.mark.parametrize("v", ["BSpMM.BBB", "BSpMM.BBF"])
def test_window_threads_per_row_variants(window_mode, monkeypatch, tpr, v):
    # both thread mappings of the windowed kernel (one or two threads per row)
    monkeypatch.setenv("BG_WINDOW_TPR", tpr)
    window_mode(97)
    n, e, f = 3000, 200000, 128
    rng = po.Rng(9500)
    s, d = rng.random_edges(n, e, True)
    A = po.frdc_from_edges(n, s, d, True)
    dA = bg.frdc_from_edges(n, s, d, True)
    dx, ox = _bits_operand(rng.random_dense(n, f), 32)
    got = bg.bspmm(v, bg.AdjacencyOperand(dA), dx, None, 32)
    want = po.bspmm(v, A, ox, None, None, 32)
    if want.prec == po.B:
        assert bits_equal(got.bits.numpy(), want.bits)
    else:
        assert np.array_equal(got.cpu().numpy(), want.f)


def _power_law_edges(n, e, seed, a=1.4):
    """Directed edges with Zipf-distributed endpoints (heavy-tailed degrees:
    a few rows of thousands of neighbours next to rows of one or two)."""
    g = np.random.default_rng(seed)
    perm = g.permutation(n)
    s = perm[np.minimum(g.zipf(a, e), n) - 1]
    d = perm[np.minimum(g.zipf(a, e), n) - 1]
    mix = g.random(e) < 0.5  # half the draws uniform, so most rows are non-empty
    s = np.where(mix, g.integers(0, n, e), s)
    return s.astype(np.int64), d.astype(np.int64)


@pytest.mark.parametrize("mode", [L.AGG_AUTO, L.AGG_WINDOW, L.AGG_SLIVERS])
@pytest.mark.parametrize("v", ["BSpMM.BBB", "BSpMM.BBF"])
def test_skewed_degree_graph_every_layout(mode, v):
    # the windowed kernel gives a warp's 32 rows one loop count per step: on a
    # heavy-tailed degree profile (max degree in the thousands) the rows of a
    # warp are far apart -- results must stay exact
    n, e = 20000, 1_500_000
    s, d = _power_law_edges(n, e, 17)
    A = po.frdc_from_edges(n, s, d, True)
    dA = bg.frdc_from_edges(n, s, d, True)
    assert dA.info().max_row_degree > 2000
    X = po.Rng(17).random_dense(n, 128)
    dx, ox = _bits_operand(X, 32)
    bg.set_aggregation(mode, 0)
    try:
        got = bg.bspmm(v, bg.AdjacencyOperand(dA), dx, None, 32)
    finally:
        bg.set_aggregation(L.AGG_AUTO, 0)
    want = po.bspmm(v, A, ox, None, None, 32)
    if want.prec == po.B:
        assert bits_equal(got.bits.numpy(), want.bits)
    else:
        assert np.array_equal(got.cpu().numpy(), want.f)


@pytest.mark.parametrize("mode", [L.AGG_AUTO, L.AGG_SLIVERS, L.AGG_TILES])
def test_hub_row_beyond_16_bit_counters(mode):
    # a hub row with ~150 K neighbours (multi-bit nibbles throughout): every
    # layout must count past 2^16 per lane, as the reference does at any degree
    n = 160_000
    hub = np.zeros(150_000, np.int64)
    s = np.concatenate([hub, np.arange(n, dtype=np.int64)])
    d = np.concatenate([np.arange(150_000, dtype=np.int64), (np.arange(n, dtype=np.int64) * 7) % n])
    A = po.frdc_from_edges(n, s, d, True)
    dA = bg.frdc_from_edges(n, s, d, True)
    X = po.Rng(31).random_dense(n, 128)
    dx, ox = _bits_operand(X, 32)
    bg.set_aggregation(mode, 0)
    try:
        for v in ("BSpMM.BBB", "BSpMM.BBF"):
            got = bg.bspmm(v, bg.AdjacencyOperand(dA), dx, None, 32)
            want = po.bspmm(v, A, ox, None, None, 32)
            if want.prec == po.B:
                assert bits_equal(got.bits.numpy(), want.bits)
            else:
                assert np.array_equal(got.cpu().numpy(), want.f)
    finally:
        bg.set_aggregation(L.AGG_AUTO, 0)


def _hub_graph(n, e, seed, a=1.3):
    s, d = _power_law_edges(n, e, seed, a)
    dA = bg.frdc_from_edges(n, s, d, True)
    deg = np.bincount(s[s != d], minlength=n) + 1  # + self loop (upper bound: duplicates merge)
    return s, d, dA, int((deg >= 2048).sum())


@pytest.mark.parametrize("mode", [L.AGG_AUTO, L.AGG_WINDOW, L.AGG_SLIVERS])
@pytest.mark.parametrize("f,wb", [(128, 32), (40, 32), (300, 32), (128, 64)])
def test_hub_rows_split_over_the_gpu(mode, f, wb):
    # rows of degree >= 2048 leave the per-row kernels and are counted by
    # the split hub kernel (hubs.cu): many hubs, every feature width, both
    # outputs -- bit-identical to the reference's per-row walk
    n, e = 60000, 4_000_000
    s, d, dA, hubs = _hub_graph(n, e, 23)
    assert hubs >= 20 and dA.info().max_row_degree > 15000
    A = po.frdc_from_edges(n, s, d, True)
    X = po.Rng(23).random_dense(n, f)
    dx, ox = _bits_operand(X, wb)
    bg.set_aggregation(mode, 0)
    try:
        for v in ("BSpMM.BBB", "BSpMM.BBF"):
            got = bg.bspmm(v, bg.AdjacencyOperand(dA), dx, None, wb)
            want = po.bspmm(v, A, ox, None, None, wb)
            if want.prec == po.B:
                assert bits_equal(got.bits.numpy(), want.bits)
            else:
                assert np.array_equal(got.cpu().numpy(), want.f)
    finally:
        bg.set_aggregation(L.AGG_AUTO, 0)


@pytest.mark.parametrize("world", [1, 3])
def test_hub_graph_model_forward_sharded_and_captured(world):
    # a 3-layer binary GCN on the power-law graph: hub rows in every rank's
    # row range, the forward captured and replayed; equal to the
    # layer-by-layer forward and to the oracle
    from paper_2305_02522_b200.sharded import forward_virtual_ranks, partition_bounds
    n, e, f, h, c = 60000, 4_000_000, 100, 128, 9
    s, d = _power_law_edges(n, e, 29, 1.3)
    plan = ["MM.FBB+BSpMM.BBB", "MM.BBB+BSpMM.BBB", "MM.BBF+BSpMM.FBF"]
    layers, X = po.build_model("gcn", f, h, c, 99, n, plan)
    g = bg.prepare_graph(n, s, d)
    m = bg.Model(to_layer_specs(bg, layers), g)
    x = torch.from_numpy(X).cuda()
    ref_out, ref_log, _ = m.forward_traced(x)
    for _ in range(3):  # eager, captured, replayed
        out = m.forward(x)
        torch.cuda.synchronize()
        assert torch.equal(out, ref_out)
    rp, _, _ = g.structure.download()
    out, lg = forward_virtual_ranks(m, x, partition_bounds(rp, n, world), logits=True)
    torch.cuda.synchronize()
    assert torch.equal(lg, ref_log) and torch.equal(out, ref_out)
    o_out, o_log, _ = po.run_model(layers, po.Graph(n, s, d), X)
    assert np.array_equal(lg.cpu().numpy(), o_log)
