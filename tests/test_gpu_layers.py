"""Single-layer entry points (ref: gcn_layer / sage_layer / graphconv_layer,
graphops.hpp:94-105, graphops.cpp:270-335) on the device against the real
reference's own layer functions (oracle/_ref, ref_layer_run): the result
bit-exact (B) or exactly equal (F), every BIN point recorded by the hooks
identical and in the same order, and the reference's error messages.  Through
the Python mirror and the C ABI it calls."""
import numpy as np
import pytest
import torch

import pyoracle as po
from helpers import bits_equal

import paper_2305_02522_b200 as bg

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not po.ref_available(), reason="oracle/_ref (reference library) not built")]

GCN, SAGE, GRAPHCONV = 0, 1, 2
FUNCS = {GCN: bg.gcn_layer, SAGE: bg.sage_layer, GRAPHCONV: bg.graphconv_layer}

CASES = [  # (kind, plan, input F?, hidden, relu)
    (GCN, ["MM.FBB", "BSpMM.BBB"], True, 64, False),
    (GCN, ["MM.BBF", "BSpMM.FBF"], False, 7, False),
    (GCN, ["MM.FBF", "BSpMM.FFF"], True, 24, True),
    (GCN, ["MM.FBB", "BSpMM.BFB"], True, 40, False),
    (GCN, ["MM.BBB", "BSpMM.BBF"], False, 33, True),
    (SAGE, ["MM.FBB", "MM.FBB", "BSpMM.BBB", "ADD.BBF"], True, 64, True),
    (SAGE, ["MM.FBF", "MM.FBF", "BSpMM.FFF", "ADD.FFF"], True, 16, True),
    (SAGE, ["MM.FBF", "MM.FBB", "BSpMM.BBF", "ADD.FFF"], True, 20, False),
    (SAGE, ["MM.BBB", "MM.BBB", "BSpMM.BBB", "ADD.BBB"], False, 32, False),
    (GRAPHCONV, ["MM.FBB", "MM.FBB", "BSpMM.BFB", "ADD.BBF"], True, 48, True),
    (GRAPHCONV, ["MM.FBF", "MM.FBB", "BSpMM.BBF", "ADD.FFF"], True, 12, False),
]


def _graph(n, e, seed):
    src, dst = po.ref_random_edges(seed, n, e, False)
    return bg.prepare_graph(n, src, dst), po.RefGraph(n, src, dst)


def _layer(kind, plan, fin, hidden, relu, seed):
    rng = np.random.default_rng(seed)
    w1 = rng.uniform(-1, 1, (fin, hidden)).astype(np.float32)
    w2 = rng.uniform(-1, 1, (fin, hidden)).astype(np.float32) if kind != GCN else None
    return bg.LayerSpec(kind, plan, w1, w2, relu)


@pytest.mark.parametrize("word_bits", [32, 64])
@pytest.mark.parametrize("case", range(len(CASES)))
def test_layer_matches_reference_layer_function(case, word_bits):
    kind, plan, f_in, hidden, relu = CASES[case]
    n, fin = 700 + 13 * case, 50 + case
    g, rg = _graph(n, 6 * n, 100 + case)
    rng = np.random.default_rng(case)
    x = rng.uniform(-1, 1, (n, fin)).astype(np.float32)
    if f_in:
        mine_x, ref_x = torch.from_numpy(x).cuda(), x
    else:
        bits = po.binarize(x, word_bits)
        mine_x = bg.BitOperand(bg.BitDenseMatrix.from_numpy(bits, n, fin, word_bits))
        ref_x = (bits, n, fin)
    layer = _layer(kind, plan, fin, hidden, relu, 7 + case)
    trace = []
    got = FUNCS[kind](mine_x, layer, g, trace=trace, prefix="layer3.", word_bits=word_bits)
    want, ref_pts = po.ref_layer_run(rg, layer, ref_x, word_bits, "layer3.", x_word_bits=word_bits)
    assert [p.label for p in trace] == [p.label for p in ref_pts]
    assert all(p.label.startswith("layer3.") for p in trace)
    for p, q in zip(trace, ref_pts):
        assert (p.bits.rows, p.bits.cols, p.bits.word_bits) == (q.rows, q.cols, q.word_bits), p.label
        assert bits_equal(p.bits.numpy(), q.bits), p.label
    if isinstance(want, tuple):
        assert isinstance(got, bg.BitOperand)
        bits, r, c, wb = want
        assert (got.bits.rows, got.bits.cols, got.bits.word_bits) == (r, c, wb)
        assert bits_equal(got.bits.numpy(), bits)
    else:
        assert isinstance(got, torch.Tensor)
        assert np.array_equal(got.cpu().numpy(), want)


def test_layer_outputs_chain_like_run_model():
    # two layer calls compose to the model forward (default GCN plan)
    n, f, h, c = 900, 60, 32, 5
    g, _ = _graph(n, 5000, 3)
    layers, X = bg.build_model_spec("gcn", f, h, c, 99, n, None)
    x = torch.from_numpy(X).cuda()
    h1 = bg.gcn_layer(x, layers[0], g, prefix="layer0.")
    h2 = bg.gcn_layer(h1, layers[1], g, prefix="layer1.")
    logits = bg.Model(layers, g).forward_traced(x)[1]
    assert torch.equal(h2, logits)


def test_layer_errors_are_the_references():
    n = 64
    g, _ = _graph(n, 300, 5)
    x = torch.zeros((n, 8), dtype=torch.float32, device="cuda")
    w = np.ones((8, 4), np.float32)
    with pytest.raises(bg.InvalidArgument, match=r"gcn_conv: expected \{mm, spmm\} plan and weights"):
        bg.gcn_layer(x, bg.LayerSpec(GCN, ["MM.FBB"], w), g)
    with pytest.raises(bg.InvalidArgument,
                       match=r"expected \{mm_self, mm_neigh, spmm, add\} plan and two weight matrices"):
        bg.sage_layer(x, bg.LayerSpec(SAGE, ["MM.FBB", "MM.FBB", "BSpMM.BBB", "ADD.BBF"], w), g)
    with pytest.raises(bg.InvalidArgument, match="inner dimensions"):
        bg.gcn_layer(x, bg.LayerSpec(GCN, ["MM.FBB", "BSpMM.BBB"], np.ones((9, 4), np.float32)), g)
    # the reference's message for the same fault, unwrapped (no "layer i")
    _, rg = _graph(n, 300, 5)
    with pytest.raises(ValueError) as ref_err:
        po.ref_layer_run(rg, bg.LayerSpec(GCN, ["MM.FBB", "BSpMM.BBB"], np.ones((9, 4), np.float32)),
                         np.zeros((n, 8), np.float32))
    with pytest.raises(bg.InvalidArgument) as mine:
        bg.gcn_layer(x, bg.LayerSpec(GCN, ["MM.FBB", "BSpMM.BBB"], np.ones((9, 4), np.float32)), g)
    assert str(mine.value) == str(ref_err.value)
