"""Models built from every layer kind -- FC (all MM variants incl. the
full-precision MM.FFF), Aggregate, Relu, BatchNorm, Scale, Binarize, GCN,
SAGE, GraphConv, Softmax -- on the device against the UNMODIFIED reference
engine (bitgnn::run_model through oracle/_ref) on the same inputs: every BIN
point bit for bit, the output within the reference's own tolerance
(|e-o|/max(1,|o|) <= 1e-6, test_acceptance.cpp:139-268) and the classes equal.
Also: the SCL-eliminated model gives the same device results."""
import numpy as np
import pytest
import torch

import pyoracle as po
from helpers import bits_equal, rel_err

import paper_2305_02522_b200 as bg
from paper_2305_02522_b200 import _lib as L

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not po.ref_available(), reason="oracle/_ref (reference library) not built")]

N, E = 300, 2400


def _w(rng, a, b):
    return rng.uniform(-1, 1, (a, b)).astype(np.float32)


def _bn(rng, c):
    return (rng.uniform(0.5, 1.5, c).astype(np.float32), rng.uniform(-0.5, 0.5, c).astype(np.float32),
            rng.uniform(-0.3, 0.3, c).astype(np.float32), rng.uniform(0.5, 2.0, c).astype(np.float32))


def _scale(rng, rows, cols):
    return bg.LayerSpec(L.LAYER_SCALE, scale_row=(0.25 + rng.uniform(size=rows)).astype(np.float32),
                        scale_col=(0.25 + rng.uniform(size=cols)).astype(np.float32))


def _models(rng, f):
    S = bg.LayerSpec
    return {
        "fc_fff_bn_relu_bin": [S(L.LAYER_FC, ["MM.FFF"], _w(rng, f, 12)), S(L.LAYER_BATCHNORM, bn=_bn(rng, 12)),
                               S(L.LAYER_RELU), S(L.LAYER_BINARIZE), S(L.LAYER_FC, ["MM.BBF"], _w(rng, 12, 5)),
                               S(L.LAYER_SOFTMAX)],
        "scale_bin_scale": [S(L.LAYER_FC, ["MM.FBF"], _w(rng, f, 10)), _scale(rng, N, 10), S(L.LAYER_BINARIZE),
                            S(L.LAYER_FC, ["MM.BBF"], _w(rng, 10, 6)), _scale(rng, N, 6), S(L.LAYER_SOFTMAX)],
        "gcn_aggregate_bn": [S(L.LAYER_GCN, ["MM.FBB", "BSpMM.BBB"], _w(rng, f, 16), relu=True),
                             S(L.LAYER_AGGREGATE, ["BSpMM.BBF"]), S(L.LAYER_BATCHNORM, bn=_bn(rng, 16)),
                             S(L.LAYER_FC, ["MM.FBF"], _w(rng, 16, 4)), S(L.LAYER_SOFTMAX)],
        "aggregate_fff_fc": [S(L.LAYER_AGGREGATE, ["BSpMM.FFF"]), S(L.LAYER_FC, ["MM.FBF"], _w(rng, f, 8), relu=True),
                             S(L.LAYER_AGGREGATE, ["BSpMM.FBF"]), S(L.LAYER_SOFTMAX)],
        "sage_relu_graphconv": [S(L.LAYER_SAGE, ["MM.FBB", "MM.FBB", "BSpMM.BBB", "ADD.BBF"], _w(rng, f, 16),
                                  _w(rng, f, 16), relu=True),
                                S(L.LAYER_GRAPHCONV, ["MM.FBF", "MM.FBF", "BSpMM.FFF", "ADD.FFF"], _w(rng, 16, 5),
                                  _w(rng, 16, 5)),
                                S(L.LAYER_SOFTMAX)],
        "fc_fbb_bin_chain": [S(L.LAYER_FC, ["MM.FBB"], _w(rng, f, 40)), S(L.LAYER_FC, ["MM.BBB"], _w(rng, 40, 24)),
                             S(L.LAYER_AGGREGATE, ["BSpMM.BBF"]), S(L.LAYER_RELU),
                             S(L.LAYER_FC, ["MM.FFF"], _w(rng, 24, 7)), S(L.LAYER_SOFTMAX)],
    }


NAMES = list(_models(np.random.default_rng(0), 8))


@pytest.mark.parametrize("wb", [32, 64])
@pytest.mark.parametrize("name", NAMES)
def test_glue_layer_models_match_reference_engine(name, wb):
    rng = np.random.default_rng(7100 + NAMES.index(name) + wb)
    f = 37
    layers = _models(rng, f)[name]
    src, dst = po.Rng(41).random_edges(N, E, False)
    x = rng.uniform(-1, 1, (N, f)).astype(np.float32)
    assert bg.validate_model(layers) == []
    m = bg.Model(layers, bg.prepare_graph(N, src, dst), word_bits=wb)
    out, logits, pts = m.forward_traced(torch.from_numpy(x).cuda())
    r_out, r_log, r_pts = po.ref_spec_run(layers, po.RefGraph(N, src, dst), x, wb)
    assert [p.label for p in pts] == [p.label for p in r_pts]
    for p, q in zip(pts, r_pts):
        assert bits_equal(p.bits.numpy(), q.bits), p.label
    got = out.cpu().numpy()
    assert rel_err(got, r_out) <= 1e-6
    assert np.array_equal(np.argmax(logits.cpu().numpy(), axis=1), np.argmax(r_log, axis=1))


def test_scl_eliminated_model_gives_identical_device_results():
    rng = np.random.default_rng(7200)
    layers = _models(rng, 37)["scale_bin_scale"]
    src, dst = po.Rng(42).random_edges(N, E, False)
    g = bg.prepare_graph(N, src, dst)
    x = torch.from_numpy(rng.uniform(-1, 1, (N, 37)).astype(np.float32)).cuda()
    a_out, _, a_pts = bg.Model(layers, g).forward_traced(x)
    r = bg.rewrite_eliminate_scl(layers)
    assert len(r) == len(layers) - 1
    b_out, _, b_pts = bg.Model(r, g).forward_traced(x)
    assert len(a_pts) == len(b_pts)
    for p, q in zip(a_pts, b_pts):
        assert torch.equal(p.bits.words, q.bits.words)
    assert torch.equal(a_out, b_out)
