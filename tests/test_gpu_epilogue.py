"""Fused F-output epilogue (north-star item 4; ops.cuh FEpi): an aggregation
whose F result feeds BatchNorm [ReLU] [Binarize] applies them in its own
stores and, with the Binarize, writes only the packed sign bits; any other F
producer gets BatchNorm [ReLU] [Binarize] as one pass.  Checked against the
UNMODIFIED reference engine (bitgnn::run_model through oracle/_ref,
graphops.cpp:337-355 for BatchNorm) on every aggregation layout and kernel
that takes the epilogue -- row groups, slivers, tiles, column windows, hub rows,
the real-valued walks -- at 32- and 64-bit words: every BIN point bit for bit,
the output within the reference tolerance, the classes equal."""
import numpy as np
import pytest
import torch

import pyoracle as po
from helpers import bits_equal, rel_err

import paper_2305_02522_b200 as bg
from paper_2305_02522_b200 import _lib as L

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not po.ref_available(), reason="oracle/_ref (reference library) not built")]

S = bg.LayerSpec


def _w(rng, a, b):
    return rng.uniform(-1, 1, (a, b)).astype(np.float32)


def _bn(rng, c):
    # mean near the data so both signs survive; one sigma below the 1e-12 floor
    g = rng.uniform(0.5, 1.5, c).astype(np.float32)
    g[::7] *= -1
    s = rng.uniform(0.5, 2.0, c).astype(np.float32)
    s[3 % c] = 0.0
    return g, rng.uniform(-0.5, 0.5, c).astype(np.float32), rng.uniform(-2, 2, c).astype(np.float32), s


def _models(rng, f, h):
    return {
        # BBF aggregation -> BN -> ReLU -> Binarize (packed straight out of the counters)
        "agg_bbf_bn_relu_bin": [S(L.LAYER_FC, ["MM.FBB"], _w(rng, f, h)), S(L.LAYER_AGGREGATE, ["BSpMM.BBF"]),
                                S(L.LAYER_BATCHNORM, bn=_bn(rng, h)), S(L.LAYER_RELU), S(L.LAYER_BINARIZE),
                                S(L.LAYER_FC, ["MM.BBF"], _w(rng, h, 6)), S(L.LAYER_SOFTMAX)],
        # BBF aggregation -> BN -> Binarize (signs of both polarities)
        "agg_bbf_bn_bin": [S(L.LAYER_FC, ["MM.FBB"], _w(rng, f, h)), S(L.LAYER_AGGREGATE, ["BSpMM.BBF"]),
                           S(L.LAYER_BATCHNORM, bn=_bn(rng, h)), S(L.LAYER_BINARIZE),
                           S(L.LAYER_AGGREGATE, ["BSpMM.BBB"]), S(L.LAYER_FC, ["MM.BBF"], _w(rng, h, 5)),
                           S(L.LAYER_SOFTMAX)],
        # BBF aggregation -> BN -> ReLU, floats out
        "agg_bbf_bn_relu": [S(L.LAYER_FC, ["MM.FBB"], _w(rng, f, h)), S(L.LAYER_AGGREGATE, ["BSpMM.BBF"]),
                            S(L.LAYER_BATCHNORM, bn=_bn(rng, h)), S(L.LAYER_RELU),
                            S(L.LAYER_FC, ["MM.FBF"], _w(rng, h, 4)), S(L.LAYER_SOFTMAX)],
        # real-valued walks: FFF and FBF aggregations -> BN -> Binarize / ReLU
        "agg_fff_bn_bin": [S(L.LAYER_AGGREGATE, ["BSpMM.FFF"]), S(L.LAYER_BATCHNORM, bn=_bn(rng, f)),
                           S(L.LAYER_BINARIZE), S(L.LAYER_FC, ["MM.BBF"], _w(rng, f, 7)), S(L.LAYER_SOFTMAX)],
        "gcn_fbf_bn_relu": [S(L.LAYER_GCN, ["MM.FBF", "BSpMM.FBF"], _w(rng, f, h)),
                            S(L.LAYER_BATCHNORM, bn=_bn(rng, h)), S(L.LAYER_RELU),
                            S(L.LAYER_FC, ["MM.FBF"], _w(rng, h, 3)), S(L.LAYER_SOFTMAX)],
        # producers without their own epilogue: BN [ReLU] [Binarize] in one pass
        "fc_fbf_bn_relu_bin": [S(L.LAYER_FC, ["MM.FBF"], _w(rng, f, h)), S(L.LAYER_BATCHNORM, bn=_bn(rng, h)),
                               S(L.LAYER_RELU), S(L.LAYER_BINARIZE), S(L.LAYER_FC, ["MM.BBF"], _w(rng, h, 5)),
                               S(L.LAYER_SOFTMAX)],
        "bn_first_bin": [S(L.LAYER_BATCHNORM, bn=_bn(rng, f)), S(L.LAYER_BINARIZE),
                         S(L.LAYER_FC, ["MM.BBF"], _w(rng, f, 6)), S(L.LAYER_SOFTMAX)],
        "fc_fff_bn_last": [S(L.LAYER_FC, ["MM.FFF"], _w(rng, f, 9)), S(L.LAYER_BATCHNORM, bn=_bn(rng, 9))],
    }


NAMES = list(_models(np.random.default_rng(0), 8, 8))


def _check(layers, n, src, dst, x, wb):
    assert bg.validate_model(layers) == []
    m = bg.Model(layers, bg.prepare_graph(n, src, dst), word_bits=wb)
    xd = torch.from_numpy(x).cuda()
    out, logits, pts = m.forward_traced(xd)
    r_out, r_log, r_pts = po.ref_spec_run(layers, po.RefGraph(n, src, dst), x, wb)
    assert [p.label for p in pts] == [p.label for p in r_pts]
    for p, q in zip(pts, r_pts):
        assert bits_equal(p.bits.numpy(), q.bits), p.label
    got = out.cpu().numpy()
    assert rel_err(got, r_out) <= 1e-6
    if got.shape[1] > 1:
        assert np.array_equal(np.argmax(logits.cpu().numpy(), axis=1), np.argmax(r_log, axis=1))
    # the captured (CUDA-graph) forward equals the traced one
    a = m.forward(xd)
    b = m.forward(xd)
    assert torch.equal(a, out) and torch.equal(b, out)


@pytest.mark.parametrize("wb", [32, 64])
@pytest.mark.parametrize("name", NAMES)
def test_epilogue_models_match_reference_engine(name, wb):
    rng = np.random.default_rng(9100 + NAMES.index(name) + wb)
    n, e, f, h = 300, 2400, 37, 40
    layers = _models(rng, f, h)[name]
    src, dst = po.Rng(43).random_edges(n, e, False)
    _check(layers, n, src, dst, rng.uniform(-1, 1, (n, f)).astype(np.float32), wb)


LAYOUTS = {"auto": L.AGG_AUTO, "slivers": L.AGG_SLIVERS, "tiles": L.AGG_TILES, "window": L.AGG_WINDOW}


@pytest.mark.parametrize("layout", list(LAYOUTS))
@pytest.mark.parametrize("name", ["agg_bbf_bn_relu_bin", "agg_bbf_bn_bin", "agg_bbf_bn_relu", "agg_fff_bn_bin"])
def test_epilogue_on_every_aggregation_layout(layout, name):
    # hidden 128 at 32-bit words: 4 words per row, the column-window kernel's shape
    rng = np.random.default_rng(9200 + list(LAYOUTS).index(layout))
    n, e, f, h = 1500, 30000, 20, 128
    layers = _models(rng, f, h)[name]
    src, dst = po.Rng(44).random_edges(n, e, False)
    x = rng.uniform(-1, 1, (n, f)).astype(np.float32)
    bg.set_aggregation(LAYOUTS[layout])
    try:
        _check(layers, n, src, dst, x, 32)
    finally:
        bg.set_aggregation(L.AGG_AUTO)


@pytest.mark.parametrize("name", ["agg_bbf_bn_relu_bin", "agg_bbf_bn_relu", "agg_fff_bn_bin"])
def test_epilogue_with_hub_rows(name):
    # a star (node 0 of degree 2999 >= kHubDeg) plus a ring: hub_bb's final pass takes the epilogue
    n = 3000
    src = [0] * (n - 1) + list(range(1, n)) + list(range(n))
    dst = list(range(1, n)) + [0] * (n - 1) + [(i + 1) % n for i in range(n)]
    rng = np.random.default_rng(9300)
    layers = _models(rng, 16, 64)[name]
    _check(layers, n, src, dst, rng.uniform(-1, 1, (n, 16)).astype(np.float32), 32)


def _kernels(fn):
    """CUDA kernel names launched by fn (torch profiler); None without CUPTI."""
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    names = [e.name for e in prof.events() if e.device_type.name == "CUDA"]
    return names or None


@pytest.mark.parametrize("name,standalone", [("agg_bbf_bn_relu_bin", False), ("agg_fff_bn_bin", False),
                                             ("gcn_fbf_bn_relu", False), ("fc_fbf_bn_relu_bin", True)])
def test_epilogue_replaces_the_standalone_passes(name, standalone):
    """No separate BatchNorm / ReLU / binarize kernel runs after a fused
    aggregation; an MM producer gets exactly one BatchNorm pass (k_bn_act_*)."""
    rng = np.random.default_rng(9400)
    n, e, f, h = 300, 2400, 37, 40
    layers = _models(rng, f, h)[name]
    src, dst = po.Rng(45).random_edges(n, e, False)
    m = bg.Model(layers, bg.prepare_graph(n, src, dst))
    x = torch.from_numpy(rng.uniform(-1, 1, (n, f)).astype(np.float32)).cuda()
    m.forward_traced(x)  # builds the views
    names = _kernels(lambda: m.forward(x))  # the first plain forward runs eagerly (no binarize traces)
    if names is None:
        pytest.skip("profiler unavailable")
    assert not any("k_bn(" in k or "k_relu" in k or "k_binarize" in k for k in names), names
    assert sum("k_bn_act" in k for k in names) == (1 if standalone else 0), names
