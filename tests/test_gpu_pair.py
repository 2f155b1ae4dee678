"""Paired F->B products (bmm_pair): a SAGE / GraphConv layer's two MM.FBB on
the same fp32 input run as one product that reads the input once.  The
untraced forward (paired) must equal the traced forward (one product per
slot, every BIN point checked against the oracle elsewhere) bit for bit, on
every kernel that takes pairs (warp per row, TMA-fed mma.sync) and on shapes
that do not pair on the TMA kernel (falls back to single products)."""
import numpy as np
import pytest
import torch

import pyoracle as po
from helpers import to_layer_specs

import paper_2305_02522_b200 as bg

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["default", "scalar", "tma", "tc", "bulk"])
def fbb_kernel(monkeypatch, request):
    if request.param != "default":
        monkeypatch.setenv("BG_FBB", request.param)
    return request.param


@pytest.mark.parametrize("wb", [32, 64])
@pytest.mark.parametrize("model,n,e,f,h,c", [("sage", 3000, 40000, 100, 128, 7), ("saint", 2500, 30000, 90, 40, 5),
                                             ("sage", 1000, 9000, 37, 100, 6), ("saint", 777, 5000, 64, 256, 9)])
def test_paired_forward_equals_per_slot_forward(fbb_kernel, wb, model, n, e, f, h, c):
    s, d = po.Rng(300 + n).random_edges(n, e, False)
    layers, X = po.build_model(model, f, h, c, 99, n)
    m = bg.Model(to_layer_specs(bg, layers), bg.prepare_graph(n, s, d), word_bits=wb)
    x = torch.from_numpy(X).cuda()
    out_t, _, _ = m.forward_traced(x)
    m.set_graph_capture(False)
    out_p = m.forward(x)
    torch.cuda.synchronize()
    assert torch.equal(out_p, out_t)
    o_out, _, _ = po.run_model(layers, po.Graph(n, s, d), X, wb)
    assert np.allclose(out_p.cpu().numpy(), o_out, rtol=1e-6, atol=1e-7)


def test_paired_forward_on_the_tma_kernel_at_scale():
    # above the warp-per-row threshold: the default dispatch takes the TMA pair
    n, e, f, h, c = 140000, 1400000, 100, 128, 47
    s, d = po.Rng(31).random_edges(n, e, False)
    layers, X = po.build_model("saint", f, h, c, 99, n)
    m = bg.Model(to_layer_specs(bg, layers), bg.prepare_graph(n, s, d))
    x = torch.from_numpy(X).cuda()
    out_t, _, _ = m.forward_traced(x)
    _, t = m.forward_timed(x)
    assert any("mm_pair[BMM.FBB]" in k.label for k in t)
    out_p = m.forward(x)
    torch.cuda.synchronize()
    assert torch.equal(out_p, out_t)


def test_paired_host_entry_point_streams_chunks():
    n, e, f, h, c = 50000, 500000, 100, 128, 47
    s, d = po.Rng(32).random_edges(n, e, False)
    layers, X = po.build_model("sage", f, h, c, 99, n)
    m = bg.Model(to_layer_specs(bg, layers), bg.prepare_graph(n, s, d))
    want, _, _ = m.forward_traced(torch.from_numpy(X).cuda())
    got = m.forward_host(X)
    assert torch.equal(got, want.cpu())
