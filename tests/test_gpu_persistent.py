"""The whole-forward persistent kernel for small graphs (persistent.cu; the
paper's cooperative cross-layer fusion): one launch
for the binary GCN chain, bit-identical to the layer-by-layer forward and to
the reference engine (oracle/_ref)."""
import numpy as np
import pytest
import torch

import pyoracle as po

import paper_2305_02522_b200 as bg

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _persistent_on():
    bg.bitgnn.set_persistent(True)
    yield
    bg.bitgnn.set_persistent(False)

CASES = [  # model, nodes, edge draws, features, hidden, classes, plan, word_bits
    ("gcn", 2708, 10556, 1433, 64, 7, None, 32),                       # Cora (BASELINE configs[0])
    ("gcn", 2708, 13264, 1433, 16, 7, None, 32),                       # the reference's acceptance model
    ("gcn", 19717, 88648, 500, 64, 3,
     ["MM.FBB+BSpMM.BBB", "MM.BBB+BSpMM.BBB", "MM.BBF+BSpMM.FBF"], 32),  # PubMed 3-layer (configs[1])
    ("gcn", 3001, 20000, 333, 128, 32, None, 64),                      # 64-bit words, widest shapes
    ("gcn", 5003, 40000, 77, 96, 13,
     ["MM.FBB+BSpMM.BBB", "MM.BBB+BSpMM.BBB", "MM.BBB+BSpMM.BBB", "MM.BBF+BSpMM.FBF"], 32),
]


def _launches(fn):
    """Kernels launched by fn (torch profiler, CUDA activity)."""
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    names = [e.name for e in prof.events() if e.device_type.name == "CUDA"]
    if not names:  # no CUPTI (e.g. under compute-sanitizer): nothing to check
        return ["(profiler unavailable)"]
    return [n for n in names if "persistent" in n]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_persistent_forward_equals_layer_by_layer(case):
    model, n, e, f, h, c, plan, wb = CASES[case]
    src, dst = bg.Rng(100).random_edges(n, e, False)
    layers, X = bg.build_model_spec(model, f, h, c, 99, n, plan)
    g = bg.prepare_graph(n, src, dst)
    m = bg.Model(layers, g, word_bits=wb)
    x = torch.from_numpy(X).cuda()
    want_out, want_log, _ = m.forward_traced(x)  # layer by layer (traced forwards never take the fused kernel)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        out = torch.empty_like(want_out)
        lg = torch.empty_like(want_log)
        for _ in range(3):  # eager, captured, replayed
            out.zero_()
            lg.zero_()
            m.forward(x, out, lg)
            s.synchronize()
            assert torch.equal(lg, want_log)
            assert torch.equal(out, want_out)
        assert _launches(lambda: m.forward(x, out, lg)), "the persistent kernel did not run"


def test_persistent_forward_matches_reference_engine():
    model, n, e, f, h, c, plan, wb = CASES[0]
    src, dst = bg.Rng(100).random_edges(n, e, False)
    layers, X = bg.build_model_spec(model, f, h, c, 99, n, plan)
    m = bg.Model(layers, bg.prepare_graph(n, src, dst))
    x = torch.from_numpy(X).cuda()
    out = m.forward(x)
    lg = torch.empty_like(out)
    m.forward(x, out, lg)
    torch.cuda.synchronize()
    if not po.ref_available():
        pytest.skip("oracle/_ref not built")
    rm = po.RefModel(po.RefGraph(n, *po.ref_random_edges(100, n, e, False)), model, f, h, c, 99, n, 32, plan)
    r_out, r_log, _ = rm.run(c, trace=False)
    assert np.array_equal(lg.cpu().numpy(), r_log)
    assert np.allclose(out.cpu().numpy(), r_out, rtol=1e-6, atol=1e-7)


def test_binary_input_model_takes_the_persistent_path():
    n, e, f, h, c = 4000, 30000, 96, 64, 5
    src, dst = bg.Rng(7).random_edges(n, e, False)
    plan = ["MM.BBB+BSpMM.BBB", "MM.BBF+BSpMM.FBF"]
    layers, X = bg.build_model_spec("gcn", f, h, c, 9, n, plan)
    g = bg.prepare_graph(n, src, dst)
    xb = bg.BitOperand(bg.binarize(torch.from_numpy(X).cuda()))
    m = bg.Model(layers, g, input_precision=bg.B)
    want_out, want_log, _ = m.forward_traced(xb)
    lg = torch.empty_like(want_log)
    out = m.forward(xb, logits=lg)
    torch.cuda.synchronize()
    assert torch.equal(out, want_out) and torch.equal(lg, want_log)
