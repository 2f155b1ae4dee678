"""GPU: the CUDA path reproduces the REAL reference's outputs, hash for hash
(tests/golden/reference_fixtures.json, generated from /root/reference by
tests/golden/make_golden.py).  Inputs come from the product's own
generators, which test_capi_cpu.py pins to the reference's."""
import hashlib
import json
import os

import numpy as np
import pytest
import torch

import paper_2305_02522_b200 as bg

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "reference_fixtures.json")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _cases():
    with open(GOLDEN) as fh:
        return json.load(fh)["cases"]


@pytest.mark.parametrize("case", _cases(), ids=lambda c: c["name"])
def test_cuda_path_reproduces_reference(case):
    n = case["nodes"]
    s, d = bg.Rng(case["graph_seed"]).random_edges(n, case["edge_draws"], False)
    layers, X = bg.build_model_spec(case["model"], case["features"], case["hidden"], case["classes"],
                                    case["model_seed"], n, case["plan"])
    assert sha(X) == case["sha_x"]
    g = bg.prepare_graph(n, s, d)
    for fr, key in ((g.structure, "frdc_loops"), (g.raw, "frdc_raw")):
        rp, ci, ti = fr.download()
        assert sha(rp) == case[key]["sha_row_ptr"]
        assert sha(ci) == case[key]["sha_col_ind"]
        assert sha(ti) == case[key]["sha_tiles"]
    assert sha(g.norm_row.cpu().numpy()) == case["sha_norm"]
    assert sha(g.mean_row.cpu().numpy()) == case["sha_mean_row"]
    assert sha(g.neighbor_count.cpu().numpy()) == case["sha_neighbor_count"]
    m = bg.Model(layers, g, word_bits=case["word_bits"])
    out, logits, pts = m.forward_traced(torch.from_numpy(X).cuda())
    assert [p.label for p in pts] == [t["label"] for t in case["trace"]]
    for p, t in zip(pts, case["trace"]):
        assert (p.bits.rows, p.bits.cols, p.bits.word_bits) == (t["rows"], t["cols"], t["word_bits"])
        assert sha(p.bits.numpy()) == t["sha"], p.label
    lg = logits.cpu().numpy()
    assert sha(lg) == case["sha_logits"], np.abs(lg[0] - np.array(case["logits_row0"], np.float32)).max()
    # softmax itself uses the device's double exp: within 1e-6 of the reference
    ref_out = torch.softmax(torch.from_numpy(lg.astype(np.float64)), dim=1).numpy()
    assert np.allclose(out.cpu().numpy(), ref_out, rtol=1e-6, atol=1e-9)
