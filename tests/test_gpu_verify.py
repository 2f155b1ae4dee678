"""verify_model on the device (ref: verify_model / VerifyReport,
runreport.cpp:51-135) against the reference's OWN verify_model report on the
same model: the engine is ours, the reference side is the reference's dense
oracle (oracle.cpp:194-317, via oracle/_ref), and every report field must
equal the reference's -- including with the corrupt_tile fault hook
(runreport.cpp:55-63, test_cli.cpp:205-224: verify must fail) and in the
full-precision mode (test_cli.cpp:226-238)."""
import numpy as np
import pytest
import torch

import pyoracle as po

import paper_2305_02522_b200 as bg

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not po.ref_available(), reason="oracle/_ref (reference library) not built")]

CASES = [  # model, nodes, edge draws, features, hidden, classes, plan
    ("gcn", 2708, 10556, 1433, 64, 7, None),
    ("gcn", 2708, 13264, 1433, 16, 7, None),
    ("sage", 900, 5000, 60, 32, 5, None),
    ("saint", 700, 4000, 45, 32, 6, None),
    ("gcn", 500, 3000, 40, 24, 6, ["MM.FBF+BSpMM.FFF", "MM.FBF+BSpMM.FFF"]),
]


def _setup(model, n, e, f, h, c, plan, gseed=100):
    src, dst = po.ref_random_edges(gseed, n, e, False)
    rg = po.RefGraph(n, src, dst)
    rm = po.RefModel(rg, model, f, h, c, 99, n, 32, plan)
    layers, X = bg.build_model_spec(model, f, h, c, 99, n, plan)
    assert np.array_equal(X, rm.features())
    return src, dst, rg, rm, layers, X


def _same(mine, ref):
    assert mine.bin_points == ref["bin_points"]
    assert mine.bin_values == ref["bin_values"]
    assert mine.bin_mismatches == ref["bin_mismatches"]
    assert mine.first_mismatch_label == ref["first_mismatch_label"]
    assert (mine.first_mismatch_row, mine.first_mismatch_col) == (ref["first_mismatch_row"],
                                                                  ref["first_mismatch_col"])
    assert mine.max_rel_logit_error == ref["max_rel_logit_error"]
    assert mine.argmax_agreement == ref["argmax_agreement"]
    assert mine.passed == ref["pass"]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_report_equals_the_references_verify_model(case):
    model, n, e, f, h, c, plan = CASES[case]
    src, dst, rg, rm, layers, X = _setup(model, n, e, f, h, c, plan)
    pts, olog = po.ref_oracle_run(rg, rm)
    m = bg.Model(layers, bg.prepare_graph(n, src, dst))
    rep = bg.verify_model(m, torch.from_numpy(X).cuda(), pts, olog)
    _same(rep, po.ref_verify_model(rg, rm))
    assert rep.passed


@pytest.mark.parametrize("k", [0, 17, 123456])
def test_corrupted_tile_fails_verify_like_the_reference(k):
    # ref: runreport.cpp:55-63 -- the engine's copy of A+I has bit 0 of tile
    # k % nnz flipped; test_cli.cpp:205-224 expects pass == false
    model, n, e, f, h, c, plan = CASES[0]
    src, dst, rg, rm, layers, X = _setup(model, n, e, f, h, c, plan)
    pts, olog = po.ref_oracle_run(rg, rm)
    g = bg.prepare_graph(n, src, dst)
    g.corrupt_tile(k)
    m = bg.Model(layers, g)
    rep = bg.verify_model(m, torch.from_numpy(X).cuda(), pts, olog)
    assert not rep.passed
    assert rep.bin_mismatches > 0 and rep.first_mismatch_label and rep.first_mismatch_row >= 0
    _same(rep, po.ref_verify_model(rg, rm, corrupt_tile=k))
    assert rep.to_dict()["pass"] is False and "first_mismatch" in rep.to_dict()


def test_full_precision_mode_compares_no_bin_points():
    # ref: test_cli.cpp:226-238 -- all-F plan against the dense reference
    plan = ["MM.FFF+BSpMM.FFF", "MM.FFF+BSpMM.FFF"]
    src, dst, rg, rm, layers, X = _setup("gcn", 400, 2500, 10, 6, 3, plan, gseed=13)
    pts, olog = po.ref_oracle_run(rg, rm, full_precision=True)
    m = bg.Model(layers, bg.prepare_graph(400, src, dst))
    rep = bg.verify_model(m, torch.from_numpy(X).cuda(), pts, olog, compare_bits=False)
    assert rep.bin_points == 0 and rep.bin_values == 0
    _same(rep, po.ref_verify_model(rg, rm, full_precision=True))
    assert rep.passed


def test_misaligned_traces_are_logic_errors():
    model, n, e, f, h, c, plan = CASES[1]
    src, dst, rg, rm, layers, X = _setup(model, n, e, f, h, c, plan)
    pts, olog = po.ref_oracle_run(rg, rm)
    m = bg.Model(layers, bg.prepare_graph(n, src, dst))
    x = torch.from_numpy(X).cuda()
    with pytest.raises(bg.LogicError, match="disagree on trace shape"):
        bg.verify_model(m, x, pts[:-1], olog)
    bad = list(pts)
    bad[1] = po.TracePoint("nope", bad[1].bits, bad[1].rows, bad[1].cols, bad[1].word_bits)
    with pytest.raises(bg.LogicError, match=r"trace point 1 misaligned \(layer0.mm.bin_w vs nope\)"):
        bg.verify_model(m, x, bad, olog)
    with pytest.raises(bg.LogicError, match="logit shapes disagree"):
        bg.verify_model(m, x, pts, olog[:, :-1])
