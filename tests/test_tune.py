"""Variant substitution (ref: tune.hpp / tune.cpp).  The enumeration is host
logic (CPU): it must produce exactly the reference's plans in the
reference's order.  The GPU test tunes over a subset of plans with a
verification callback backed by the oracle (test infrastructure)."""
import numpy as np
import pytest
import torch

import pyoracle as po
from helpers import rel_err

from paper_2305_02522_b200 import _lib as L
from paper_2305_02522_b200 import tune as T


def test_legal_variants_match_the_reference_counts():
    # kernels.hpp:19-22 valid(): 7 BMM, 8 BSpMM, 3 ADD variants
    assert [v.name() for v in T.legal_variants(L.BMM)] == [
        "BMM.FFB", "BMM.FBF", "BMM.FBB", "BMM.BFF", "BMM.BFB", "BMM.BBF", "BMM.BBB"]
    assert len(T.legal_variants(L.BSPMM)) == 8
    assert [v.name() for v in T.legal_variants(L.ADD)] == ["ADD.FFF", "ADD.BBF", "ADD.BBB"]
    assert [v.name() for v in T.legal_variants(L.BMM, L.B, None, L.F)] == ["BMM.BFF", "BMM.BBF"]


@pytest.mark.skipif(not po.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("model,layers", [("gcn", 1), ("gcn", 2), ("gcn", 3), ("sage", 2), ("saint", 2), ("saint", 3)])
def test_enumeration_equals_the_reference(model, layers):
    assert T.enumerate_plans(T.skeleton(model, layers)) == po.ref_enumerate_plans(model, layers)


@pytest.mark.gpu
def test_tune_picks_the_fastest_verified_plan():
    n, e, f, h, c = 2708, 13264, 1433, 64, 7
    s, d = po.Rng(100).random_edges(n, e, False)
    plans = T.enumerate_plans(T.skeleton("gcn", 2))
    chosen = [["MM.FBB+BSpMM.BBB", "MM.BBF+BSpMM.FBF"]] + plans[:5] + plans[-3:]

    def verify(plan, logits):
        layers, X = po.build_model("gcn", f, h, c, 99, n, plan)
        _, o_log, _ = po.run_model(layers, po.Graph(n, s, d), X)
        err = rel_err(logits.cpu().numpy(), o_log)
        return err <= 1e-5, err

    r = T.tune_model("gcn", n, s, d, f, h, c, plans=chosen, reps=3, verify=verify)
    assert r.candidates == len(chosen)
    assert all(cand.verified for cand in r.evaluated)
    assert r.best.median_ms == min(cand.median_ms for cand in r.evaluated)
    assert r.best.median_ms > 0


@pytest.mark.gpu
def test_tune_without_a_passing_candidate_raises():
    n, e = 200, 900
    s, d = po.Rng(7).random_edges(n, e, False)
    with pytest.raises(Exception, match="no candidate passed verification"):
        T.tune_model("gcn", n, s, d, 40, 16, 3, plans=[["MM.FBB+BSpMM.BBB", "MM.BBF+BSpMM.FBF"]], reps=1,
                     verify=lambda plan, logits: (False, 1.0))
