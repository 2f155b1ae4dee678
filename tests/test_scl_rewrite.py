"""SCL elimination (ref: rewrite_eliminate_scl, graphops.cpp:357-368; tests
test_graphops.cpp:348-400, test_acceptance.cpp:370-420): a Scale node directly
ahead of a Binarize is dropped, any other Scale stays, and dropping it changes
nothing observable -- checked through the real reference engine."""
import numpy as np
import pytest

import pyoracle as po

import paper_2305_02522_b200 as bg
from paper_2305_02522_b200 import _lib as L


def _scale(rng, rows, cols):
    return bg.LayerSpec(L.LAYER_SCALE, scale_row=(0.25 + rng.uniform(size=rows)).astype(np.float32),
                        scale_col=(0.25 + rng.uniform(size=cols)).astype(np.float32))


def _w(rng, a, b):
    return rng.uniform(-1, 1, (a, b)).astype(np.float32)


def test_scale_ahead_of_binarize_is_dropped_and_others_kept():
    rng = np.random.default_rng(308)
    pruned = [bg.LayerSpec(L.LAYER_FC, ["MM.FBF"], _w(rng, 6, 8)), _scale(rng, 15, 8),
              bg.LayerSpec(L.LAYER_BINARIZE), bg.LayerSpec(L.LAYER_FC, ["MM.BBF"], _w(rng, 8, 4)),
              bg.LayerSpec(L.LAYER_SOFTMAX)]
    after = bg.rewrite_eliminate_scl(pruned)
    assert len(after) == 4 and after[1].kind == L.LAYER_BINARIZE
    assert [l.kind for l in after] == [pruned[i].kind for i in (0, 2, 3, 4)]
    kept = [bg.LayerSpec(L.LAYER_FC, ["MM.FBF"], _w(rng, 6, 8)), _scale(rng, 15, 8), bg.LayerSpec(L.LAYER_RELU),
            bg.LayerSpec(L.LAYER_BINARIZE), bg.LayerSpec(L.LAYER_FC, ["MM.BBF"], _w(rng, 8, 4)),
            bg.LayerSpec(L.LAYER_SOFTMAX)]
    assert len(bg.rewrite_eliminate_scl(kept)) == len(kept)
    # a trailing Scale (nothing after it) stays
    tail = kept[:2]
    assert len(bg.rewrite_eliminate_scl(tail)) == 2
    assert bg.rewrite_eliminate_scl([]) == []


@pytest.mark.skipif(not po.ref_available(), reason="oracle/_ref (reference library) not built")
def test_dropping_the_scale_changes_nothing_in_the_reference_engine():
    rng = np.random.default_rng(309)
    for it in range(25):
        f0, f1, f2 = rng.integers(2, 9), rng.integers(2, 9), rng.integers(2, 7)
        m = [bg.LayerSpec(L.LAYER_FC, ["MM.FBF"], _w(rng, f0, f1)), _scale(rng, 9, f1),
             bg.LayerSpec(L.LAYER_BINARIZE), bg.LayerSpec(L.LAYER_FC, ["MM.BBF"], _w(rng, f1, f2))]
        if it % 2:
            m += [_scale(rng, 9, f2), bg.LayerSpec(L.LAYER_BINARIZE), bg.LayerSpec(L.LAYER_FC, ["MM.BBF"], _w(rng, f2, f2))]
        m.append(bg.LayerSpec(L.LAYER_SOFTMAX))
        r = bg.rewrite_eliminate_scl(m)
        assert len(r) < len(m)
        x = rng.uniform(-1, 1, (9, f0)).astype(np.float32)
        oa, _, ta = po.ref_spec_run(m, None, x)
        ob, _, tb = po.ref_spec_run(r, None, x)
        assert len(ta) == len(tb)
        for p, q in zip(ta, tb):
            assert np.array_equal(p.bits, q.bits)
        assert np.array_equal(oa, ob)
