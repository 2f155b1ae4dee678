"""GPU: the row-sharded forward on one B200 in "virtual
ranks" mode -- every rank's row range runs through the same per-range
kernels -- is bit-identical to the single-GPU forward and to the oracle for
1/2/3/4/8 shards (the row partition never changes an accumulation order)."""
import numpy as np
import pytest
import torch

import pyoracle as po
from helpers import to_layer_specs

import paper_2305_02522_b200 as bg
from paper_2305_02522_b200 import sharded
from paper_2305_02522_b200.sharded import forward_virtual_ranks, partition_bounds

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("model,n,e,f,h,c,plan", [
    ("gcn", 2708, 13264, 1433, 64, 7, None),
    ("sage", 2708, 10556, 1433, 64, 7, None),
    ("saint", 2708, 10556, 1433, 64, 7, None),
    ("gcn", 19717, 88648, 500, 64, 3, ["MM.FBB+BSpMM.BBB", "MM.BBB+BSpMM.BBB", "MM.BBF+BSpMM.FBF"]),
    ("gcn", 1003, 9000, 70, 40, 5, ["MM.FBF+BSpMM.FFF", "MM.FBB+BSpMM.BBB", "MM.BBF+BSpMM.FBF"]),
])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_sharded_matches_single_gpu(model, n, e, f, h, c, plan, world):
    s, d = po.Rng(100).random_edges(n, e, False)
    layers, X = po.build_model(model, f, h, c, 99, n, plan)
    g = bg.prepare_graph(n, s, d)
    m = bg.Model(to_layer_specs(bg, layers), g)
    x = torch.from_numpy(X).cuda()
    ref_out, ref_log, _ = m.forward_traced(x)
    rp, _, _ = g.structure.download()
    bounds = partition_bounds(rp, n, world)
    assert bounds[0] == 0 and bounds[-1] == n and all(b % 4 == 0 for b in bounds[:-1])
    out, lg = forward_virtual_ranks(m, x, bounds, logits=True)
    torch.cuda.synchronize()
    assert torch.equal(lg, ref_log)
    assert torch.equal(out, ref_out)
    o_out, o_log, _ = po.run_model(layers, po.Graph(n, s, d), X)
    assert np.array_equal(lg.cpu().numpy(), o_log)


def test_partition_is_balanced_by_tiles():
    s, d = po.Rng(3).random_edges(20000, 400000, False)
    g = bg.prepare_graph(20000, s, d)
    rp, _, _ = g.structure.download()
    b = partition_bounds(rp, 20000, 8)
    tiles = [int(rp[b[k + 1] // 4] if b[k + 1] < 20000 else rp[-1]) - int(rp[b[k] // 4]) for k in range(8)]
    assert max(tiles) - min(tiles) <= 0.02 * sum(tiles) / 8 + 64
    assert [g.partition_rows(8, k) for k in range(8)] == [(b[k], b[k + 1]) for k in range(8)]


@pytest.mark.parametrize("world", [1, 3, 8])
def test_sharded_dense_graph_through_windowed_aggregation(world):
    # a dense graph forced onto the column-windowed BBB kernel: each rank's
    # row range gets its own row-block sizing; still bit-identical
    from paper_2305_02522_b200 import _lib as L
    n, e, f, h, c = 6000, 900000, 300, 128, 41
    s, d = po.Rng(100).random_edges(n, e, False)
    layers, X = po.build_model("gcn", f, h, c, 99, n)
    g = bg.prepare_graph(n, s, d)
    m = bg.Model(to_layer_specs(bg, layers), g)
    x = torch.from_numpy(X).cuda()
    bg.set_aggregation(L.AGG_WINDOW, 500)
    try:
        ref_out, ref_log, _ = m.forward_traced(x)
        rp, _, _ = g.structure.download()
        out, lg = forward_virtual_ranks(m, x, partition_bounds(rp, n, world), logits=True)
        torch.cuda.synchronize()
    finally:
        bg.set_aggregation(L.AGG_AUTO, 0)
    assert torch.equal(lg, ref_log)
    assert torch.equal(out, ref_out)
    o_out, o_log, _ = po.run_model(layers, po.Graph(n, s, d), X)
    assert np.array_equal(lg.cpu().numpy(), o_log)


def test_sharded_model_host_entry_point_single_rank():
    # bench.py's e2e path under torchrun: this rank's pinned host rows in,
    # its output rows out; with one rank it is the whole forward
    n, e, f, h, c = 3000, 60000, 300, 128, 41
    s, d = po.Rng(100).random_edges(n, e, False)
    layers, X = po.build_model("gcn", f, h, c, 99, n)
    g = bg.prepare_graph(n, s, d)
    specs = to_layer_specs(bg, layers)
    want = bg.Model(specs, g).forward(torch.from_numpy(X).cuda()).cpu()
    sm = sharded.ShardedModel(specs, g, None, 1, 0)
    got = sm.forward_host(torch.from_numpy(X).pin_memory())
    torch.cuda.synchronize()
    assert torch.equal(got, want)


def test_sharded_timed_forward_single_rank_labels_and_output():
    # bench.py's per-op table under torchrun: same labels as the 1-GPU forward
    n, e, f, h, c = 3000, 60000, 300, 128, 41
    s, d = po.Rng(100).random_edges(n, e, False)
    layers, X = po.build_model("gcn", f, h, c, 99, n)
    g = bg.prepare_graph(n, s, d)
    specs = to_layer_specs(bg, layers)
    m = bg.Model(specs, g)
    x = torch.from_numpy(X).cuda()
    want, t1 = m.forward_timed(x)
    sm = sharded.ShardedModel(specs, g, None, 1, 0)
    got, t2 = sm.forward_timed(x)
    assert torch.equal(got, want)
    assert [k.label for k in t2] == [k.label for k in t1]
    assert all(k.ms >= 0 for k in t2) and t2[0].ms > 0
