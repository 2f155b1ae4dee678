"""Degenerate inputs through the whole engine, against the oracle: graphs
without edges, a single node, self loops only, rows not a multiple of the
4-row tile, tiny inputs through the streamed host entry point, and more
shards than tile rows (empty ranks)."""
import numpy as np
import pytest
import torch

import pyoracle as po
from helpers import bits_equal, to_layer_specs

import paper_2305_02522_b200 as bg
from paper_2305_02522_b200.sharded import forward_virtual_ranks, partition_bounds

pytestmark = pytest.mark.gpu


def _run(model, n, src, dst, f=37, h=40, c=5):
    layers, X = po.build_model(model, f, h, c, 99, n)
    src = np.asarray(src, np.int64)
    dst = np.asarray(dst, np.int64)
    m = bg.Model(to_layer_specs(bg, layers), bg.prepare_graph(n, src, dst))
    out, logits, pts = m.forward_traced(torch.from_numpy(X).cuda())
    o_out, o_log, o_pts = po.run_model(layers, po.Graph(n, src, dst), X)
    assert [p.label for p in pts] == [p.label for p in o_pts]
    for p, q in zip(pts, o_pts):
        assert bits_equal(p.bits.numpy(), q.bits), p.label
    assert np.array_equal(logits.cpu().numpy(), o_log)
    assert np.allclose(out.cpu().numpy(), o_out, rtol=1e-6, atol=1e-7)
    out2 = m.forward(torch.from_numpy(X).cuda())
    torch.cuda.synchronize()
    assert torch.equal(out2, out)
    return m, X, out


@pytest.mark.parametrize("model", ["gcn", "sage", "saint"])
@pytest.mark.parametrize("n", [1, 3, 4, 5, 9, 130])
def test_graph_without_edges(model, n):
    _run(model, n, [], [])


@pytest.mark.parametrize("model", ["gcn", "sage", "saint"])
def test_self_loops_only_and_duplicates(model):
    n = 11
    src = list(range(n)) + [2, 2, 2]
    dst = list(range(n)) + [3, 3, 3]
    _run(model, n, src, dst)


@pytest.mark.parametrize("model", ["gcn", "sage"])
def test_star_graph_hub(model):
    n = 1001
    src = [0] * (n - 1) + list(range(1, n))
    dst = list(range(1, n)) + [0] * (n - 1)
    _run(model, n, src, dst)


@pytest.mark.parametrize("rows", [1, 7, 17, 4097])
def test_host_entry_point_on_small_inputs(rows):
    s, d = po.Rng(5).random_edges(rows, 4 * rows, False)
    m, X, out = _run("gcn", rows, s, d)
    got = m.forward_host(X)
    assert torch.equal(got, out.cpu())


def test_more_shards_than_tile_rows():
    n = 10  # 3 tile rows
    s, d = po.Rng(6).random_edges(n, 30, False)
    layers, X = po.build_model("gcn", 37, 40, 5, 99, n)
    g = bg.prepare_graph(n, s, d)
    m = bg.Model(to_layer_specs(bg, layers), g)
    x = torch.from_numpy(X).cuda()
    ref, _, _ = m.forward_traced(x)
    rp, _, _ = g.structure.download()
    for world in (2, 3, 5, 8):
        b = partition_bounds(rp, n, world)
        assert b[0] == 0 and b[-1] == n and all(b[i] <= b[i + 1] for i in range(world))
        out = forward_virtual_ranks(m, x, b)
        torch.cuda.synchronize()
        assert torch.equal(out, ref), world


def test_zero_row_operands():
    w = bg.BitOperand(bg.binarize(torch.rand(37, 20, device="cuda") - 0.5))
    x = torch.zeros((0, 37), dtype=torch.float32, device="cuda")
    out = bg.bmm("BMM.FBB", x, w)
    assert out.bits.rows == 0
    outf = bg.bmm("BMM.FBF", x, w)
    assert tuple(outf.shape) == (0, 20)
    assert tuple(bg.softmax_rows(torch.zeros((0, 5), device="cuda")).shape) == (0, 5)
