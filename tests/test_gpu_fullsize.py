"""Parity at the BASELINE.json shapes: the CUDA engine against the unmodified
reference engine (bitgnn::run_model, oracle/_ref, OpenMP on the host) on the
same generated inputs -- every binarization point bit for bit, the logits
exactly, the predicted classes identical.

Inputs: random_edges(Rng(100)) and build_model(seed 99) (rng.hpp,
modelconfig.cpp), checked equal between the two sides.  The reference graph
is assembled from the device-built FRDC arrays through the reference's
validating FrdcMatrix constructor (its own prepare_graph sorts 115 M edges on
one core: 44 s for Reddit); the FRDC build itself is pinned byte-for-byte
against the reference at every size its builder finishes in seconds
(test_gpu_parity / test_gpu_golden, and the Flickr case below)."""
import numpy as np
import pytest
import torch

import pyoracle as po
from helpers import bits_equal, rel_err

import paper_2305_02522_b200 as bg

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not po.ref_available(), reason="oracle/_ref (reference library) not built")]

# name: (model, nodes, edge draws, features, hidden, classes, plan) -- bench.py WORKLOADS
SHAPES = {
    "pubmed": ("gcn", 19_717, 88_648, 500, 64, 3,
               ["MM.FBB+BSpMM.BBB", "MM.BBB+BSpMM.BBB", "MM.BBF+BSpMM.FBF"]),
    "flickr": ("sage", 89_250, 899_756, 500, 256, 7, None),
    "reddit": ("gcn", 232_965, 114_615_892, 602, 128, 41, None),
    "products": ("saint", 2_449_029, 61_859_140, 100, 128, 47, None),
}


@pytest.mark.parametrize("wl", list(SHAPES))
def test_full_size_model_matches_reference_engine(wl):
    model, n, e, f, h, c, plan = SHAPES[wl]
    src, dst = bg.Rng(100).random_edges(n, e, False)
    r_src, r_dst = po.ref_random_edges(100, n, e, False)
    assert np.array_equal(src, r_src) and np.array_equal(dst, r_dst)
    layers, X = bg.build_model_spec(model, f, h, c, 99, n, plan)
    g = bg.prepare_graph(n, src, dst)
    m = bg.Model(layers, g)
    out, logits, pts = m.forward_traced(torch.from_numpy(X).cuda())
    torch.cuda.synchronize()

    a, r = g.structure.download(), g.raw.download()
    rg = po.RefGraph.from_frdc(n, po.Frdc(n, n, *a), po.Frdc(n, n, *r))
    rm = po.RefModel(rg, model, f, h, c, 99, n, 32, plan)
    assert np.array_equal(rm.features(), X)
    r_out, r_log, r_pts = rm.run(c)

    assert [p.label for p in pts] == [p.label for p in r_pts]
    for p, q in zip(pts, r_pts):
        assert (p.bits.rows, p.bits.cols) == (q.rows, q.cols), p.label
        assert bits_equal(p.bits.numpy(), q.bits), p.label
    lg = logits.cpu().numpy()
    assert np.array_equal(lg, r_log), rel_err(lg, r_log)
    assert np.array_equal(np.argmax(lg, axis=1), np.argmax(r_log, axis=1))
    assert np.allclose(out.cpu().numpy(), r_out, rtol=1e-6, atol=1e-7)


def test_flickr_frdc_equals_reference_prepare_graph():
    # the reference builds this one itself in seconds: both adjacency
    # structures (A + I and loop-free A) byte-identical
    model, n, e, *_ = SHAPES["flickr"]
    src, dst = bg.Rng(100).random_edges(n, e, False)
    g = bg.prepare_graph(n, src, dst)
    rg = po.RefGraph(n, src, dst)
    for which, mine in ((0, g.structure), (1, g.raw)):
        ref = rg.frdc(which)
        rp, ci, ti = mine.download()
        assert np.array_equal(rp, ref.row_ptr) and np.array_equal(ci, ref.col_ind) and np.array_equal(ti, ref.tiles)


@pytest.mark.parametrize("wl,world", [("reddit", 8), ("products", 8), ("reddit", 3)])
def test_full_size_sharded_ranges_equal_single_gpu(wl, world):
    # the 8-GPU configuration's per-rank work (every rank's row range through
    # the sharded engine in one process) is bit-identical to the 1-GPU forward
    from paper_2305_02522_b200.sharded import forward_virtual_ranks, partition_bounds
    model, n, e, f, h, c, plan = SHAPES[wl]
    src, dst = bg.Rng(100).random_edges(n, e, False)
    layers, X = bg.build_model_spec(model, f, h, c, 99, n, plan)
    g = bg.prepare_graph(n, src, dst)
    m = bg.Model(layers, g)
    x = torch.from_numpy(X).cuda()
    out1, log1, _ = m.forward_traced(x)
    rp, _, _ = g.structure.download()
    b = partition_bounds(rp, n, world)
    out, lg = forward_virtual_ranks(m, x, b, logits=True)
    torch.cuda.synchronize()
    assert torch.equal(lg, log1)
    assert torch.equal(out, out1)


@pytest.mark.parametrize("wl", ["pubmed", "flickr", "reddit"])
def test_full_size_64_bit_words_match_reference_engine(wl):
    # the same models packed in 64-bit words (big-endian u32 pairs,
    # bitdense.hpp:61-107) on both sides
    model, n, e, f, h, c, plan = SHAPES[wl]
    src, dst = bg.Rng(100).random_edges(n, e, False)
    layers, X = bg.build_model_spec(model, f, h, c, 99, n, plan)
    g = bg.prepare_graph(n, src, dst)
    m = bg.Model(layers, g, word_bits=64)
    out, logits, pts = m.forward_traced(torch.from_numpy(X).cuda())
    torch.cuda.synchronize()
    a, r = g.structure.download(), g.raw.download()
    rg = po.RefGraph.from_frdc(n, po.Frdc(n, n, *a), po.Frdc(n, n, *r))
    rm = po.RefModel(rg, model, f, h, c, 99, n, 64, plan)
    r_out, r_log, r_pts = rm.run(c)
    assert [p.label for p in pts] == [p.label for p in r_pts]
    for p, q in zip(pts, r_pts):
        assert p.bits.word_bits == 64 and bits_equal(p.bits.numpy(), q.bits), p.label
    assert np.array_equal(logits.cpu().numpy(), r_log)


def _sha(a):
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("wl", ["reddit", "products"])
def test_full_size_frdc_equals_reference_prepare_graph_digests(wl):
    # The device FRDC build at the full BASELINE shapes against the REAL
    # reference's own prepare_graph (frdc_from_edges x2 + scales,
    # graphops.cpp:146-170), recorded once in the dev container by
    # tests/golden/make_fullsize_frdc.py: every array byte-identical.
    import json
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", "fullsize_frdc.json")) as fh:
        want = json.load(fh)["shapes"][wl]
    model, n, e, *_ = SHAPES[wl]
    src, dst = bg.Rng(100).random_edges(n, e, False)
    assert (_sha(src), _sha(dst)) == (want["sha_src"], want["sha_dst"])
    g = bg.prepare_graph(n, src, dst)
    for key, mine in (("loops", g.structure), ("raw", g.raw)):
        rp, ci, ti = mine.download()
        w = want[key]
        assert ti.shape[0] == w["nnz_tiles"] and mine.nnz_bits == w["nnz_bits"], key
        assert _sha(rp) == w["sha_row_ptr"], key
        assert _sha(ci) == w["sha_col_ind"], key
        assert _sha(ti) == w["sha_tiles"], key
    assert _sha(g.norm_row.cpu().numpy()) == want["sha_norm"]
    assert _sha(g.mean_row.cpu().numpy()) == want["sha_mean_row"]
    assert _sha(g.neighbor_count.cpu().numpy()) == want["sha_neighbor_count"]
