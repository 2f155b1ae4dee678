"""CUDA path vs the oracle (C restatement of the reference) on the same seeded
inputs.  Integer/bit outputs bit-exact; F outputs bit-exact too (the device
kernels accumulate in the reference's order), logits at the north-star
tolerance 1e-5 relative where stated."""
import numpy as np
import pytest
import torch

import pyoracle as po
from helpers import bits_equal, to_layer_specs, rel_err, argmax_agreement

import paper_2305_02522_b200 as bg

pytestmark = pytest.mark.gpu


def cuda(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()


# ---------------------------------------------------------------- bitdense ---
@pytest.mark.parametrize("wb", [32, 64])
@pytest.mark.parametrize("shape", [(1, 1), (3, 31), (5, 32), (7, 33), (64, 602), (17, 1433), (0, 5), (4, 0)])
def test_binarize_matches_oracle(shape, wb):
    rng = po.Rng(11 + shape[0] + shape[1])
    x = rng.random_dense(*shape)
    if x.size:
        x.flat[::7] = 0.0
        x.flat[1::11] = -0.0
    got = bg.binarize(cuda(x), wb).numpy()
    assert bits_equal(got, po.binarize(x, wb))


def test_binarize_known_answer_and_nan():
    # ref: test_bitdense.cpp:54-68  [0.5,-2,-0.1,0] -> 0x90000000
    got = bg.binarize(cuda([[0.5, -2.0, -0.1, 0.0]])).numpy()
    assert got[0, 0] == 0x90000000
    x = np.array([[np.nan, -0.0, np.inf, -np.inf]], np.float32)
    assert bits_equal(bg.binarize(cuda(x)).numpy(), po.binarize(x))


@pytest.mark.parametrize("axis", [0, 1])
def test_binarize_with_scale_matches_oracle(axis):
    x = po.Rng(3).random_dense(37, 45)
    x[:, 5] = 0.0
    bits, sc = bg.binarize_with_scale(cuda(x), axis)
    assert bits_equal(bits.numpy(), po.binarize(x))
    assert np.array_equal(sc.cpu().numpy(), po.l1_scales(x, axis))


@pytest.mark.parametrize("wb", [32, 64])
def test_transpose_and_unpack(wb):
    x = po.Rng(5).random_dense(70, 45)
    b = bg.binarize(cuda(x), wb)
    t = bg.transpose(b)
    assert bits_equal(t.numpy(), po.transpose_bits(po.binarize(x, wb), 70, 45, wb))
    assert torch.equal(bg.unpack(b).cpu(), torch.from_numpy(np.where(x >= 0, 1.0, -1.0).astype(np.float32)))


# -------------------------------------------------------------------- FRDC ---
def frdc_equal(dev, ora):
    rp, ci, ti = dev.download()
    return (np.array_equal(rp, ora.row_ptr) and np.array_equal(ci, ora.col_ind)
            and np.array_equal(ti, ora.tiles))


@pytest.mark.parametrize("loops", [False, True])
@pytest.mark.parametrize("n,m,allow_self", [(1, 0, False), (5, 9, True), (37, 150, True), (200, 4000, True),
                                            (1001, 20000, False), (2708, 13264, False)])
def test_frdc_from_edges_byte_identical(n, m, allow_self, loops):
    s, d = po.Rng(100 + n).random_edges(n, m, allow_self)
    dev = bg.frdc_from_edges(n, s, d, loops)
    ora = po.frdc_from_edges(n, s, d, loops)
    assert frdc_equal(dev, ora)
    assert dev.nnz_bits == ora.nnz_bits()
    assert np.array_equal(dev.degree().cpu().numpy(), ora.row_popcounts().astype(np.int32))


def test_frdc_known_tiles():
    # ref: test_bitsparse.cpp:31-54
    m = bg.frdc_from_edges(8, [1, 0], [2, 5], False)
    rp, ci, ti = m.download()
    assert list(rp) == [0, 2, 2] and list(ci) == [0, 1] and list(ti) == [0x0200, 0x4000]
    m = bg.frdc_from_edges(4, [0, 1, 1, 2, 2, 3], [1, 0, 2, 1, 3, 2], True)
    assert list(m.download()[2]) == [0xCE73]
    m = bg.frdc_from_edges(6, [0, 0, 0, 5, 2], [3, 3, 3, 5, 4], False)
    assert m.nnz_bits == 3
    m = bg.frdc_from_edges(10, [], [], False)
    assert m.nnz_tiles == 0 and list(m.download()[0]) == [0, 0, 0, 0]


def test_frdc_out_of_range_names_offender():
    with pytest.raises(bg.InvalidArgument) as e:
        bg.frdc_from_edges(4, [0, 2], [1, 9], False)
    assert "(2, 9)" in str(e.value) and "4 nodes" in str(e.value)


def test_frdc_from_host_validation():
    # ref: test_bitsparse.cpp:117-129
    with pytest.raises(bg.InvalidArgument):
        bg.FrdcMatrix.from_host(5, 5, [0, 1, 2], [0, 1], [0x8000, 0x0800])
    with pytest.raises(bg.InvalidArgument):
        bg.FrdcMatrix.from_host(4, 4, [0, 1], [0], [0])
    with pytest.raises(bg.InvalidArgument):
        bg.FrdcMatrix.from_host(8, 8, [0, 2, 1], [0, 1], [0x8000, 0x8000])
    with pytest.raises(bg.InvalidArgument):
        bg.FrdcMatrix.from_host(4, 8, [0, 2], [1, 1], [0x8000, 0x4000])
    with pytest.raises(bg.InvalidArgument):
        bg.FrdcMatrix.from_host(4, 8, [0, 1], [2], [0x8000])
    m = bg.FrdcMatrix.from_host(4, 8, [0, 1], [1], [0x8000])
    assert m.nnz_bits == 1


def test_prepare_graph_scales_exact():
    s, d = po.Rng(100).random_edges(2708, 13264, False)
    g = bg.prepare_graph(2708, s, d)
    o = po.Graph(2708, s, d)
    assert frdc_equal(g.structure, o.structure) and frdc_equal(g.raw, o.raw)
    assert np.array_equal(g.norm_row.cpu().numpy(), o.norm)
    assert np.array_equal(g.mean_row.cpu().numpy(), o.mean_row)
    assert np.array_equal(g.neighbor_count.cpu().numpy(), o.neighbor_count)


def test_normalized_two_node_graph():
    # ref: test_graphops.cpp:117-136
    g = bg.prepare_graph(2, [0, 1], [1, 0])
    assert list(g.structure.download()[2]) == [0xCC00]
    assert np.allclose(g.norm_row.cpu().numpy(), 1 / np.sqrt(2.0))


# ----------------------------------------------------------------- kernels ---
def _operand(kind, x, wb, scale=None):
    if kind == po.F:
        return cuda(x), po.Mat.dense(x)
    b = po.binarize(x, wb)
    dev = bg.BitOperand(bg.BitDenseMatrix.from_numpy(b, x.shape[0], x.shape[1], wb))
    return dev, po.Mat.binary(b, x.shape[0], x.shape[1], wb)


def _check_out(dev, ora, exact=True):
    if ora.prec == po.B:
        assert isinstance(dev, bg.BitOperand)
        assert bits_equal(dev.bits.numpy(), ora.bits)
    else:
        got = dev.cpu().numpy()
        if exact:
            assert np.array_equal(got, ora.f), rel_err(got, ora.f)
        else:
            assert rel_err(got, ora.f) <= 1e-6


BMM_VARIANTS = [f"BMM.{a}{b}{c}" for a in "FB" for b in "FB" for c in "FB" if (a, b, c) != ("F", "F", "F")]


@pytest.mark.parametrize("wb", [32, 64])
@pytest.mark.parametrize("v", BMM_VARIANTS)
@pytest.mark.parametrize("mkn", [(1, 1, 1), (7, 13, 5), (40, 33, 21), (33, 602, 128), (65, 128, 41), (9, 70, 300),
                                 (257, 602, 128), (48, 31, 127), (130, 100, 47), (64, 1433, 64), (35, 64, 16)])
def test_bmm_every_variant(v, wb, mkn):
    m, k, n = mkn
    rng = po.Rng(1000 + m + k + n)
    A, W = rng.random_dense(m, k), rng.random_dense(k, n)
    tv = po.parse_variant(v)
    da, oa = _operand(tv[1], A, wb)
    dw, ow = _operand(tv[2], W, wb)
    if tv[2] == po.B:  # weights carry their column scale, like run_mm_slot
        sc = po.l1_scales(W, po.COL)
        dw.scale = torch.from_numpy(sc).cuda()
        dw.scale_axis = bg.bitgnn.COL
        ow.scale = sc
    _check_out(bg.bmm(v, da, dw, wb), po.bmm(v, oa, ow, wb))


BSPMM_VARIANTS = [f"BSpMM.{a}{b}{c}" for a in "FB" for b in "FB" for c in "FB"]


@pytest.mark.parametrize("wb", [32, 64])
@pytest.mark.parametrize("v", BSPMM_VARIANTS)
@pytest.mark.parametrize("nef", [(5, 9, 3), (37, 150, 31), (64, 400, 33), (200, 4000, 40), (17, 40, 1),
                                 (300, 30000, 128), (150, 3000, 70), (90, 800, 520), (120, 2500, 300),
                                 (64, 900, 250), (200, 1500, 1000),
                                 # narrow F rows (sliver.cu k_sl_f_sub: 8 / 16 lanes per row)
                                 (400, 5000, 7), (600, 9000, 16), (500, 6000, 9), (1000, 20000, 2)])
def test_bspmm_every_variant(v, wb, nef):
    n, e, f = nef
    rng = po.Rng(2000 + n + e + f)
    s, d = rng.random_edges(n, e, True)
    A = po.frdc_from_edges(n, s, d, False)
    dA = bg.frdc_from_edges(n, s, d, False)
    srow = (0.1 + np.array([rng.uniform() for _ in range(n)])).astype(np.float32)
    scol = (0.1 + np.array([rng.uniform() for _ in range(n)])).astype(np.float32)
    X = rng.random_dense(n, f)
    tv = po.parse_variant(v)
    dx, ox = _operand(tv[1], X, wb)
    fac = tv[2] == po.F
    adj = bg.AdjacencyOperand(dA, cuda(srow[None])[0] if fac else None, cuda(scol[None])[0] if fac else None)
    got = bg.bspmm(v, adj, dx, None, wb)
    want = po.bspmm(v, A, ox, srow if fac else None, scol if fac else None, wb)
    _check_out(got, want)


def test_isolated_node_thresholds_to_one():
    # ref: test_kernels.cpp:305-321
    A = bg.frdc_from_edges(3, [1, 2], [2, 1], False)
    X = po.Rng(111).random_dense(3, 5)
    xb = bg.BitOperand(bg.binarize(cuda(X)))
    b = bg.bspmm("BSpMM.BBB", bg.AdjacencyOperand(A), xb)
    assert all(b.bits.bit(0, j) for j in range(5))
    f = bg.bspmm("BSpMM.BBF", bg.AdjacencyOperand(A), xb)
    assert torch.all(f[0] == 0.0)


def test_bspmm_rejects_inconsistent_factorization():
    # ref: test_kernels.cpp:323-349
    rng = po.Rng(112)
    s, d = rng.random_edges(8, 20, True)
    A = bg.frdc_from_edges(8, s, d, False)
    X = cuda(rng.random_dense(8, 4))
    xb = bg.BitOperand(bg.binarize(X))
    sr = torch.rand(8, device="cuda") + 0.1
    with pytest.raises(bg.InvalidArgument):
        bg.bspmm("BSpMM.BBB", bg.AdjacencyOperand(A, sr, sr), xb)
    with pytest.raises(bg.InvalidArgument):
        bg.bspmm("BSpMM.BFF", bg.AdjacencyOperand(A), xb)
    with pytest.raises(bg.InvalidArgument):
        bg.bspmm("BSpMM.FBF", bg.AdjacencyOperand(A), xb)
    with pytest.raises(bg.InvalidArgument):
        bg.bspmm("BSpMM.BBB", bg.AdjacencyOperand(A), X)
    with pytest.raises(bg.InvalidArgument):
        bg.bspmm("BSpMM.BBB", bg.AdjacencyOperand(A), bg.BitOperand(xb.bits, sr))
    with pytest.raises(bg.InvalidArgument):
        bg.bspmm("BSpMM.BBB", bg.AdjacencyOperand(A), bg.BitOperand(bg.binarize(cuda(rng.random_dense(7, 4)))))


def test_add_known_answers():
    # ref: test_kernels.cpp:350-377
    a, b = cuda([[1.5, -2.0]]), cuda([[0.25, 1.0]])
    f = bg.add("ADD.FFF", a, b).cpu().numpy()
    assert f[0, 0] == 1.75 and f[0, 1] == -1.0
    ba = bg.BitOperand(bg.binarize(cuda([[1, 1, -1]])))
    bb = bg.BitOperand(bg.binarize(cuda([[1, -1, -1]])))
    s = bg.add("ADD.BBF", ba, bb).cpu().numpy()
    assert list(s[0]) == [2.0, 0.0, -2.0]
    o = bg.add("ADD.BBB", ba, bb)
    assert o.bits.bit(0, 0) and o.bits.bit(0, 1) and not o.bits.bit(0, 2)
    with pytest.raises(bg.InvalidArgument):
        bg.add("ADD.BFB", ba, b)
    with pytest.raises(bg.InvalidArgument):
        bg.add("ADD.FFF", a, cuda(np.zeros((2, 2))))


def test_concat_known_answer():
    # ref: test_kernels.cpp:398-416
    a = bg.BitOperand(bg.binarize(cuda([[1, -1, 1]])))
    b = bg.BitOperand(bg.binarize(cuda([[-1, 1, 1, -1, 1]])))
    c = bg.concat("CONCAT.BBB", a, b)
    assert c.bits.cols == 8 and c.bits.numpy()[0, 0] == 0xAD000000
    d = bg.concat("CONCAT.BBF", a, b).cpu().numpy()
    assert list(d[0]) == [1, -1, 1, -1, 1, 1, -1, 1]


# ------------------------------------------------------------------ models ---
def _compare_model(model, n, e, f, h, c, seed_g=100, seed_m=99, plan=None, exact_logits=True):
    s, d = po.Rng(seed_g).random_edges(n, e, False)
    og = po.Graph(n, s, d)
    layers, X = po.build_model(model, f, h, c, seed_m, n, plan)
    o_out, o_log, o_pts = po.run_model(layers, og, X)
    g = bg.prepare_graph(n, s, d)
    m = bg.Model(to_layer_specs(bg, layers), g)
    out, logits, pts = m.forward_traced(cuda(X))
    assert [p.label for p in pts] == [p.label for p in o_pts]
    for p, q in zip(pts, o_pts):
        assert (p.bits.rows, p.bits.cols) == (q.rows, q.cols), p.label
        assert bits_equal(p.bits.numpy(), q.bits), p.label
    lg = logits.cpu().numpy()
    if exact_logits:
        assert np.array_equal(lg, o_log), rel_err(lg, o_log)
    assert rel_err(lg, o_log) <= 1e-5
    assert argmax_agreement(lg, o_log) == 1.0
    assert np.allclose(out.cpu().numpy(), o_out, rtol=1e-6, atol=1e-7)
    # the plain (graph-captured) forward agrees with the traced one
    for _ in range(3):
        out2 = m.forward(cuda(X))
    torch.cuda.synchronize()
    assert torch.equal(out2, out)
    return m, X


@pytest.mark.parametrize("model", ["gcn", "sage", "saint"])
def test_cora_shape_models_match_oracle(model):
    _compare_model(model, 2708, 13264, 1433, 64, 7)


def test_acceptance_cora_gcn_hidden16():
    # ref: test_acceptance.cpp:332-356
    _compare_model("gcn", 2708, 13264, 1433, 16, 7)


def test_pubmed_three_layer_gcn():
    plan = ["MM.FBB+BSpMM.BBB", "MM.BBB+BSpMM.BBB", "MM.BBF+BSpMM.FBF"]
    _compare_model("gcn", 19717, 88648, 500, 64, 3, plan=plan)


def test_word_bits_64_model():
    s, d = po.Rng(7).random_edges(300, 2000, False)
    layers, X = po.build_model("gcn", 70, 40, 5, 9, 300)
    og = po.Graph(300, s, d)
    o_out, o_log, o_pts = po.run_model(layers, og, X, word_bits=64)
    m = bg.Model(to_layer_specs(bg, layers), bg.prepare_graph(300, s, d), word_bits=64)
    out, logits, pts = m.forward_traced(cuda(X))
    assert all(bits_equal(p.bits.numpy(), q.bits) for p, q in zip(pts, o_pts))
    assert np.array_equal(logits.cpu().numpy(), o_log)


def test_timing_labels_match_reference():
    # ref: test_graphops.cpp:192-217
    s, d = po.Rng(303).random_edges(12, 30, False)
    layers, X = po.build_model("gcn", 6, 8, 4, 5, 12)
    m = bg.Model(to_layer_specs(bg, layers), bg.prepare_graph(12, s, d))
    _, t = m.forward_timed(cuda(X))
    assert [k.label for k in t] == ["layer0.mm[BMM.FBB]", "layer0.spmm[BSpMM.BBB]",
                                    "layer1.mm[BMM.BBF]", "layer1.spmm[BSpMM.FBF]", "layer2.softmax"]
    assert all(k.ms >= 0 for k in t)


def test_fault_injection_is_detected():
    # ref: runreport.cpp:55-63, test_cli.cpp:205-224
    s, d = po.Rng(100).random_edges(2708, 13264, False)
    layers, X = po.build_model("gcn", 1433, 16, 7, 99, 2708)
    og = po.Graph(2708, s, d)
    _, o_log, o_pts = po.run_model(layers, og, X)
    g = bg.prepare_graph(2708, s, d)
    g.corrupt_tile(0)
    m = bg.Model(to_layer_specs(bg, layers), g)
    _, logits, pts = m.forward_traced(cuda(X))
    mism = sum(int(np.count_nonzero(p.bits.numpy() != q.bits)) for p, q in zip(pts, o_pts))
    assert mism > 0 or not np.array_equal(logits.cpu().numpy(), o_log)


def test_host_forward_matches_device_forward():
    s, d = po.Rng(100).random_edges(2708, 13264, False)
    layers, X = po.build_model("gcn", 1433, 64, 7, 99, 2708)
    m = bg.Model(to_layer_specs(bg, layers), bg.prepare_graph(2708, s, d))
    dev = m.forward(cuda(X)).cpu()
    host, lg = m.forward_host(torch.from_numpy(X).pin_memory(), logits=True)
    assert torch.equal(host, dev)


def test_invalid_model_messages():
    layers = [bg.LayerSpec(bg._lib.LAYER_GCN, ["MM.FBB", "BSpMM.FBF"], np.ones((4, 4), np.float32))]
    errs = bg.validate_model(layers)
    assert "layer 0 gcn_conv: mm output tag does not feed the spmm input" in errs
    assert "model output must be full precision, got a binary tail" not in errs
    with pytest.raises(bg.InvalidArgument) as e:
        bg.Model(layers + [bg.LayerSpec(bg._lib.LAYER_BINARIZE)], bg.prepare_graph(4, [0], [1]))
    assert str(e.value).startswith("invalid model:")


@pytest.mark.parametrize("model,plan", [("gcn", None), ("sage", None), ("saint", None),
                                        ("gcn", ["MM.FBB+BSpMM.BBB", "MM.BBB+BSpMM.BBB", "MM.BBF+BSpMM.FBF"]),
                                        ("gcn", ["MM.FBF+BSpMM.FBF", "MM.FBF+BSpMM.FBF"])])
def test_streamed_host_forward_matches_device_forward(model, plan):
    # bg_model_forward_host streams X in row chunks (layer-0 MM per chunk) and
    # copies the output out per chunk; results must equal the device forward
    n, e = 19717, 88648
    s, d = po.Rng(100).random_edges(n, e, False)
    layers, X = po.build_model(model, 500, 64, 3, 99, n, plan)
    m = bg.Model(to_layer_specs(bg, layers), bg.prepare_graph(n, s, d))
    dev = m.forward(cuda(X)).cpu()
    _, dev_log, _ = m.forward_traced(cuda(X))
    for _ in range(2):  # repeated calls reuse the copy stream, events and buffers
        host, lg = m.forward_host(torch.from_numpy(X).pin_memory(), logits=True)
        assert torch.equal(host, dev)
        assert torch.equal(lg, dev_log.cpu())
    host2 = m.forward_host(X)  # pageable input
    assert torch.equal(host2, dev)


@pytest.mark.parametrize("v", ["BSpMM.FFF", "BSpMM.FBF", "BSpMM.BFF"])
@pytest.mark.parametrize("f", [1, 5, 7, 8, 9, 13, 16])
def test_narrow_rows_equal_warp_per_row(monkeypatch, v, f):
    # k_sl_f_sub (8 or 16 lanes per row) against k_sl_f (a warp per row,
    # BG_SLF_WARP=1): the same ascending double sums, so bit-identical
    n, e = 3000, 40000
    rng = po.Rng(7000 + f)
    s, d = rng.random_edges(n, e, False)
    dA = bg.frdc_from_edges(n, s, d, False)
    srow = (0.1 + np.array([rng.uniform() for _ in range(n)])).astype(np.float32)
    scol = (0.1 + np.array([rng.uniform() for _ in range(n)])).astype(np.float32)
    X = rng.random_dense(n, f)
    tv = po.parse_variant(v)
    dx, _ = _operand(tv[1], X, 32)
    fac = tv[2] == po.F
    adj = bg.AdjacencyOperand(dA, cuda(srow[None])[0] if fac else None, cuda(scol[None])[0] if fac else None)
    sub = bg.bspmm(v, adj, dx, None, 32).cpu()
    monkeypatch.setenv("BG_SLF_WARP", "1")
    warp = bg.bspmm(v, adj, dx, None, 32).cpu()
    assert torch.equal(sub, warp)
