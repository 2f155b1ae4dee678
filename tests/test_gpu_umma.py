"""MM.FBB on every kernel (BG_FBB forces one): the tcgen05 tensor cores (bmm.cu k_fbb_umma /
k_fbb_umma2, opt-in BG_FBB=umma|umma2), the TMA-fed and direct mma.sync kernels and the
warp-per-row popcount kernel:
+-1 int8 operands in shared memory, s32 accumulators in TMEM.  Bit-exact
against the oracle on tile-aligned and ragged shapes (partial 128-row tiles,
odd K, N below the 128-column MMA, 64-bit words)."""
import numpy as np
import pytest
import torch

import pyoracle as po
from helpers import bits_equal

import paper_2305_02522_b200 as bg

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["tc", "umma", "umma2", "tma", "imma", "scalar", "bulk", "tmem", "tmem2"])
def umma(monkeypatch, request):
    # umma: LDG-fed conversion; umma2: bulk-copied fp32 sub-tiles (TMA ring);
    # and the non-tcgen05 paths the default dispatch picks by shape: the
    # TMA-fed mma.sync kernel, the direct mma.sync kernel, a warp per row
    monkeypatch.setenv("BG_FBB", request.param)


@pytest.mark.parametrize("wb", [32, 64])
@pytest.mark.parametrize("mkn", [(128, 602, 128), (1000, 602, 128), (257, 33, 21), (300, 100, 128), (129, 500, 64),
                                 (5, 17, 7), (4096, 301, 96), (640, 1024, 128), (77, 64, 32), (2000, 1433, 64),
                                 (333, 200, 72), (50, 90, 40), (2711, 1433, 100)])
def test_fbb_umma_matches_oracle(umma, wb, mkn):
    m, k, n = mkn
    rng = po.Rng(4242 + m + k + n)
    A, W = rng.random_dense(m, k), rng.random_dense(k, n)
    A.flat[::13] = 0.0
    A.flat[5::17] = -0.0
    wbits = po.binarize(W, wb)
    dw = bg.BitOperand(bg.BitDenseMatrix.from_numpy(wbits, k, n, wb))
    ow = po.Mat.binary(wbits, k, n, wb)
    sc = po.l1_scales(W, po.COL)
    dw.scale = torch.from_numpy(sc).cuda()
    dw.scale_axis = bg.bitgnn.COL
    ow.scale = sc
    got = bg.bmm("BMM.FBB", torch.from_numpy(A).cuda(), dw, wb)
    want = po.bmm("BMM.FBB", po.Mat.dense(A), ow, wb)
    assert bits_equal(got.bits.numpy(), want.bits)


@pytest.mark.parametrize("wb", [32, 64])
@pytest.mark.parametrize("mkn", [(128, 602, 41), (1000, 128, 47), (257, 33, 21), (300, 100, 128), (5, 17, 7),
                                 (4096, 301, 96), (77, 64, 32), (2000, 1433, 64), (333, 200, 72)])
def test_fbf_matches_oracle(umma, wb, mkn):
    # MM.FBF: float((alpha_r * dot) * beta_c) in double with row scales of X
    # and column scales of W (kernels.cpp:179-190) -- exact
    m, k, n = mkn
    rng = po.Rng(5151 + m + k + n)
    A, W = rng.random_dense(m, k), rng.random_dense(k, n)
    A.flat[::11] = 0.0
    wbits = po.binarize(W, wb)
    dw = bg.BitOperand(bg.BitDenseMatrix.from_numpy(wbits, k, n, wb))
    ow = po.Mat.binary(wbits, k, n, wb)
    sc = po.l1_scales(W, po.COL)
    dw.scale = torch.from_numpy(sc).cuda()
    dw.scale_axis = bg.bitgnn.COL
    ow.scale = sc
    got = bg.bmm("BMM.FBF", torch.from_numpy(A).cuda(), dw, wb)
    want = po.bmm("BMM.FBF", po.Mat.dense(A), ow, wb)
    assert np.array_equal(got.cpu().numpy(), want.f)


@pytest.mark.parametrize("mkn", [(120000, 602, 128), (20000, 500, 256), (100003, 301, 96)])
def test_default_fbb_at_dispatch_sizes(mkn):
    # the default dispatch at the sizes where the 2-CTA tcgen05 kernel
    # (fbb_tmem.cu, cta_group::2) takes over: Reddit-like rows, Flickr-like
    # 256 columns, a ragged shape -- against the oracle
    m, k, n = mkn
    rng = po.Rng(777 + m + k + n)
    A, W = rng.random_dense(m, k), rng.random_dense(k, n)
    A.flat[::13] = 0.0
    A.flat[5::17] = -0.0
    wbits = po.binarize(W, 32)
    dw = bg.BitOperand(bg.BitDenseMatrix.from_numpy(wbits, k, n, 32))
    ow = po.Mat.binary(wbits, k, n, 32)
    got = bg.bmm("BMM.FBB", torch.from_numpy(A).cuda(), dw, 32)
    want = po.bmm("BMM.FBB", po.Mat.dense(A), ow, 32)
    assert bits_equal(got.bits.numpy(), want.bits)


@pytest.mark.parametrize("mkn", [(1000, 602, 128), (300, 100, 128), (4096, 301, 96), (257, 33, 21)])
def test_fbb_special_values(umma, mkn):
    # the fp32 -> +-1 conversion of every kernel on the values a sign test
    # can get wrong: -0.0 (>= 0), NaN (not >= 0, either sign), +-inf,
    # subnormals of both signs, the smallest normals
    m, k, n = mkn
    rng = po.Rng(9090 + m + k + n)
    A, W = rng.random_dense(m, k), rng.random_dense(k, n)
    special = np.array([0.0, -0.0, np.nan, -np.nan, np.inf, -np.inf, 1e-45, -1e-45, 1e-40, -1e-40,
                        np.finfo(np.float32).tiny, -np.finfo(np.float32).tiny], dtype=np.float32)
    idx = rng.random_dense(1, m * k // 3).ravel()
    pos = (np.abs(idx) * 1e6).astype(np.int64) % (m * k)
    A.flat[pos] = special[np.arange(pos.size) % special.size]
    wbits = po.binarize(W, 32)
    dw = bg.BitOperand(bg.BitDenseMatrix.from_numpy(wbits, k, n, 32))
    ow = po.Mat.binary(wbits, k, n, 32)
    got = bg.bmm("BMM.FBB", torch.from_numpy(A).cuda(), dw, 32)
    want = po.bmm("BMM.FBB", po.Mat.dense(A), ow, 32)
    assert bits_equal(got.bits.numpy(), want.bits)
