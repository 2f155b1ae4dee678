"""One forced F->B product (BG_FBB selects the kernel) checked against the
oracle: python scripts/fbb_debug.py M K N"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import numpy as np
import torch
import pyoracle as po
import paper_2305_02522_b200 as bg

m, k, n = (int(v) for v in sys.argv[1:4])
wb = 32
rng = po.Rng(4242 + m + k + n)
A, W = rng.random_dense(m, k), rng.random_dense(k, n)
wbits = po.binarize(W, wb)
dw = bg.BitOperand(bg.BitDenseMatrix.from_numpy(wbits, k, n, wb))
ow = po.Mat.binary(wbits, k, n, wb)
got = bg.bmm("BMM.FBB", torch.from_numpy(A).cuda(), dw, wb)
torch.cuda.synchronize()
want = po.bmm("BMM.FBB", po.Mat.dense(A), ow, wb)
g, w = got.bits.numpy(), want.bits
bad = (g != w).any(axis=1)
print("equal:", np.array_equal(g, w), "rows differing:", int(bad.sum()),
      "per 32-row quarter of each tile:", [int(bad[q::1].reshape(-1)[:0].sum()) for q in range(0)] or
      [int(sum(bad[t * 128 + 32 * q: t * 128 + 32 * q + 32].sum() for t in range((len(bad) + 127) // 128))) for q in range(4)])
if not np.array_equal(g, w):
    i = int(np.nonzero((g != w).any(axis=1))[0][0])
    print("row", i, "got", [hex(v) for v in g[i]], "want", [hex(v) for v in w[i]])
