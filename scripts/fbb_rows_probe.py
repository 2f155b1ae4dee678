"""Time MM.FBB (K=602, N=128, Reddit's layer 0) at shard-sized row counts on
each kernel (BG_FBB=scalar|tma): where the few-rows dispatch threshold sits."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2305_02522_b200 as bg  # noqa: E402

k, n = 602, 128
W = torch.rand(k, n, device="cuda") - 0.5
w = bg.BitOperand(bg.binarize(W))
for rows in (29121, 58242, 116483, 232965):
    X = torch.rand(rows, k, device="cuda") - 0.5
    res = []
    for kern in ("scalar", "tma"):
        os.environ["BG_FBB"] = kern
        for _ in range(3):
            bg.bmm("BMM.FBB", X, w)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            bg.bmm("BMM.FBB", X, w)
        b.record()
        b.synchronize()
        res.append((kern, round(a.elapsed_time(b) / 20 * 1e3, 1)))
    print(rows, res, flush=True)
