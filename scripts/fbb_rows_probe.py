"""Time MM.FBB on each kernel (BG_FBB=...) at the BASELINE shapes and their
shard-sized row counts: where the dispatch thresholds sit.
usage: fbb_rows_probe.py [kernels, default "default scalar tma tmem"]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2305_02522_b200 as bg  # noqa: E402

kerns = sys.argv[1:] or ["default", "scalar", "tma", "tmem"]
shapes = [(29121, 602, 128), (58242, 602, 128), (116483, 602, 128), (232965, 602, 128),  # Reddit (8/4/2/1 shards)
          (11157, 500, 256), (44625, 500, 256), (89250, 500, 256),                        # Flickr
          (19717, 500, 64), (2708, 1433, 64)]                                              # PubMed, Cora
for rows, k, n in shapes:
    W = torch.rand(k, n, device="cuda") - 0.5
    w = bg.BitOperand(bg.binarize(W))
    X = torch.rand(rows, k, device="cuda") - 0.5
    flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")  # 256 MB > L2
    res = []
    for kern in kerns:
        if kern == "default":
            os.environ.pop("BG_FBB", None)
        else:
            os.environ["BG_FBB"] = kern
        for _ in range(3):
            bg.bmm("BMM.FBB", X, w)
        ts = []
        for _ in range(10):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            bg.bmm("BMM.FBB", X, w)
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        res.append((kern, round(sorted(ts)[len(ts) // 2], 1)))
    print((rows, k, n), res, flush=True)
os.environ.pop("BG_FBB", None)
