"""A/B of one FBB shape under several environment settings, interleaved:
python scripts/fbb_ab.py ROWS K N 'ENV=a' 'ENV=b' ...  (each setting re-imports nothing:
the variables are read per call where the kernel reads them)"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2305_02522_b200 as bg  # noqa: E402

rows, k, n = (int(v) for v in sys.argv[1:4])
settings = sys.argv[4:]
W = torch.rand(k, n, device="cuda") - 0.5
w = bg.BitOperand(bg.binarize(W))
X = torch.rand(rows, k, device="cuda") - 0.5
flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
res = {s: [] for s in settings}
for rep in range(5):
    for st in settings:
        for kv in st.split(","):
            key, val = kv.split("=")
            os.environ[key] = val
        for _ in range(2):
            bg.bmm("BMM.FBB", X, w)
        for _ in range(10):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            bg.bmm("BMM.FBB", X, w)
            b.record()
            b.synchronize()
            res[st].append(a.elapsed_time(b) * 1e3)
for st, ts in res.items():
    ts.sort()
    print(st, "median", round(ts[len(ts) // 2], 1), "min", round(ts[0], 1))
