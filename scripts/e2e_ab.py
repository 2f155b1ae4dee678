"""A/B of the host entry point (bg_model_forward_host) under environment
settings, interleaved in one process: python scripts/e2e_ab.py [wl] 'A=1' 'B=2,C=3' ..."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
import paper_2305_02522_b200 as bg

wl = sys.argv[1]
settings = sys.argv[2:] or ["X=1"]
model_name, n, e, f, h, c, plan = bench.WORKLOADS[wl]
src, dst = bg.Rng(bench.GRAPH_SEED).random_edges(n, e, False)
layers, X = bg.build_model_spec(model_name, f, h, c, bench.MODEL_SEED, n, plan)
g = bg.prepare_graph(n, src, dst)
m = bg.Model(layers, g)
xh = torch.from_numpy(X).pin_memory()
ref = None
res = {s: [] for s in settings}
for rep in range(6):
    for st in settings:
        for kv in st.split(","):
            k, v = kv.split("=")
            os.environ[k] = v
        for _ in range(2):
            out = m.forward_host(xh)
        torch.cuda.synchronize()
        for _ in range(5):
            t = time.perf_counter()
            out = m.forward_host(xh)
            res[st].append((time.perf_counter() - t) * 1e3)
        o = out if isinstance(out, torch.Tensor) else torch.as_tensor(out)
        if ref is None:
            ref = o.clone()
        assert torch.equal(o, ref), st
        for kv in st.split(","):
            os.environ.pop(kv.split("=")[0], None)
for st, ts in res.items():
    ts.sort()
    print(st, "median", round(ts[len(ts) // 2], 3), "ms  min", round(ts[0], 3))
