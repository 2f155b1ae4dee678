"""BSpMM.BBB on a Reddit-size graph with a heavy-tailed degree profile
(Zipf endpoints) vs the uniform one, per aggregation layout (CUDA events).
The windowed kernel gives a warp's 32 rows one loop count per step
(DESIGN.md 4.5); this measures what a skewed profile costs it."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2305_02522_b200 as bg  # noqa: E402
from paper_2305_02522_b200 import _lib as L  # noqa: E402

sys.path.insert(0, "tests")
sys.path.insert(0, "oracle")
from test_gpu_window import _power_law_edges  # noqa: E402

n, e = 232_965, 114_615_892
out = {}
for name in (sys.argv[1:] or ("uniform", "zipf1.4")):
    if name == "uniform":
        s, d = bg.Rng(100).random_edges(n, e, False)
    else:
        s, d = _power_law_edges(n, e, 100)
    A = bg.frdc_from_edges(n, s, d, True)
    x = bg.BitOperand(bg.binarize(torch.rand(n, 128, device="cuda") - 0.5))
    info = A.info()
    res = {"nnz_bits": info.nnz_bits, "max_degree": info.max_row_degree}
    for mode, mname in ((L.AGG_AUTO, "auto"), (L.AGG_WINDOW, "window"), (L.AGG_SLIVERS, "slivers")):
        bg.set_aggregation(mode, 0)
        for _ in range(3):
            bg.bspmm("BSpMM.BBB", bg.AdjacencyOperand(A), x)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            bg.bspmm("BSpMM.BBB", bg.AdjacencyOperand(A), x)
        b.record()
        b.synchronize()
        ms = a.elapsed_time(b) / 10
        res[mname] = {"ms_per_call_incl_alloc": round(ms, 4), "gteps": round(info.nnz_bits / ms / 1e6, 1)}
    bg.set_aggregation(L.AGG_AUTO, 0)
    out[name] = res
    print(name, json.dumps(res), flush=True)
