"""Per-op device times of the sharded forward at Reddit shape with W virtual
ranks (every rank's range in this process, so each op's time is the sum over
ranks): how the aggregation layout choice behaves at shard size."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2305_02522_b200 as bg  # noqa: E402
from paper_2305_02522_b200 import _lib as L  # noqa: E402
from paper_2305_02522_b200.sharded import partition_bounds  # noqa: E402
from paper_2305_02522_b200.bitgnn import KernelTiming, _mat, _stream  # noqa: E402
import ctypes as C  # noqa: E402

n, e, f, h, c = 232_965, 114_615_892, 602, 128, 41
src, dst = bg.Rng(100).random_edges(n, e, False)
layers, X = bg.build_model_spec("gcn", f, h, c, 99, n, None)
g = bg.prepare_graph(n, src, dst)
m = bg.Model(layers, g)
x = torch.from_numpy(X).cuda()
rp, _, _ = g.structure.download()
for world in (1, 2, 4, 8):
    b = np.asarray(partition_bounds(rp, n, world), np.int64)
    for mode in ((L.AGG_AUTO,) if os.environ.get("AUTO_ONLY") else (L.AGG_AUTO, L.AGG_WINDOW, L.AGG_SLIVERS)):
        bg.set_aggregation(mode, 0)
        out = torch.empty((n, c), device="cuda")
        arr = (L.KernelTiming * 64)()
        cnt = C.c_int()
        cx = _mat(x)
        for _ in range(3):
            L.check(L.lib().bg_model_forward_sharded_timed(m._h, None, C.byref(cx), b.ctypes.data, world, 0,
                                                           out.data_ptr(), arr, 64, C.byref(cnt), _stream()))
        t = {arr[i].label.decode(): round(arr[i].ms, 3) for i in range(cnt.value)}
        print(world, mode, t, flush=True)
bg.set_aggregation(L.AGG_AUTO, 0)
