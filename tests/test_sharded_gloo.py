"""CPU, world_size 2 over gloo: the host-side protocol of the row-sharded
forward -- tile-row partition (C ABI bg_partition_bounds), row-local dense
transforms, all-gather of the packed aggregation operand before each
neighbour aggregation, reassembly -- reproduces the single-process forward.
Compute here is the oracle (there is no GPU on this box); the same
partition and exchange points are what bg_model_forward_sharded runs with
NCCL on the GPUs."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _allgather_rows(local: np.ndarray, bounds, rank, world):
    """All-gather uneven row slices (pad to the largest slice)."""
    width = local.shape[1]
    mx = max(bounds[k + 1] - bounds[k] for k in range(world))
    buf = torch.zeros((mx, width), dtype=torch.from_numpy(local[:0]).dtype)
    buf[: local.shape[0]] = torch.from_numpy(local)
    parts = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf)
    return np.concatenate([parts[k][: bounds[k + 1] - bounds[k]].numpy() for k in range(world)])


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import pyoracle as po
        from paper_2305_02522_b200.sharded import partition_bounds

        n, e = 1001, 9000
        s, d = po.Rng(100).random_edges(n, e, False)
        layers, X = po.build_model("gcn", 70, 40, 5, 99, n)
        g = po.Graph(n, s, d)
        bounds = partition_bounds(g.structure.row_ptr, n, world)
        allb = [None] * world
        dist.all_gather_object(allb, bounds)
        assert all(b == bounds for b in allb)
        r0, r1 = bounds[rank], bounds[rank + 1]
        # layer 0: MM.FBB row-local on this rank's rows
        w1 = layers[0].w1
        wb = po.Mat.binary(po.binarize(w1), *w1.shape)
        wb.scale = po.l1_scales(w1, po.COL)
        h1 = po.bmm("MM.FBB", po.Mat.dense(X[r0:r1]), wb).bits
        # exchange point: the packed aggregation operand
        h1_full = _allgather_rows(h1.view(np.int32), bounds, rank, world).view(np.uint32)
        h2 = po.bspmm("BSpMM.BBB", g.structure, po.Mat.binary(h1_full, n, w1.shape[1])).bits[r0:r1]
        h2_full = _allgather_rows(h2.view(np.int32), bounds, rank, world).view(np.uint32)
        w2 = layers[1].w1
        wb2 = po.Mat.binary(po.binarize(w2), *w2.shape)
        wb2.scale = po.l1_scales(w2, po.COL)
        y = po.bmm("MM.BBF", po.Mat.binary(h2_full, n, w1.shape[1]), wb2).f  # replicated (cheap)
        logits = po.bspmm("BSpMM.FBF", g.structure, po.Mat.dense(y)).f[r0:r1]
        gathered = _allgather_rows(logits, bounds, rank, world)
        if rank == 0:
            _, ref_log, _ = po.run_model(layers, g, X)
            q.put(bool(np.array_equal(gathered, ref_log)))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_gloo_protocol_matches_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(240)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5) is True
