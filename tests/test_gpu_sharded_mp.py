"""GPU, several PROCESSES: the product's row-sharded forward
(bg_model_forward_sharded) with a real exchange between ranks.

World 2 and 3 run as separate processes on the one B200 of the test box.
Each rank holds only its slice of the graph (bg_graph_shard), computes its
node rows through the engine and exchanges the packed aggregation operand
through bg_comm_create_external with a host-staged gloo all-gather (NCCL
refuses two ranks on one device, and the engine code around the exchange is
the same).  Every rank's output rows must be torch.equal to the 1-GPU
forward's.  A 1-rank NCCL communicator runs the NCCL exchange code itself,
graph-captured, in-process (per-rank semantics of run_model,
graphops.cpp:390-484)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SHAPES = {  # model, nodes, edge draws, features, hidden, classes, plan
    "reddit": ("gcn", 232_965, 114_615_892, 602, 128, 41, None),
    "pubmed3": ("gcn", 19_717, 88_648, 500, 64, 3,
                ["MM.FBB+BSpMM.BBB", "MM.BBB+BSpMM.BBB", "MM.BBF+BSpMM.FBF"]),
    "saint": ("saint", 300_000, 7_500_000, 100, 128, 47, None),
    "sage": ("sage", 89_250, 899_756, 500, 256, 7, None),
    # a binary model input straight into the fused MM.BBF + BSpMM.FBF layer
    "gcn_bin_in": ("gcn", 5_000, 40_000, 96, 64, 5, ["MM.BBF+BSpMM.FBF"]),
}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, shape, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import paper_2305_02522_b200 as bg
        from paper_2305_02522_b200.sharded import ShardedModel

        model, n, e, f, h, c, plan = SHAPES[shape]
        src, dst = bg.Rng(100).random_edges(n, e, False)
        layers, X = bg.build_model_spec(model, f, h, c, 99, n, plan)
        g = bg.prepare_graph(n, src, dst)
        x = torch.from_numpy(X).cuda()
        binary_in = plan is not None and plan[0].startswith("MM.B")
        if binary_in:  # a binary model input (the fused-GCN input-copy path)
            bits = bg.binarize(x)
            x = bg.BitOperand(bits)
        m1 = bg.Model(layers, g, input_precision=bg.B if binary_in else bg.F)
        want_out, want_log, _ = m1.forward_traced(x)
        sm = ShardedModel(layers, g, dist, world, rank, transport="host",
                          input_precision=bg.B if binary_in else bg.F)
        del m1, g  # this rank now holds its FRDC slice only
        torch.cuda.synchronize()
        r0, r1 = sm.row0, sm.row1
        ok = True
        for _ in range(2):  # repeated forwards reuse the pool and views
            lg = torch.empty((r1 - r0, c), dtype=torch.float32, device="cuda")
            out = sm.forward(x, logits=lg)
            torch.cuda.synchronize()
            ok &= bool(torch.equal(out, want_out[r0:r1])) and bool(torch.equal(lg, want_log[r0:r1]))
        info = (rank, r0, r1, ok, sm.comm.calls, sm.graph.structure.node_rows, sm.graph.structure.nnz_tiles)
        gathered = [None] * world
        dist.all_gather_object(gathered, info)
        if rank == 0:
            q.put(gathered)
    except Exception as ex:  # surfaces in the parent
        import traceback
        q.put(("error", rank, traceback.format_exc()))
        raise
    finally:
        dist.destroy_process_group()


def _run(world, shape):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, shape, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=900)
    for p in procs:
        p.join(120)
    assert not (isinstance(res, tuple) and res[0] == "error"), res
    assert all(p.exitcode == 0 for p in procs)
    return res


@pytest.mark.timeout(1200)
@pytest.mark.parametrize("world,shape", [(2, "reddit"), (3, "reddit"), (2, "pubmed3"), (3, "saint"),
                                         (2, "sage"), (3, "gcn_bin_in")])
def test_multiprocess_sharded_forward_equals_single_gpu(world, shape):
    res = _run(world, shape)
    n = SHAPES[shape][1]
    assert [r[0] for r in res] == list(range(world))
    assert res[0][1] == 0 and res[-1][2] == n
    assert all(res[k][2] == res[k + 1][1] for k in range(world - 1))  # contiguous ranges
    for rank, r0, r1, ok, calls, shard_rows, shard_tiles in res:
        assert ok, f"rank {rank} rows [{r0}, {r1}) differ from the 1-GPU forward"
        assert calls > 0  # the exchange really ran
        assert shard_rows == r1 - r0  # each rank holds its FRDC slice only
    assert sum(r[6] for r in res) > 0


@pytest.mark.parametrize("shape", ["pubmed3", "sage", "saint"])
def test_one_rank_nccl_exchange_graph_captured(shape):
    # bg_comm_create with world 1: the grouped NCCL broadcast code path runs
    # (and is captured in the CUDA graph with the kernels from the second call)
    sys.path.insert(0, ROOT)
    import paper_2305_02522_b200 as bg
    from paper_2305_02522_b200.sharded import ShardedModel

    model, n, e, f, h, c, plan = SHAPES[shape]
    src, dst = bg.Rng(100).random_edges(n, e, False)
    layers, X = bg.build_model_spec(model, f, h, c, 99, n, plan)
    g = bg.prepare_graph(n, src, dst)
    x = torch.from_numpy(X).cuda()
    want = bg.Model(layers, g).forward_traced(x)[0]
    sm = ShardedModel(layers, g, None, 1, 0, transport="nccl1")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        out = torch.empty((n, c), dtype=torch.float32, device="cuda")
        for _ in range(4):  # eager, capture, replay, replay
            out.zero_()
            sm.forward(x, out)
            s.synchronize()
            assert torch.equal(out, want)
    _, tl = sm.forward_timed(x)
    assert any(t.label.endswith("allgather") for t in tl)
