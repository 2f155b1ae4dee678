"""Is a small-graph forward host-bound?  Per step: host time of the public
forward call (no sync) vs device time (CUDA events over many steps).
usage: python scripts/host_probe.py [cora|pubmed ...]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2305_02522_b200 as bg

for wl in sys.argv[1:] or ["cora", "pubmed"]:
    model_name, n, e, f, h, c, plan = bench.WORKLOADS[wl]
    src, dst = bg.Rng(bench.GRAPH_SEED).random_edges(n, e, False)
    layers, X = bg.build_model_spec(model_name, f, h, c, bench.MODEL_SEED, n, plan)
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        g = bg.prepare_graph(n, src, dst)
        m = bg.Model(layers, g)
        x = torch.from_numpy(X).cuda()
        out = torch.empty((n, c), dtype=torch.float32, device="cuda")
        for _ in range(50):
            m.forward(x, out)
        stream.synchronize()
        K = 2000
        t0 = time.perf_counter()
        for _ in range(K):
            m.forward(x, out)
        t_host = (time.perf_counter() - t0) / K * 1e6
        stream.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(K):
            m.forward(x, out)
        e1.record(stream)
        e1.synchronize()
        t_dev = e0.elapsed_time(e1) / K * 1e3
        # device time of one captured forward replayed back to back from a
        # graph of 20 forwards (no host in between)
        m.set_graph_capture(False)  # its kernels go straight into the outer capture
        m.forward(x, out); stream.synchronize()
        cg = torch.cuda.CUDAGraph()
        with torch.cuda.graph(cg, stream=stream):
            for _ in range(20):
                m.forward(x, out)
        cg.replay(); stream.synchronize()
        e0.record(stream)
        for _ in range(50):
            cg.replay()
        e1.record(stream)
        e1.synchronize()
        t_gg = e0.elapsed_time(e1) / (50 * 20) * 1e3
    print(f"{wl}: host per forward call {t_host:.1f} us, device per step {t_dev:.1f} us, "
          f"forward inside a graph of 20 {t_gg:.1f} us")
