#!/usr/bin/env python
"""Record the REAL reference's own FRDC build at the full BASELINE shapes.

Runs the unmodified reference (oracle/_ref, compiled from
/root/reference/proj/src) -- random_edges(Rng(100)) (rng.hpp:66-80) then
prepare_graph (graphops.cpp:146-170, i.e. frdc_from_edges twice,
bitsparse.cpp:72-112, plus the degree scales) -- at the Reddit and
ogbn-products shapes, and writes SHA-256 digests of both adjacency
structures (A+I and loop-free A) and of the scale vectors to
tests/golden/fullsize_frdc.json.  The reference's single-threaded sorts take
~45 s (Reddit) and ~20 s (products) here, once; the GPU box, where
/root/reference is absent, compares the device-built FRDC against these
digests (tests/test_gpu_fullsize.py).

    python tests/golden/make_fullsize_frdc.py
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import pyoracle as po  # noqa: E402

# name: (nodes, edge draws) -- bench.py WORKLOADS, graph seed 100
SHAPES = {"reddit": (232_965, 114_615_892), "products": (2_449_029, 61_859_140)}


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    out = {"generator": "tests/golden/make_fullsize_frdc.py (reference prepare_graph via oracle/_ref)",
           "graph_seed": 100, "shapes": {}}
    for name, (n, e) in SHAPES.items():
        t = time.time()
        src, dst = po.ref_random_edges(100, n, e, False)
        rg = po.RefGraph(n, src, dst)
        rec = {"nodes": n, "edge_draws": e, "edges": int(src.shape[0]),
               "sha_src": sha(src), "sha_dst": sha(dst)}
        for which, key in ((0, "loops"), (1, "raw")):
            f = rg.frdc(which)
            rec[key] = {"nnz_tiles": int(f.nnz), "nnz_bits": int(f.nnz_bits()),
                        "sha_row_ptr": sha(f.row_ptr), "sha_col_ind": sha(f.col_ind),
                        "sha_tiles": sha(f.tiles)}
        norm, mean, cnt = rg.scales()
        rec.update(sha_norm=sha(norm), sha_mean_row=sha(mean), sha_neighbor_count=sha(cnt))
        out["shapes"][name] = rec
        print(name, f"{time.time() - t:.1f}s", rec["loops"]["nnz_tiles"], flush=True)
        del rg
    with open(os.path.join(HERE, "fullsize_frdc.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
