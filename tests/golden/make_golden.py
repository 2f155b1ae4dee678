#!/usr/bin/env python
"""Generate tests/golden/reference_fixtures.json from the REAL reference.

Runs the unmodified reference library (oracle/_ref, compiled from
/root/reference/proj/src by oracle/Makefile) on small seeded configurations
and records SHA-256 digests of everything the parity tests compare:
generated inputs (edges, X, W), both FRDC structures, every binarization
trace point (labels in order) and the logits / softmax output.  The fixtures
travel with the repo, so the GPU box (where /root/reference is absent) can
check the oracle and the CUDA path against the reference's own outputs.

    python tests/golden/make_golden.py
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import pyoracle as po  # noqa: E402

# (name, model, nodes, edge draws, features, hidden, classes, graph seed, model seed, plan, word_bits)
CASES = [
    ("acceptance_cora_gcn_h16", "gcn", 2708, 13264, 1433, 16, 7, 100, 99, None, 32),
    ("cora_gcn_h64", "gcn", 2708, 10556, 1433, 64, 7, 100, 99, None, 32),
    ("cora_sage_h64", "sage", 2708, 10556, 1433, 64, 7, 100, 99, None, 32),
    ("cora_saint_h64", "saint", 2708, 10556, 1433, 64, 7, 100, 99, None, 32),
    ("pubmed_gcn_3layer", "gcn", 19717, 88648, 500, 64, 3, 100, 99,
     ["MM.FBB+BSpMM.BBB", "MM.BBB+BSpMM.BBB", "MM.BBF+BSpMM.FBF"], 32),
    ("small_gcn_wb64", "gcn", 300, 2000, 70, 40, 5, 7, 9, None, 64),
    ("small_gcn_full_precision_norm", "gcn", 500, 3000, 40, 24, 6, 11, 12,
     ["MM.FBF+BSpMM.FFF", "MM.FBF+BSpMM.FFF"], 32),
    ("small_sage_mixed", "sage", 400, 2500, 33, 20, 5, 13, 14,
     ["MM.FBF+MM.FBB+BSpMM.BBF+ADD.FFF", "MM.FBF+MM.FBF+BSpMM.FFF+ADD.FFF"], 32),
    ("small_graphconv_bfb", "saint", 350, 2400, 45, 32, 4, 15, 16,
     ["MM.FBB+MM.FBB+BSpMM.BFB+ADD.BBF", "MM.FBB+MM.FBB+BSpMM.BBB+ADD.BBB", "MM.BBF"], 32),
]


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    if not po.ref_available():
        po.build()
    out = {"generator": "tests/golden/make_golden.py (real reference via oracle/_ref)",
           "cases": []}
    for (name, model, n, e, f, h, c, gs, ms, plan, wb) in CASES:
        src, dst = po.ref_random_edges(gs, n, e, False)
        rg = po.RefGraph(n, src, dst)
        rm = po.RefModel(rg, model, f, h, c, ms, n, wb, plan)
        X = rm.features()
        ws = rm.weights()
        o, lg, pts = rm.run(c)
        a, r = rg.frdc(0), rg.frdc(1)
        norm, mean, cnt = rg.scales()
        out["cases"].append({
            "name": name, "model": model, "nodes": n, "edge_draws": e, "features": f,
            "hidden": h, "classes": c, "graph_seed": gs, "model_seed": ms, "plan": plan,
            "word_bits": wb, "edges": int(src.shape[0]),
            "sha_src": sha(src), "sha_dst": sha(dst), "sha_x": sha(X),
            "sha_w": [[sha(w) if w is not None else None for w in pair] for pair in ws],
            "frdc_loops": {"nnz": a.nnz, "sha_row_ptr": sha(a.row_ptr), "sha_col_ind": sha(a.col_ind),
                           "sha_tiles": sha(a.tiles)},
            "frdc_raw": {"nnz": r.nnz, "sha_row_ptr": sha(r.row_ptr), "sha_col_ind": sha(r.col_ind),
                         "sha_tiles": sha(r.tiles)},
            "sha_norm": sha(norm), "sha_mean_row": sha(mean), "sha_neighbor_count": sha(cnt),
            "trace": [{"label": p.label, "rows": p.rows, "cols": p.cols, "word_bits": p.word_bits,
                       "sha": sha(p.bits)} for p in pts],
            "sha_logits": sha(lg), "logits_row0": [float(v) for v in lg[0]],
            "sha_out": sha(o),
        })
        print(name, "trace points", len(pts), flush=True)
    with open(os.path.join(HERE, "reference_fixtures.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
