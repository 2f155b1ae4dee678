"""bench.py's algorithmic-byte accounting against SURVEY.md §8(d)'s per-kernel
budget for the Reddit shape (FBB 564.7 MB, BBB 684.5 MB, BBF 41.9 MB, FBF
753.4 MB, softmax 76.4 MB), the roofline object, and the workload metadata."""
import importlib.util
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
bench = importlib.util.module_from_spec(spec)
spec.loader.exec_module(bench)

# Reddit FRDC sizes (112,757,282 tiles over ceil(N/4) tile rows)
N = 232_965
SHAPES = {"nodes": N, "features": 602, "hidden": 128, "classes": 41, "model": "gcn", "last_conv": 1,
          "loops_tile_rows": (N + 3) // 4, "loops_nnz_tiles": 112_757_282,
          "raw_tile_rows": (N + 3) // 4, "raw_nnz_tiles": 0}


@pytest.mark.parametrize("label,mb", [("layer0.mm[BMM.FBB]", 564.7), ("layer0.spmm[BSpMM.BBB]", 684.5),
                                      ("layer1.mm[BMM.BBF]", 41.9), ("layer1.spmm[BSpMM.FBF]", 753.4),
                                      ("layer2.softmax", 76.4)])
def test_reddit_bytes_match_the_survey_budget(label, mb):
    assert bench.kernel_bytes(label, SHAPES) / 1e6 == pytest.approx(mb, abs=0.05)


def test_paired_product_counts_two_weights_and_results_one_input():
    one = bench.kernel_bytes("layer0.mm_self[BMM.FBB]", SHAPES)
    pair = bench.kernel_bytes("layer0.mm_pair[BMM.FBB]", SHAPES)
    x = 4 * N * 602
    assert pair - x == 2 * (one - x)


def test_non_kernel_labels_count_nothing():
    assert bench.kernel_bytes("layer0.allgather", SHAPES) == 0
    assert bench.kernel_bytes("layer1.relu", SHAPES) == 0


def test_roofline_object_fields():
    dom = {"label": "layer1.spmm[BSpMM.FBF]", "ms": 0.66, "alg_bytes": 753_422_156}
    r = bench.roofline_obj(dom, 1141.5, 6545.9, "measured")
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["frac"] == pytest.approx(1141.5 / 6545.9, abs=1e-4)
    if "l2_to_sm_bytes" in r:  # from the committed ncu capture
        assert r["l2_to_sm_gbs"] == pytest.approx(r["l2_to_sm_bytes"] / 0.66e-3 / 1e9, rel=1e-3)


def test_workload_config_names_the_baseline_shapes():
    c = bench.workload_config("reddit", 114_727_589)
    assert c["nodes"] == N and c["features"] == 602 and c["classes"] == 41 and c["model_family"] == "gcn"
    for wl in bench.WORKLOADS:
        assert bench.workload_config(wl)["workload"]
    assert bench.peaks()[0] > 1000


def _ref_available():
    import sys
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po
    return po.ref_available()


@pytest.mark.skipif(not _ref_available(), reason="oracle/_ref (reference library) not built")
def test_reference_arm_never_maps_the_product_library():
    # The reference arm runs the unmodified reference only: its process must
    # not map libbitgnn_b200.so (the driver voids the ratio if it does).
    import json
    import subprocess
    import sys
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--workload", "cora", "--steps", "2", "--warmup", "3"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    libs = line["native_so_loaded"]
    assert "oracle/_ref/libbitgnn_ref.so" in libs
    assert not any("libbitgnn_b200" in x for x in libs), libs
    cb = line["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1
    assert cb["host_cpu"]["logical_cpus"] >= 1
    kb = cb["kernelbench_bspmm_bbb_1thread"]
    assert kb["values_match"] and kb["edges"] > 0 and kb["gteps"] > 0


def test_packed_layers_count_bits_and_fused_softmax():
    # products-shape SAINT: layer 1's MMs and the FC read the packed two-valued
    # activation; the FC writes logits and probabilities
    n = 2_449_029
    sh = {"nodes": n, "features": 100, "hidden": 128, "classes": 47, "model": "saint", "last_conv": 2,
          "loops_tile_rows": (n + 3) // 4, "loops_nnz_tiles": 0, "raw_tile_rows": (n + 3) // 4,
          "raw_nnz_tiles": 61_854_024, "packed_layers": [1, 2], "fused_softmax_layer": 2}
    w = 4 * 128 * 4 + 4 * 128
    assert bench.kernel_bytes("layer1.mm_self[BMM.FBB]", sh) == 16 * n + w + 16 * n
    assert bench.kernel_bytes("layer2.mm[BMM.FBF]", sh) == 16 * n + 4 * 47 * 4 + 4 * 47 + 2 * 4 * n * 47
    assert bench.kernel_bytes("layer0.mm_pair[BMM.FBB]", sh) == 400 * n + 2 * (4 * 128 * 4 + 4 * 128 + 16 * n)
