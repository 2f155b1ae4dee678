"""CPU: the C-ABI library loads and exports every entry point the header
declares, and its host-side logic (variant algebra, model validation,
synthetic-input generators) matches the reference -- no GPU needed."""
import ctypes
import hashlib
import json
import os
import re
import subprocess

import numpy as np
import pytest

import pyoracle as po

import paper_2305_02522_b200 as bg
from paper_2305_02522_b200 import _lib as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "bitgnn_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(bg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    syms = declared_symbols()
    assert len(syms) >= 45
    lib = ctypes.CDLL(L.LIB_PATH)
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # and the Python binding declares a prototype for each
    assert set(syms) <= set(L.PROTOTYPES)


def test_only_the_c_abi_is_exported():
    out = subprocess.run(["nm", "-D", "--defined-only", L.LIB_PATH], capture_output=True, text=True).stdout
    names = [l.split()[-1] for l in out.splitlines() if " T " in l]
    assert names and all(n.startswith("bg_") for n in names), [n for n in names if not n.startswith("bg_")][:5]


def test_library_is_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", L.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_variant_tables():
    # ref: test_kernels.cpp:79-95 -- 7 BMM, 8 BSpMM, 3 ADD, 3 CONCAT members
    counts = {}
    for op in range(4):
        counts[op] = sum(bg.KernelVariant(op, a, b, c).valid() for a in (0, 1) for b in (0, 1) for c in (0, 1))
    assert counts == {0: 7, 1: 8, 2: 3, 3: 3}


def test_variant_parse_and_names():
    # ref: test_kernels.cpp:97-112
    for name in ["BMM.FBB", "BMM.BBB", "BSpMM.FBF", "BSpMM.BBB", "ADD.BBF", "CONCAT.FFF"]:
        assert bg.KernelVariant.parse(name).name() == name
    assert bg.KernelVariant.parse("MM.FBB").name() == "BMM.FBB"
    assert bg.KernelVariant.parse("mm.fbb").name() == "BMM.FBB"
    assert bg.KernelVariant.parse("bspmm.bbf").name() == "BSpMM.BBF"
    assert not bg.KernelVariant.parse("BMM.FFF").valid()
    for bad in ["BMM", "BMM.FF", "BMM.FFFF", "BMM.XYZ", "NOPE.FFF"]:
        with pytest.raises(bg.InvalidArgument):
            bg.KernelVariant.parse(bad)


def test_validate_model_messages():
    # ref: graphops.cpp:172-268 (messages asserted by test_graphops.cpp:406-469)
    K = L
    W = np.ones((4, 4), np.float32)
    ok = [bg.LayerSpec(K.LAYER_GCN, ["MM.FBB", "BSpMM.BBB"], W), bg.LayerSpec(K.LAYER_GCN, ["MM.BBF", "BSpMM.FBF"], W),
          bg.LayerSpec(K.LAYER_SOFTMAX)]
    assert bg.validate_model(ok) == []
    errs = bg.validate_model(ok, has_graph=False)
    assert errs == ["model uses graph layers but carries no graph"]
    assert bg.validate_model([]) == ["model has no layers"]
    errs = bg.validate_model([bg.LayerSpec(K.LAYER_GCN, ["MM.FBB"], W)])
    assert errs == ["layer 0 gcn_conv: expected 2 plan slots, got 1"]
    errs = bg.validate_model([bg.LayerSpec(K.LAYER_GCN, ["BSpMM.FBB", "BSpMM.BBF"])])
    assert "layer 0 gcn_conv mm: expected a MM variant, got BSpMM.FBB" in errs
    assert "layer 0 gcn_conv: missing weights" in errs
    errs = bg.validate_model([bg.LayerSpec(K.LAYER_FC, ["MM.FBB"], W)])
    assert errs == ["model output must be full precision, got a binary tail"]
    errs = bg.validate_model([bg.LayerSpec(K.LAYER_SAGE, ["MM.FBB", "MM.FBF", "BSpMM.BBB", "ADD.BBF"], W, W)])
    assert "layer 0 sage_conv: mm_neigh output tag does not feed the spmm input" in errs
    errs = bg.validate_model([bg.LayerSpec(K.LAYER_SOFTMAX)], input_precision=bg.B)
    assert errs[0] == "layer 0 softmax: expects a full-precision input"
    errs = bg.validate_model([bg.LayerSpec(K.LAYER_BATCHNORM)])
    assert "layer 0 batchnorm: missing parameters" in errs
    errs = bg.validate_model([bg.LayerSpec(K.LAYER_FC, ["MM.FFF"], W), bg.LayerSpec(K.LAYER_SCALE)])
    assert errs == ["layer 1 scale: missing factors"]


def test_product_rng_matches_oracle_and_reference_fixtures():
    # the product's own generator (std::mt19937_64 in the C++ host code)
    a = bg.Rng(100).random_edges(2708, 13264, False)
    b = po.Rng(100).random_edges(2708, 13264, False)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    layers, X = bg.build_model_spec("saint", 33, 16, 5, 99, 120)
    ol, oX = po.build_model("saint", 33, 16, 5, 99, 120)
    assert np.array_equal(X, oX)
    for l, m in zip(layers, ol):
        for w in ("w1", "w2"):
            x, y = getattr(l, w), getattr(m, w)
            assert (x is None and y is None) or np.array_equal(x, y)
    fx = json.load(open(os.path.join(ROOT, "tests", "golden", "reference_fixtures.json")))["cases"][0]
    s, d = bg.Rng(fx["graph_seed"]).random_edges(fx["nodes"], fx["edge_draws"], False)
    assert hashlib.sha256(s.tobytes()).hexdigest() == fx["sha_src"]
    assert hashlib.sha256(d.tobytes()).hexdigest() == fx["sha_dst"]


def test_operand_validation_is_host_side():
    # argument errors surface before any device work (no GPU needed)
    with pytest.raises(bg.InvalidArgument):
        bg.BitDenseMatrix.empty(2, 2, word_bits=48)
    buf = ctypes.create_string_buffer(8)
    assert L.lib().bg_variant_name(L.Variant(0, 0, 1, 1), buf, 8) == 0 and buf.value == b"BMM.FBB"


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="checks the no-GPU behaviour")
def test_device_work_fails_loudly_without_a_gpu():
    # no CPU fallback anywhere: device entry points report a CUDA error and
    # host tensors are rejected instead of being computed on the host
    import numpy as np
    import torch
    src = np.array([0, 1], np.int64)
    dst = np.array([1, 2], np.int64)
    g = ctypes.c_void_p()
    rc = L.lib().bg_prepare_graph(src.ctypes.data, dst.ctypes.data, 2, 4, ctypes.byref(g), None)
    assert rc == L.BG_CUDA_ERROR
    assert L.lib().bg_last_error()
    with pytest.raises(bg.InvalidArgument, match="CUDA tensors"):
        bg.binarize(torch.zeros(2, 3))
