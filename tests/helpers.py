"""Shared helpers for the parity tests: build inputs with the oracle's rng and
compare the CUDA path (through the C ABI) with the oracle / reference."""
from __future__ import annotations

import numpy as np

import pyoracle as po


def bits_equal(a: np.ndarray, b: np.ndarray) -> bool:
    return a.shape == b.shape and np.array_equal(a.view(np.uint32), b.view(np.uint32))


def to_layer_specs(bgmod, layers):
    """oracle Layer list -> product LayerSpec list (same weights)."""
    kinds = {po.GCN: bgmod._lib.LAYER_GCN, po.SAGE: bgmod._lib.LAYER_SAGE,
             po.GRAPHCONV: bgmod._lib.LAYER_GRAPHCONV, po.FC: bgmod._lib.LAYER_FC,
             po.SOFTMAX: bgmod._lib.LAYER_SOFTMAX}
    return [bgmod.LayerSpec(kinds[l.kind], list(l.plan), l.w1, l.w2, l.relu) for l in layers]


def rel_err(got: np.ndarray, want: np.ndarray) -> float:
    """max |e - o| / max(1, |o|)  (ref: runreport.cpp:108-120)."""
    if want.size == 0:
        return 0.0
    return float(np.max(np.abs(got.astype(np.float64) - want.astype(np.float64)) /
                        np.maximum(1.0, np.abs(want.astype(np.float64)))))


def argmax_agreement(got: np.ndarray, want: np.ndarray) -> float:
    """Engine class agrees when the reference value there is the row max
    (ref: runreport.cpp:121-131, exact-tie rule)."""
    if got.shape[0] == 0:
        return 1.0
    pick = np.argmax(got, axis=1)
    return float(np.mean(want[np.arange(want.shape[0]), pick] == want.max(axis=1)))
