"""Variant substitution on the GPU (ref: tune.hpp, tune.cpp:100-178).

`legal_variants` / `enumerate_plans` restate the reference's enumeration: every
tag-consistent chain of kernel variants per layer kind, first input F, final
output F.  `tune_model` builds one model per candidate plan on the same seeded
weights (build_model order, modelconfig.cpp:99-173), times every candidate
with CUDA events on the device (the CUDA-graph forward, like `bench.py`), and
keeps the fastest one that passes verification.

Verification is the caller's: the reference checks each candidate against its
dense simulated-binarization oracle (runreport.cpp:51-135).  That oracle is
test infrastructure here and never part of the product path, so `tune_model`
takes a `verify(plan, logits) -> (passed, max_rel_error)` callback; the tests
pass one backed by `oracle/`, a deployment passes its own (or none: every
candidate counts as verified, as with `verified = -1` in `BenchReport`).
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence, Tuple

import torch

from . import _lib as L
from ._lib import RuntimeFailure
from .bitgnn import KernelVariant, Model, build_model_spec, prepare_graph

TAGS = (L.F, L.B)


def legal_variants(op: int, in1: Optional[int] = None, in2: Optional[int] = None,
                   out: Optional[int] = None) -> List[KernelVariant]:
    """Every valid variant of `op` matching the fixed tags (None = free)
    (ref: legal_variants, tune.cpp:100-117; validity from KernelVariant::valid)."""
    found = []
    for a, b, c in itertools.product(TAGS, TAGS, TAGS):
        if (in1 is not None and a != in1) or (in2 is not None and b != in2) or (out is not None and c != out):
            continue
        v = KernelVariant(op, a, b, c)
        if v.valid():
            found.append(v)
    return found


def _layer_choices(kind: str, tag_in: int) -> List[Tuple[List[KernelVariant], int]]:
    """Per-layer chains and their output tag (ref: layer_choices, tune.cpp:27-70)."""
    if kind == "gcn":
        return [([mm, sp], sp.out) for mm in legal_variants(L.BMM, tag_in)
                for sp in legal_variants(L.BSPMM, mm.out)]
    if kind in ("sage", "graphconv"):
        return [([ms, mn, sp, ad], ad.out)
                for ms in legal_variants(L.BMM, tag_in) for mn in legal_variants(L.BMM, tag_in)
                for sp in legal_variants(L.BSPMM, mn.out) for ad in legal_variants(L.ADD, ms.out, sp.out)]
    if kind == "fc":
        return [([mm], mm.out) for mm in legal_variants(L.BMM, tag_in)]
    if kind == "aggregate":
        return [([sp], sp.out) for sp in legal_variants(L.BSPMM, tag_in)]
    raise RuntimeFailure("tune: layer kind carries no kernel slots")


def enumerate_plans(kinds: Sequence[str], tag_in: int = L.F) -> List[List[str]]:
    """Every tag-consistent plan whose last output is F, as '+'-joined chains
    per layer (ref: enumerate_plans, tune.cpp:119-125)."""
    plans: List[List[str]] = []

    def rec(at: int, tag: int, acc: List[str]):
        if at == len(kinds):
            if tag == L.F:
                plans.append(list(acc))
            return
        for chain, out in _layer_choices(kinds[at], tag):
            acc.append("+".join(v.name() for v in chain))
            rec(at + 1, out, acc)
            acc.pop()

    rec(0, tag_in, [])
    return plans


def skeleton(model: str, layers: int) -> List[str]:
    """ref: skeleton_of, tune.cpp:84-96."""
    if model == "gcn":
        return ["gcn"] * layers
    if model == "sage":
        return ["sage"] * layers
    return ["graphconv"] * (layers - 1) + ["fc"]


@dataclass
class TuneCandidate:
    plan: List[str]
    verified: bool = False
    median_ms: float = 0.0
    max_rel_logit_error: float = 0.0


@dataclass
class TuneResult:
    best: Optional[TuneCandidate] = None
    candidates: int = 0
    evaluated: List[TuneCandidate] = field(default_factory=list)


def _time_forward(model: Model, x: torch.Tensor, reps: int) -> float:
    for _ in range(2):  # first call eager, second captures the CUDA graph
        model.forward(x)
    stream = torch.cuda.current_stream()
    times = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        model.forward(x)
        b.record(stream)
        b.synchronize()
        times.append(a.elapsed_time(b))
    times.sort()
    return times[len(times) // 2]


def tune_model(model: str, nodes: int, src, dst, features: int, hidden: int, classes: int,
               seed: int = 99, layers: int = 2, plans: Optional[Sequence[Sequence[str]]] = None,
               reps: int = 5, verify: Optional[Callable[[List[str], torch.Tensor], Tuple[bool, float]]] = None
               ) -> TuneResult:
    """ref: tune_model, tune.cpp:127-178.  `plans` restricts the search (an
    explicit config plan); otherwise every plan of the model skeleton."""
    chains = [list(p) for p in plans] if plans else enumerate_plans(skeleton(model, layers), L.F)
    graph = prepare_graph(nodes, src, dst)
    result = TuneResult()
    for plan in chains:
        specs, X = build_model_spec(model, features, hidden, classes, seed, nodes, plan)
        m = Model(specs, graph)
        x = torch.from_numpy(X).cuda()
        out, logits, _ = m.forward_traced(x)
        cand = TuneCandidate(plan=plan)
        if verify is None:
            cand.verified = True
        else:
            cand.verified, cand.max_rel_logit_error = verify(plan, logits)
        if cand.verified:
            cand.median_ms = _time_forward(m, x, reps)
            if result.best is None or cand.median_ms < result.best.median_ms:
                result.best = cand
        result.evaluated.append(cand)
    result.candidates = len(result.evaluated)
    if result.best is None:
        raise RuntimeFailure("tune: no candidate passed verification")
    return result
