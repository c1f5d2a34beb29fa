"""CPU oracle of the layer-sensitivity sweep (TEST INFRASTRUCTURE ONLY).

Restates, on top of ``pillars_oracle.forward``, the paper's mixed-precision search
 as SPEC.md pins it -- the reference package never implemented
its ``sensitivity`` module:

* sweep: one layer at a time INT8 on the FP32 base, every other
  layer FP32; the score of a plan is the head-output error against the FP32 forward
  on the same samples, rel_err = sqrt(sum (y - y_fp32)^2 / sum y_fp32^2) over all
  heads and samples, summed in f64 (the engine's sweep uses the same score);
* select_topk: most sensitive (largest error) first, ties to the
  lower layer index;
* greedy_candidates: FP16 on the first i ranked layers, INT8
  elsewhere, i = 1..k;
* exhaustive_search: every k-subset in FP16 on the INT8 base, the
  best (lowest error) subset, ties to the lexicographically first subset, refused
  above 10^4 subsets.

Only ``tests/`` import this module.
"""

from __future__ import annotations

import itertools
import math

import numpy as np

from . import pillars_oracle as O

GUARD = 10_000


def _precisions(graph, default, overrides):
    return {l.index: overrides.get(l.index, default) for l in graph.layers if l.weight is not None}


def heads_of(graph, sample, stats, precisions, acc=np.float32):
    with O.accumulate_in(acc):
        out = O.forward(O.folded_graph(graph, precisions), sample, stats=stats)
    return out if isinstance(out, tuple) else (out,)


def plan_sq_sums(graph, samples, stats, precisions, refs, acc=np.float32):
    """(sum (y - y_ref)^2, sum y_ref^2) in f64 over all heads and samples."""
    e = r = 0.0
    for sample, ref in zip(samples, refs):
        for y, y0 in zip(heads_of(graph, sample, stats, precisions, acc), ref):
            d = np.asarray(y, np.float64) - np.asarray(y0, np.float64)
            e += float(np.sum(d * d))
            r += float(np.sum(np.asarray(y0, np.float64) ** 2))
    return e, r


def rel_err(pair) -> float:
    e, r = pair
    return math.sqrt(e / r) if r > 0 else math.inf


def fp32_refs(graph, samples):
    fp32 = _precisions(graph, "fp32", {})
    return [heads_of(graph, s, None, fp32) for s in samples]


def sweep(graph, samples, stats, acc=np.float32) -> dict[int, float]:
    """{layer index: error of the plan with only that layer INT8}."""
    refs = fp32_refs(graph, samples)
    layers = [l.index for l in graph.layers if l.weight is not None]
    return {i: rel_err(plan_sq_sums(graph, samples, stats, _precisions(graph, "fp32", {i: "int8"}), refs, acc))
            for i in layers}


def select_topk(errors: dict[int, float], k: int) -> list[int]:
    """SPEC.md:373-380."""
    if not 1 <= k <= len(errors):
        raise ValueError(f"k={k} out of range [1, {len(errors)}]")
    return [i for i, _ in sorted(errors.items(), key=lambda kv: (-kv[1], kv[0]))][:k]


def greedy_candidates(ranking, k) -> list[tuple[int, ...]]:
    """FP16 sets of the greedy plans."""
    return [tuple(ranking[:j]) for j in range(1, k + 1)]


def exhaustive_search(graph, samples, stats, k, layers=None, acc=np.float32):
    """best FP16 k-subset on the INT8 base -> (subset, error, all errors)."""
    layers = sorted(layers if layers is not None else [l.index for l in graph.layers if l.weight is not None])
    n = math.comb(len(layers), k)
    if n > GUARD:
        raise ValueError(f"exhaustive search over C({len(layers)}, {k}) = {n} subsets exceeds the guard {GUARD}")
    refs = fp32_refs(graph, samples)
    errs = {}
    for sub in itertools.combinations(layers, k):
        precs = _precisions(graph, "int8", {i: "fp16" for i in sub})
        errs[sub] = rel_err(plan_sq_sums(graph, samples, stats, precs, refs, acc))
    best = min(errs, key=lambda sub: (errs[sub], sub))
    return best, errs[best], errs
