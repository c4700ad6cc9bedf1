"""Critical-layer calibration on the GPU (reference bench.py:118-144).

`calibrate_layer` picks the probing layer whose anchor-probe Top-N tracks the
full-probe Top-N best over candidate layers 2..L-1 (ties toward the middle
layer), exactly as the reference's `calibrate_layer` does, but takes explicit
chunk lists instead of running the reference's byte-4-gram retrieval
(`cases.retrieve`, outside the fused path). Every probe, score and Top-N runs on
the device kernels; only the per-layer overlap means are host scalars.
"""

from __future__ import annotations

import math

import numpy as np

from .fusion import PROBE_ANCHORS, PROBE_FULL, FusionEngine, top_n_positions
from .metrics import selection_overlap


def layer_overlaps(engine: FusionEngine, chunk_ids, query_tokens, ratio: float,
                   candidates=None, against_oracle: bool = False) -> dict[int, float]:
    """Per candidate layer: overlap of the anchor-probe Top-N with the
    full-probe Top-N (bench.py:129-136), or with the Top-N of the exact
    full-forward importance when `against_oracle` (fusion.py:331-346)."""
    cfg = engine.config
    candidates = list(range(2, cfg.n_layers)) if candidates is None else list(candidates)
    fused = engine.assemble_context(chunk_ids)
    n = int(math.ceil(ratio * fused.n_ctx))
    anchor = engine.probe_query(query_tokens, fused, PROBE_ANCHORS, layers=max(candidates))
    full = None if against_oracle else engine.probe_query(query_tokens, fused, PROBE_FULL,
                                                          layers=max(candidates))
    out = {}
    for layer in candidates:
        a = top_n_positions(engine.score_against_keys(anchor, fused, layer), n)
        if against_oracle:
            b = top_n_positions(engine.importance_at(fused.token_ids, query_tokens, layer), n)
        else:
            b = top_n_positions(engine.score_against_keys(full, fused, layer), n)
        out[layer] = selection_overlap(a, b)
    return out


def calibrate_layer(engine: FusionEngine, chunk_lists, queries, ratio: float = 0.2) -> dict:
    """bench.py:118-144 over explicit (chunk_ids, query) pairs."""
    cfg = engine.config
    candidates = list(range(2, cfg.n_layers))
    overlaps: dict[int, list[float]] = {layer: [] for layer in candidates}
    for chunk_ids, query in zip(chunk_lists, queries):
        qt = list(query.encode("utf-8")) if isinstance(query, str) else list(query)
        for layer, ov in layer_overlaps(engine, chunk_ids, qt, ratio, candidates).items():
            overlaps[layer].append(ov)
    means = {layer: float(np.mean(v)) for layer, v in overlaps.items()}
    middle = int(math.ceil(cfg.n_layers / 2))
    best = max(means.values())
    tied = [layer for layer, m in means.items() if abs(m - best) < 1e-12]
    recommended = min(tied, key=lambda layer: (abs(layer - middle), layer))
    return {"recommended": recommended, "mean_overlap": means}
