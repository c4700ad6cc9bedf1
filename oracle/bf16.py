"""CPU ORACLE — test infrastructure only, never the product path.

The bf16 noise floor of the fused path (SURVEY.md §8c "parity criteria" (2)):
the reference algorithm (`qcfuse_oracle`) run on bf16-rounded weights and
bf16-rounded chunk KV, against the same algorithm in float32. Its error is the
part of any bf16 engine's deviation that storage precision alone forces; the
stated tolerance of the B200 bf16 path is a multiple of it.

Everything else in these runs is the float32 reference arithmetic
(`fusion.py:234-263` assembly, `446-490` recompute, `536-540` query forward).
To separate selection from arithmetic, the fused KV and logits are compared
for a GIVEN selection (`conditional_run`): the engine's selection is fed to
the reference recompute, so a differing pick does not masquerade as KV error.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import qcfuse_oracle as O


def bf16_round(a) -> np.ndarray:
    """Round-to-nearest-even to bfloat16, returned as float32 (torch's cast)."""
    a = np.ascontiguousarray(np.asarray(a, np.float32))
    u = a.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    out = r.view(np.float32).copy()
    nan = np.isnan(a)
    out[nan] = a[nan]
    return out


def rounded_weights(w: O.Weights) -> O.Weights:
    """Projection matrices rounded to bf16; embedding and LayerNorm parameters
    stay float32 (the B200 engine keeps them float32: model.py weights layout)."""
    layers = [O.Layer(bf16_round(l.wq), bf16_round(l.wk), bf16_round(l.wv), bf16_round(l.wo),
                      bf16_round(l.w1), bf16_round(l.w2), l.ln1_g, l.ln1_b, l.ln2_g, l.ln2_b)
              for l in w.layers]
    return O.Weights(w.cfg, w.emb, layers, w.lnf_g, w.lnf_b)


def rounded_chunks(chunks: list[O.Chunk]) -> list[O.Chunk]:
    return [O.Chunk(c.tokens, [O.KV(bf16_round(kv.keys), bf16_round(kv.values), kv.positions) for kv in c.kv],
                    c.key_norms, c.anchors) for c in chunks]


@dataclass
class CondOut:
    keys: list[np.ndarray]      # per layer [1 + n_ctx, Hkv, D] updated fused K
    values: list[np.ndarray]
    logits: np.ndarray          # [V] first-token logits


def conditional_run(w: O.Weights, chunks: list[O.Chunk], query, sel) -> CondOut:
    """assemble -> recompute(sel) -> query forward (fusion.py:519-540 with the
    selection given instead of probed)."""
    fused = O.assemble(w, chunks)
    upd = O.recompute(w, fused, np.asarray(sel, np.int64))
    qt = O.query_forward(w, upd, query)
    return CondOut(upd.keys, upd.values, qt.logits[-1])


def rel_l2(a, b) -> float:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    den = float(np.linalg.norm(b))
    return float(np.linalg.norm(a - b)) / den if den > 0 else float(np.linalg.norm(a - b))


def compare(test: CondOut, ref: CondOut, sel) -> dict:
    """Per-layer relative L2 of the fused K and V (all rows, and the selected
    rows alone), first-logit relative L2 and max-abs, top-1 agreement."""
    sel = np.asarray(sel, np.int64)
    out = {"k_all": [], "v_all": [], "k_sel": [], "v_sel": []}
    for tk, tv, rk, rv in zip(test.keys, test.values, ref.keys, ref.values):
        out["k_all"].append(rel_l2(tk, rk))
        out["v_all"].append(rel_l2(tv, rv))
        if sel.size:
            out["k_sel"].append(rel_l2(tk[sel], rk[sel]))
            out["v_sel"].append(rel_l2(tv[sel], rv[sel]))
    out["logits_rel_l2"] = rel_l2(test.logits, ref.logits)
    out["logits_max_abs"] = float(np.abs(np.asarray(test.logits, np.float64) - ref.logits).max())
    out["top1_equal"] = bool(int(np.argmax(test.logits)) == int(np.argmax(ref.logits)))
    return out


def floor(w: O.Weights, chunks: list[O.Chunk], query, sel, ref: CondOut | None = None) -> dict:
    """The bf16 noise floor for one request and selection (`ref`: the float32
    conditional run for `sel`, when already computed)."""
    ref = ref or conditional_run(w, chunks, query, sel)
    low = conditional_run(rounded_weights(w), rounded_chunks(chunks), query, sel)
    return compare(low, ref, sel)


def floor_probe(w: O.Weights, chunks: list[O.Chunk], query, ratio: float) -> dict:
    """Probe + scoring + Top-N of the reference on bf16-rounded inputs vs
    float32 (fusion.py:269-326, 148-158): critical-layer score relative L2 and
    selection overlap -- what a bf16 probe can be expected to reach -- plus the
    float32 run itself (`ref`: selection, scores, first logits)."""
    ref = O.run(w, chunks, query, ratio)
    low = O.run(rounded_weights(w), rounded_chunks(chunks), query, ratio)
    n = max(ref.selection.size, 1)
    return {"overlap": len(np.intersect1d(ref.selection, low.selection)) / n,
            "scores_rel_l2": rel_l2(low.scores, ref.scores), "ref": ref}


def overlap(a, b) -> float:
    a, b = np.asarray(a), np.asarray(b)
    return len(np.intersect1d(a, b)) / max(b.size, 1)


def cutoff_margin(scores, sel) -> float:
    """Relative gap between the smallest selected and the largest unselected
    score (how far the selection is from a tie at the cut)."""
    s = np.asarray(scores, np.float64)
    mask = np.zeros(s.size, bool)
    mask[np.asarray(sel, np.int64) - 1] = True
    if mask.all() or not mask.any():
        return float("inf")
    lo, hi = s[mask].min(), s[~mask].max()
    return float((lo - hi) / max(abs(lo), 1e-30))


TOLERANCE_FACTOR = 2.0   # bf16 engine error <= 2x the bf16 noise floor


def check_against_floor(gpu: dict, fl: dict, factor: float = TOLERANCE_FACTOR, atol: float = 1e-7) -> list[str]:
    """Violations of the stated tolerance (empty list = pass)."""
    bad = []
    for key in ("k_all", "v_all", "k_sel", "v_sel"):
        for li, (g, f) in enumerate(zip(gpu[key], fl[key])):
            if g > factor * f + atol:
                bad.append(f"{key}[layer {li + 1}] {g:.3e} > {factor} x floor {f:.3e}")
    if gpu["logits_rel_l2"] > factor * fl["logits_rel_l2"] + atol:
        bad.append(f"logits rel L2 {gpu['logits_rel_l2']:.3e} > {factor} x floor {fl['logits_rel_l2']:.3e}")
    if not gpu["top1_equal"]:
        bad.append("top-1 token differs from the float32 reference")
    return bad
