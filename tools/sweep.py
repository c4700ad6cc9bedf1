"""BASELINE configs[3] / configs[4] sweeps on one B200 (JSON lines to stdout).

  python tools/sweep.py ratio     # configs[4]: recompute ratio 5..50% vs full prefill / full reuse
                                  #   (Llama-3-8B shape, 10x512, q32; --config llama3-8b-gqa for GQA-8)
  python tools/sweep.py critical  # configs[3]: critical-layer sweep, Mistral-7B shape (GQA-8),
                                  #   64x512 = 32k context, r .15

Per point: device TTFT (CUDA-graph replay, CUDA events, median of --steps after
--warmup), and selection/logit fidelity against the exact full computation on
the same GPU (FullCompute logits; Top-N of the full-forward importance at the
probing layer, fusion.py:331-346), plus the reference calibrate_layer metric
(anchor-probe vs full-probe Top-N overlap, bench.py:118-144) for the layer sweep.
"""

from __future__ import annotations

import argparse
import dataclasses
import json
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
import paper_2604_08585_b200 as Q  # noqa: E402
from paper_2604_08585_b200.calibrate import layer_overlaps  # noqa: E402
from paper_2604_08585_b200.fusion import top_n_positions  # noqa: E402
from paper_2604_08585_b200.metrics import selection_overlap  # noqa: E402


def ttft(eng, policy, ratio, ids, query, steps, warmup):
    plan, b = eng.prefill(policy, ratio, ids, query)
    s = torch.cuda.current_stream()
    for _ in range(warmup):
        b.graph.replay()
    times = []
    for _ in range(steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        b.graph.replay()
        e1.record(s)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    logits = b.logits[0].cpu().numpy().copy()
    sel = b.rc_pos[:plan.n_sel].cpu().numpy().astype(np.int64).copy()
    b.graph = None
    eng._bufs.clear()
    return statistics.median(times), logits, sel


def fidelity(logits, full_logits):
    rel = float(np.abs(logits - full_logits).max() / np.abs(full_logits).max())
    return {"logit_rel_err_vs_full": rel, "top1_agrees_with_full": bool(np.argmax(logits) == np.argmax(full_logits))}


def sweep_ratio(args):
    cfgd = dict(bench.CONFIGS[args.config])
    Qm, cfg, w, store, eng, ids, toks = bench.build_engine(cfgd, "bf16", torch.device("cuda"), cfgd["n_chunks"])
    query = np.random.default_rng(10_000).integers(0, 256, cfgd["q"]).tolist()
    full_ms, full_logits, _ = ttft(eng, "FullCompute", 1.0, ids, query, args.steps, args.warmup)
    reuse_ms, reuse_logits, _ = ttft(eng, "FullReuse", 0.0, ids, query, args.steps, args.warmup)
    fused = eng.assemble_context(ids)
    imp = eng.oracle_importance(fused.token_ids, query)
    print(json.dumps({"config": args.config, "policy": "FullCompute", "ttft_ms": full_ms}), flush=True)
    print(json.dumps({"config": args.config, "policy": "FullReuse", "ttft_ms": reuse_ms,
                      "fused_over_full": reuse_ms / full_ms, **fidelity(reuse_logits, full_logits)}), flush=True)
    for r in [0.05, 0.10, 0.15, 0.20, 0.25, 0.30, 0.35, 0.40, 0.45, 0.50]:
        ms, logits, sel = ttft(eng, "QCFuse", r, ids, query, args.steps, args.warmup)
        ov = selection_overlap(sel, top_n_positions(imp, sel.size))
        print(json.dumps({"config": args.config, "policy": "QCFuse", "ratio": r, "n_selected": int(sel.size),
                          "ttft_ms": ms, "fused_over_full": ms / full_ms, "overlap_vs_full_importance": ov,
                          **fidelity(logits, full_logits)}), flush=True)


def sweep_critical(args):
    cfgd = dict(bench.CONFIGS[args.config])
    dev = torch.device("cuda")
    base = Q.ModelConfig(n_layers=cfgd["n_layers"], n_heads=cfgd["n_heads"], d_model=cfgd["d_model"],
                         d_head=cfgd["d_head"], d_ff=cfgd["d_ff"], seed=1234, n_kv_heads=cfgd.get("n_kv_heads"))
    w0 = Q.init_weights(base, dtype="bf16", device=dev)
    toks = [np.random.default_rng(i).integers(0, 256, cfgd["chunk_len"]) for i in range(cfgd["n_chunks"])]
    query = np.random.default_rng(10_000).integers(0, 256, cfgd["q"]).tolist()
    full_ms = full_logits = None
    for c in args.layers:
        cfg = dataclasses.replace(base, critical_layer=c)
        w = dataclasses.replace(w0, config=cfg)
        store = Q.ChunkStore(f"/tmp/qcf-sweep-{c}", cfg, dtype="bf16", device=dev, persist=False)
        ids = [store.precompute(w, t, 0.05, f"chunk{i}").chunk_id for i, t in enumerate(toks)]
        eng = Q.FusionEngine(w, store)
        if full_ms is None:
            full_ms, full_logits, _ = ttft(eng, "FullCompute", 1.0, ids, query, max(3, args.steps // 4), 2)
            print(json.dumps({"config": args.config, "policy": "FullCompute", "ttft_ms": full_ms}), flush=True)
        ms, logits, sel = ttft(eng, "QCFuse", cfgd["ratio"], ids, query, args.steps, args.warmup)
        fused = eng.assemble_context(ids)
        imp = eng.importance_at(fused.token_ids, query, c)
        ov_imp = selection_overlap(sel, top_n_positions(imp, sel.size))
        ov_cal = layer_overlaps(eng, ids, query, cfgd["ratio"], candidates=[c])[c]
        print(json.dumps({"config": args.config, "critical_layer": c, "n_ctx": fused.n_ctx,
                          "n_selected": int(sel.size), "ttft_ms": ms, "fused_over_full": ms / full_ms,
                          "overlap_vs_full_importance": ov_imp, "calibrate_overlap_anchor_vs_full_probe": ov_cal,
                          **fidelity(logits, full_logits)}), flush=True)
        del eng, store, fused, w
        torch.cuda.empty_cache()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["ratio", "critical"])
    ap.add_argument("--config", default=None)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--layers", type=int, nargs="*", default=[2, 4, 8, 12, 16, 20, 24, 28, 31])
    args = ap.parse_args()
    if args.config is None:
        args.config = "llama3-8b" if args.mode == "ratio" else "mistral-7b-32k"
    (sweep_ratio if args.mode == "ratio" else sweep_critical)(args)


if __name__ == "__main__":
    main()
