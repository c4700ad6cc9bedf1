"""bf16 parity at full depth: BASELINE configs[1] (Llama-3-8B shape, L32 H32
D128 d4096 F14336, 10x512 chunks, q32, r .15, c 16) against the CPU oracle on
the same inputs, with the tolerance of BASELINE.md §5 (run as
`python bench.py --parity`, or directly). One request (oracle time dominates:
~1-3 min of host BLAS).

Inputs shared by both sides:
* weights: drawn on the GPU by `qcf_init_uniform` in float32 and copied to the
  host for the oracle. That kernel is bit-exact to the oracle's splitmix64
  restatement (tests/test_gpu_kernels.py::test_init_*); here 4096 random
  entries of every tensor are re-drawn with `O.draw_uniform_f32` and compared
  before anything else runs (drawing all 7.5e9 in numpy takes ~5 min);
* chunk KV: the GPU float32 precompute (the .qcfk parity bridge),
  anchors/norms recomputed by the oracle from it.

Checks (same as tests/test_gpu_bf16_parity.py at L=4): fused KV per layer,
logits and scores <= 2 x the bf16 noise floor (the oracle on bf16-rounded
weights and chunk KV), top-1 equal, selection overlap >= floor overlap - 0.02;
fp32 scoring mode selection bit-exact. Writes one JSON object (stdout, and
--out)."""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle import bf16 as B  # noqa: E402
from oracle import qcfuse_oracle as O  # noqa: E402


def host_weights(w32, oc: O.Config) -> O.Weights:
    d, kvd = oc.d_model, oc.n_kv_heads * oc.d_head
    layers = []
    for dl in w32.layers:
        wqkv = dl.wqkv.cpu().numpy().T          # [d][d + 2 kvd]
        one, zero = np.ones(d, np.float32), np.zeros(d, np.float32)
        layers.append(O.Layer(np.ascontiguousarray(wqkv[:, :d]), np.ascontiguousarray(wqkv[:, d:d + kvd]),
                              np.ascontiguousarray(wqkv[:, d + kvd:]), np.ascontiguousarray(dl.wo.cpu().numpy().T),
                              np.ascontiguousarray(dl.w1.cpu().numpy().T), np.ascontiguousarray(dl.w2.cpu().numpy().T),
                              one, zero, one.copy(), zero.copy()))
    return O.Weights(oc, w32.emb.cpu().numpy(), layers, np.ones(d, np.float32), np.zeros(d, np.float32))


def verify_sampled(ow: O.Weights, oc: O.Config, n: int = 4096) -> int:
    """Re-draw n random entries of every tensor with the oracle's stream."""
    rng = np.random.default_rng(0)
    mats = [ow.emb] + [m for l in ow.layers for m in (l.wq, l.wk, l.wv, l.wo, l.w1, l.w2)]
    off, checked = 0, 0
    for m in mats:
        r, c = m.shape
        idx = rng.integers(0, r * c, n).astype(np.uint64)
        u = O.u64_to_unit(O.splitmix64_at(oc.seed, np.uint64(off) + idx))
        want = (O.W_LO + u * (O.W_HI - O.W_LO)).astype(np.float32)
        got = m.reshape(-1)[idx]
        if not np.array_equal(got, want):
            raise AssertionError("GPU-drawn weights differ from the oracle stream")
        off += r * c
        checked += n
    return checked


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import paper_2604_08585_b200 as Q
    t0 = time.time()
    oc = O.Config(n_layers=args.layers, n_heads=32, d_model=4096, d_head=128, d_ff=14336)
    cfg = Q.ModelConfig(n_layers=args.layers, n_heads=32, d_model=4096, d_head=128, d_ff=14336)
    w32 = Q.init_weights(cfg, dtype="f32")
    ow = host_weights(w32, oc)
    n_checked = verify_sampled(ow, oc)
    ex = Q.fusion._executor_for(w32)
    chunks = []
    for i in range(10):
        toks = np.random.default_rng(i).integers(0, 256, 512)
        tk, tv, _ = ex.forward_full(torch.as_tensor(toks.astype(np.int32), device="cuda"), 0)
        keys, vals = tk.cpu().numpy(), tv.cpu().numpy()
        del tk, tv
        norms = np.linalg.norm(keys[oc.critical_layer - 1], axis=2).mean(axis=1).astype(np.float32)
        chunks.append(O.Chunk(toks, [O.KV(keys[li], vals[li], np.arange(512)) for li in range(oc.n_layers)],
                              norms, O.extract_anchors(norms, 0.05)))
    del ex
    Q.fusion._EXECUTORS.pop(w32, None)
    del w32
    torch.cuda.empty_cache()
    t_inputs = time.time() - t0
    query = np.random.default_rng(10_000).integers(0, 256, 32)

    w = Q.init_weights(cfg, dtype="bf16", scoring="fp32")
    res = {}
    with __import__("tempfile").TemporaryDirectory() as td:
        for mode in ("native", "fp32"):
            store = Q.ChunkStore(Path(td) / mode, cfg, dtype="bf16", persist=False, scoring=mode)
            ids = [store.add_record(c.tokens, torch.as_tensor(np.stack([x.keys for x in c.kv])).cuda(),
                                    torch.as_tensor(np.stack([x.values for x in c.kv])).cuda(),
                                    c.key_norms, c.anchors).chunk_id for c in chunks]
            plan, b = Q.FusionEngine(w, store).prefill("QCFuse", 0.15, ids, query.tolist(), use_graph=False)
            torch.cuda.synchronize()
            n = plan.n_ctx
            res[mode] = (b.rc_pos[:plan.n_sel].cpu().numpy().astype(np.int64), b.scores[:n].cpu().numpy().copy(),
                         B.CondOut([b.fk[li, :n + 1].float().cpu().numpy() for li in range(oc.n_layers)],
                                   [b.fv[li, :n + 1].float().cpu().numpy() for li in range(oc.n_layers)],
                                   b.logits[0].cpu().numpy().copy()))
            del b, store
            torch.cuda.empty_cache()
    t_gpu = time.time() - t0 - t_inputs

    fp = B.floor_probe(ow, chunks, query, 0.15)
    ref = fp["ref"]
    sel, scores, got = res["native"]
    if np.array_equal(sel, ref.selection):
        ref_c = B.CondOut(ref.updated.keys, ref.updated.values, ref.first_logits)
    else:
        ref_c = B.conditional_run(ow, chunks, query, sel)
    fl = B.floor(ow, chunks, query, sel, ref_c)
    cmp = B.compare(got, ref_c, sel)
    bad = B.check_against_floor(cmp, fl)
    ov = B.overlap(sel, ref.selection)
    s_err = B.rel_l2(scores, ref.scores)
    if s_err > B.TOLERANCE_FACTOR * fp["scores_rel_l2"] + 1e-7:
        bad.append("scores rel L2 above 2x floor")
    if ov < fp["overlap"] - 0.02:
        bad.append("selection overlap below floor - 0.02")
    if int(np.argmax(got.logits)) != int(np.argmax(ref.first_logits)):
        bad.append("top-1 differs")
    sel32, scores32, _ = res["fp32"]
    out = {
        "config": f"configs[1] Llama-3-8B shape L{oc.n_layers} H32 D128 d4096 F14336, 10x512, q32, r .15, c {oc.critical_layer}",
        "weights_sample_checked": n_checked,
        "bf16": {"pass": not bad, "violations": bad, "overlap": ov, "floor_overlap": fp["overlap"],
                 "scores_rel_l2": s_err, "floor_scores_rel_l2": fp["scores_rel_l2"],
                 "ratio_max": max(g / f for k in ("k_all", "v_all", "k_sel", "v_sel") for g, f in zip(cmp[k], fl[k])),
                 "logits_rel_l2": cmp["logits_rel_l2"], "floor_logits_rel_l2": fl["logits_rel_l2"],
                 "top1_equal": int(np.argmax(got.logits)) == int(np.argmax(ref.first_logits)),
                 "gpu": cmp, "floor": fl},
        "fp32_scoring": {"bit_exact": bool(np.array_equal(sel32, ref.selection)), "n_sel": int(sel32.size),
                         "cutoff_margin_rel": B.cutoff_margin(ref.scores, ref.selection),
                         "max_score_err_rel": float(np.abs(scores32.astype(np.float64) - ref.scores).max()
                                                    / np.abs(ref.scores).max())},
        "seconds": {"inputs": t_inputs, "gpu": t_gpu, "oracle": time.time() - t0 - t_inputs - t_gpu},
    }
    line = json.dumps(out)
    print(line)
    if args.out:
        Path(args.out).write_text(json.dumps(out, indent=1) + "\n")
    if bad or not out["fp32_scoring"]["bit_exact"]:
        sys.exit(1)


if __name__ == "__main__":
    main()
