"""Generate the golden fixtures by running the REFERENCE implementation.

Run in the build container only (needs /root/reference):

    python tests/golden/make_golden.py

It imports `qcfuse` from /root/reference/pkg/src read-only, runs the reference's
own fused path (`FusionEngine.run("QCFuse", …)`, `assemble_context`,
`probe_query`, `score_critical`, `recompute_selected`) on seeded synthetic
inputs, and writes small `.npz` fixtures next to this script. Nothing under
/root/reference is copied; the reference's own known-answer file
`tests/data/golden_logits_ab.json` is re-serialised as data.
"""

from __future__ import annotations

import json
import shutil
import sys
import tempfile
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
HERE = Path(__file__).resolve().parent


def _import_reference():
    sys.path.insert(0, str(REF / "src"))
    import qcfuse.fusion as fusion  # noqa: E402
    import qcfuse.model as model  # noqa: E402
    import qcfuse.store as store  # noqa: E402
    return model, store, fusion


def _case(model, store_mod, fusion, cfg_kwargs, chunk_sizes, n_query, ratio,
          anchor_ratio, chunk_seed0, query_seed, max_new, full_rows: bool):
    cfg = model.ModelConfig(**cfg_kwargs)
    w = model.init_weights(cfg)
    tmp = Path(tempfile.mkdtemp(prefix="qcf-golden-"))
    try:
        st = store_mod.ChunkStore(tmp / "store", cfg)
        eng = fusion.FusionEngine(w, st)
        chunk_tokens, cids = [], []
        for i, n in enumerate(chunk_sizes):
            toks = np.random.default_rng(chunk_seed0 + i).integers(0, 256, n)
            chunk_tokens.append(toks.astype(np.int64))
            cids.append(st.precompute(w, [int(t) for t in toks], anchor_ratio, f"c{i}").chunk_id)
        query = np.random.default_rng(query_seed).integers(0, 256, n_query).astype(np.int64)
        qlist = [int(t) for t in query]

        fused = eng.assemble_context(cids)
        probe = eng.probe_query(qlist, fused, fusion.PROBE_ANCHORS)
        scores = eng.score_critical(probe, fused)
        sel = fusion.select_topn(scores, ratio)
        upd, _ = eng.recompute_selected(fused, sel)
        res = eng.run("QCFuse", ratio, cids, qlist, max_new=max_new)
        assert np.array_equal(res.selection.indices, sel.indices)
        full = eng.oracle_run(fused.token_ids, qlist, max_new=max_new)

        c = cfg.critical_layer
        s64 = np.sort(scores.astype(np.float64))[::-1]
        n = sel.indices.size
        gap = float((s64[n - 1] - s64[n]) / s64[n - 1]) if 0 < n < s64.size else float("nan")
        out = {
            "cfg": json.dumps(cfg.to_dict()),
            "ratio": ratio, "anchor_ratio": anchor_ratio,
            "query": query,
            "first_logits": res.first_logits.astype(np.float32),
            "full_logits": full["first_logits"].astype(np.float32),
            "answer": np.asarray(res.answer_tokens, np.int64),
            "full_answer": np.asarray(full["answer_tokens"], np.int64),
            "offsets": np.asarray(fused.offsets, np.int64),
            "q_c": probe.queries[c - 1].astype(np.float32),
            "prefix_positions": probe.prefix_positions.astype(np.int64),
            "scores": scores.astype(np.float32),
            "selection": sel.indices.astype(np.int64),
            "cutoff_rel_gap": gap,
        }
        for i, toks in enumerate(chunk_tokens):
            rec = st.get_record(cids[i])
            out[f"chunk{i}_tokens"] = toks
            out[f"chunk{i}_anchors"] = rec.anchor_indices.astype(np.int64)
            out[f"chunk{i}_norms"] = rec.key_norms.astype(np.float32)
        L = cfg.n_layers
        sample = np.unique(np.clip(np.array([0, 1, 2, fused.n_ctx // 3, fused.n_ctx // 2,
                                             fused.n_ctx - 1, fused.n_ctx]), 0, fused.n_ctx))
        out["sample_rows"] = sample
        for li in range(L):
            fk, fv = fused.layer_kv[li].keys, fused.layer_kv[li].values
            uk, uv = upd.layer_kv[li].keys, upd.layer_kv[li].values
            if full_rows:
                out[f"fused_k{li}"], out[f"fused_v{li}"] = fk, fv
                out[f"upd_k{li}"], out[f"upd_v{li}"] = uk, uv
            else:
                out[f"fused_k{li}"] = fk[sample]
                out[f"fused_v{li}"] = fv[sample]
                srow = sel.indices[:: max(1, sel.indices.size // 8)][:8]
                out[f"upd_rows{li}"] = srow
                out[f"upd_k{li}"] = uk[srow]
                out[f"upd_v{li}"] = uv[srow]
            out[f"fused_ksum{li}"] = np.float64(fk.astype(np.float64).sum())
            out[f"fused_vsum{li}"] = np.float64(fv.astype(np.float64).sum())
            out[f"upd_ksum{li}"] = np.float64(uk.astype(np.float64).sum())
            out[f"upd_vsum{li}"] = np.float64(uv.astype(np.float64).sum())
        return out
    finally:
        shutil.rmtree(tmp, ignore_errors=True)


def main():
    model, store_mod, fusion = _import_reference()

    # (1) the reference's own frozen logits fixture, re-serialised as data
    src = json.loads((REF / "tests/data/golden_logits_ab.json").read_text())
    (HERE / "ref_golden_logits_ab.json").write_text(json.dumps(src, indent=1))

    # (2) the reference conftest "small" config (L4 H2 d32 dh16 dff64 seed 1234)
    small = dict(n_layers=4, n_heads=2, d_model=32, d_head=16, d_ff=64, seed=1234)
    for k, (sizes, nq, r, ar) in enumerate([((20, 24), 6, 0.3, 0.25),
                                             ((16, 18, 12), 4, 0.5, 0.05),
                                             ((9,), 1, 0.2, 0.3)]):
        d = _case(model, store_mod, fusion, small, sizes, nq, r, ar, 100 + 10 * k, 500 + k,
                  max_new=8, full_rows=True)
        np.savez_compressed(HERE / f"small_case{k}.npz", **d)

    # (3) BASELINE config 1: L4 H4 D64 d256 F1024, 4x128 chunks, q16, r .15
    tiny = dict(n_layers=4, n_heads=4, d_model=256, d_head=64, d_ff=1024, seed=1234)
    for k in range(6):
        d = _case(model, store_mod, fusion, tiny, (128, 128, 128, 128), 16, 0.15, 0.05,
                  0, 10_000 + k, max_new=8 if k == 0 else 1, full_rows=False)
        np.savez_compressed(HERE / f"tiny_case{k}.npz", **d)
        print(f"tiny case {k}: N={d['selection'].size} cutoff rel gap {d['cutoff_rel_gap']:.3e}")

    # (4) splitmix64 + init vectors for a Llama-width slice (first draws of each tensor)
    cfg = model.ModelConfig(n_layers=32, n_heads=32, d_model=4096, d_head=128, d_ff=14336,
                            seed=1234)
    shapes = [(cfg.vocab_size, cfg.d_model)]
    for _ in range(cfg.n_layers):
        shapes += [(4096, 4096)] * 4 + [(4096, 14336), (14336, 4096)]
    starts, off = [], 0
    for r, c in shapes:
        starts.append(off)
        off += r * c
    steps = np.concatenate([np.arange(s, s + 16, dtype=np.uint64) for s in starts[:13]]
                           + [np.arange(off - 16, off, dtype=np.uint64)])
    u = model.uniform_from_u64(model.splitmix64_at(cfg.seed, steps))
    vals = (model.WEIGHT_LOW + u * (model.WEIGHT_HIGH - model.WEIGHT_LOW)).astype(np.float32)
    np.savez_compressed(HERE / "init_llama_probe.npz", steps=steps, values=vals,
                        total=np.uint64(off))
    print("wrote fixtures to", HERE)


if __name__ == "__main__" and len(sys.argv) == 1:
    main()


def extra_fixtures():
    """Reference-written .qcfk chunk + manifest, random_select / epic_select
    outputs, policy schedules (host-logic parity)."""
    model, store_mod, fusion = _import_reference()
    import qcfuse.pipeline as pipeline
    cfg = model.ModelConfig(n_layers=4, n_heads=2, d_model=32, d_head=16, d_ff=64, seed=1234)
    w = model.init_weights(cfg)
    root = HERE / "ref_store"
    if root.exists():
        shutil.rmtree(root)
    st = store_mod.ChunkStore(root, cfg)
    toks = [int(t) for t in np.random.default_rng(77).integers(0, 256, 19)]
    rec = st.precompute(w, toks, 0.25, "ref-chunk")
    out = {"chunk_id": rec.chunk_id, "anchors": rec.anchor_indices.tolist(),
           "fingerprint": store_mod.config_fingerprint(cfg)}
    rs = {}
    for seed, n, r in [(0, 37, 0.3), (5, 100, 0.15), (9, 7, 1.0), (3, 50, 0.0)]:
        rs[f"{seed}_{n}_{r}"] = fusion.random_select(seed, n, r).indices.tolist()
    out["random_select"] = rs
    out["epic"] = fusion.epic_select(40, 0.2, [(1, 15), (16, 25)]).indices.tolist()
    sch = pipeline.policy_schedule("QCFuse", 51, 256, 16, model.ModelConfig(), pipeline.CostModel())
    out["schedule_qcfuse"] = {"ttft": sch.ttft, "compute_end": sch.compute_end, "pre": sch.pre_phase}
    (HERE / "host_logic.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "extra":
    extra_fixtures()


def baseline_fixtures():
    """Reference selections of the comparison policies (fusion.py:352-411):
    CacheBlend / KVShare (layer-1 deviation, received attention), QCLast, QCAll,
    on the reference conftest config and BASELINE config 1 -> baselines.npz."""
    model, store_mod, fusion = _import_reference()
    out = {}
    cases = [("small", dict(n_layers=4, n_heads=2, d_model=32, d_head=16, d_ff=64, seed=1234), (20, 24, 17), 6, 0.3),
             ("small2", dict(n_layers=4, n_heads=2, d_model=32, d_head=16, d_ff=64, seed=1234), (33, 12), 4, 0.15),
             ("tiny", dict(n_layers=4, n_heads=4, d_model=256, d_head=64, d_ff=1024, seed=1234), (128, 128), 16, 0.15)]
    for name, cfgk, sizes, nq, ratio in cases:
        cfg = model.ModelConfig(**cfgk)
        w = model.init_weights(cfg)
        tmp = Path(tempfile.mkdtemp(prefix="qcf-golden-"))
        try:
            st = store_mod.ChunkStore(tmp / "store", cfg)
            eng = fusion.FusionEngine(w, st)
            cids, toks_all = [], []
            for i, n in enumerate(sizes):
                toks = np.random.default_rng(300 + i).integers(0, 256, n)
                toks_all.append(toks.astype(np.int64))
                cids.append(st.precompute(w, [int(t) for t in toks], 0.1, f"c{i}").chunk_id)
            query = [int(t) for t in np.random.default_rng(900).integers(0, 256, nq)]
            fused = eng.assemble_context(cids)
            new_k, new_v, attn = eng._layer1_recompute_pass(fused)
            dev = eng._kv_deviation(fused, new_k, new_v)
            out[f"{name}_cfg"] = json.dumps(cfg.to_dict())
            out[f"{name}_ratio"] = ratio
            out[f"{name}_query"] = np.asarray(query, np.int64)
            out[f"{name}_n_chunks"] = len(sizes)
            for i, t in enumerate(toks_all):
                out[f"{name}_chunk{i}_tokens"] = t
            out[f"{name}_deviation"] = dev.astype(np.float32)
            out[f"{name}_received"] = attn[:, :, 1:].mean(axis=(0, 1)).astype(np.float32)
            for pol in ("CacheBlend", "KVShare", "QCLast", "QCAll"):
                out[f"{name}_{pol}"] = eng.select(pol, ratio, fused, query).indices.astype(np.int64)
        finally:
            shutil.rmtree(tmp, ignore_errors=True)
    np.savez_compressed(HERE / "baselines.npz", **out)
    print("wrote", HERE / "baselines.npz")


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "baselines":
    baseline_fixtures()


def calibration_fixtures():
    """The reference's calibrate_layer (bench.py:118-144) on a 6-layer config
    (candidate layers 2..5) over text chunks it retrieves itself
    (cases.retrieve): records the chunk token lists each query retrieved, the
    per-layer mean overlaps and the recommended layer -> calibrate.npz."""
    model, store_mod, fusion = _import_reference()
    import qcfuse.bench as bench  # noqa: E402
    import qcfuse.cases as cases  # noqa: E402
    cfg = model.ModelConfig(n_layers=6, n_heads=2, d_model=32, d_head=16, d_ff=64, seed=4321)
    w = model.init_weights(cfg)
    texts = ["the quick brown fox jumps over the lazy dog near the river bank",
             "a fused cache keeps the keys and values of every retrieved chunk",
             "rotary position embeddings rotate pairs of key dimensions by angle",
             "selective recompute refreshes the tokens the query attends to most",
             "the river bank was flooded after the storm and the fox swam across",
             "values are copied while keys are re-rotated to their fused offsets"]
    queries = ["which tokens does the query attend to", "where did the fox swim", "how are keys rotated"]
    tmp = Path(tempfile.mkdtemp(prefix="qcf-golden-"))
    out = {"cfg": json.dumps(cfg.to_dict()), "ratio": 0.2, "top_k": 3, "n_queries": len(queries)}
    try:
        st = store_mod.ChunkStore(tmp / "store", cfg)
        eng = fusion.FusionEngine(w, st)
        for i, t in enumerate(texts):
            toks = [int(b) for b in t.encode("utf-8")]
            st.precompute(w, toks, 0.05, f"t{i}")
            out[f"text{i}_tokens"] = np.asarray(toks, np.int64)
        out["n_texts"] = len(texts)
        res = bench.calibrate_layer(eng, queries, ratio=0.2, top_k=3)
        for qi, q in enumerate(queries):
            out[f"query{qi}"] = np.asarray(list(q.encode("utf-8")), np.int64)
            ids = cases.retrieve(st, q, 3)
            for ci, cid in enumerate(ids):
                out[f"query{qi}_chunk{ci}_tokens"] = np.asarray(st.load_meta(cid).token_ids, np.int64)
        out["recommended"] = int(res["recommended"])
        out["layers"] = np.asarray(sorted(res["mean_overlap"]), np.int64)
        out["mean_overlap"] = np.asarray([res["mean_overlap"][k] for k in sorted(res["mean_overlap"])], np.float64)
    finally:
        shutil.rmtree(tmp, ignore_errors=True)
    np.savez_compressed(HERE / "calibrate.npz", **out)
    print("wrote", HERE / "calibrate.npz", out["recommended"], out["mean_overlap"])


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "calibrate":
    calibration_fixtures()
