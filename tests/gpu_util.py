"""Helpers shared by the GPU parity tests (oracle = checker only)."""

from __future__ import annotations

import json

import numpy as np
import torch

from oracle import qcfuse_oracle as O


def oracle_cfg_from_golden(z) -> O.Config:
    d = json.loads(str(z["cfg"]))
    return O.Config(**{k: d[k] for k in ("n_layers", "n_heads", "d_model", "d_head", "d_ff",
                                         "rope_theta", "ln_eps", "seed", "critical_layer")})


def to_model_config(oc: O.Config):
    import paper_2604_08585_b200 as Q
    return Q.ModelConfig(n_layers=oc.n_layers, n_heads=oc.n_heads, d_model=oc.d_model,
                         d_head=oc.d_head, d_ff=oc.d_ff, rope_theta=oc.rope_theta, ln_eps=oc.ln_eps,
                         seed=oc.seed, critical_layer=oc.critical_layer, n_kv_heads=oc.n_kv_heads)


def device_weights(ow: O.Weights, dtype: str):
    import paper_2604_08585_b200 as Q
    cfg = to_model_config(ow.cfg)
    return Q.ModelWeights.from_host(cfg, ow.emb, ow.layers, dtype=dtype)


def load_oracle_chunks(store, chunks: list[O.Chunk]) -> list[str]:
    """Put oracle-precomputed chunk KV into the device pool (isolates the fused
    path from precompute rounding, like the reference's .qcfk bridge)."""
    ids = []
    for c in chunks:
        k = torch.as_tensor(np.stack([kv.keys for kv in c.kv]))
        v = torch.as_tensor(np.stack([kv.values for kv in c.kv]))
        rec = store.add_record(c.tokens, k.to(store.device), v.to(store.device), c.key_norms,
                               c.anchors, "oracle")
        ids.append(rec.chunk_id)
    return ids


def golden_setup(golden_dir, name, dtype="f32", tmp=None):
    import paper_2604_08585_b200 as Q
    z = np.load(golden_dir / f"{name}.npz")
    oc = oracle_cfg_from_golden(z)
    ow = O.init_weights(oc)
    nc = len([k for k in z.files if k.startswith("chunk") and k.endswith("_tokens")])
    chunks = [O.precompute_chunk(ow, z[f"chunk{i}_tokens"], float(z["anchor_ratio"])) for i in range(nc)]
    w = device_weights(ow, dtype)
    store = Q.ChunkStore(tmp, w.config, dtype=dtype, persist=False)
    ids = load_oracle_chunks(store, chunks)
    eng = Q.FusionEngine(w, store)
    return z, oc, ow, chunks, w, store, ids, eng
