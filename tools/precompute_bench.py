"""Chunk precompute throughput: 64 Llama-3-8B-shape chunks of
512 tokens, one at a time (ChunkStore.precompute) vs batched
(ChunkStore.precompute_batch, 16 chunks per layer stack)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import json
import tempfile
import time
import numpy as np
import torch
import bench
import paper_2604_08585_b200 as Q

cfgd = dict(bench.CONFIGS["llama3-8b"])
cfg = Q.ModelConfig(n_layers=cfgd["n_layers"], n_heads=cfgd["n_heads"], d_model=cfgd["d_model"],
                    d_head=cfgd["d_head"], d_ff=cfgd["d_ff"], seed=1234)
w = Q.init_weights(cfg, dtype="bf16")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
toks = [np.random.default_rng(i).integers(0, 256, 512) for i in range(n)]
res = {"chunks": n, "chunk_len": 512}
for mode in ("sequential", "batched", "sequential", "batched"):
    st = Q.ChunkStore(tempfile.mkdtemp(), cfg, dtype="bf16", persist=False)
    warm = [np.random.default_rng(10_000 + i).integers(0, 256, 512) for i in range(16)]
    if mode == "batched":
        st.precompute_batch(w, warm, 0.05)          # warm-up: same batch shape (allocations, maps)
    else:
        st.precompute(w, warm[0], 0.05)
    st = Q.ChunkStore(tempfile.mkdtemp(), cfg, dtype="bf16", persist=False)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if mode == "batched":
        st.precompute_batch(w, toks, 0.05)
    else:
        for t in toks:
            st.precompute(w, t, 0.05)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    res[f"{mode}_s"] = round(dt, 3)
    res[f"{mode}_chunks_per_s"] = round(n / dt, 1)
    del st
    torch.cuda.empty_cache()
print(json.dumps(res))
