"""One fused QCFuse prefill step inside an NVTX range 'profile_step' (for
`ncu --nvtx --nvtx-include profile_step/`).

  python tools/profile_step.py [config] [policy] [batch]
batch > 1 profiles the bench's batched step (BASELINE configs[2]: B requests of
10 chunks drawn from a 64-chunk pool, one prefill_batch launch sequence)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import bench

cfgd = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "llama3-8b"])
policy = sys.argv[2] if len(sys.argv) > 2 else "QCFuse"
B = int(sys.argv[3]) if len(sys.argv) > 3 else 1
pool = 64 if B > 1 else cfgd["n_chunks"]
Q, cfg, w, store, eng, ids, toks = bench.build_engine(cfgd, "bf16", torch.device("cuda"), pool)
ratio = cfgd["ratio"] if policy == "QCFuse" else 1.0
chunk_lists, queries = [], []
for i in range(B):
    g = np.random.default_rng(1_000_000 + i)
    chunk_lists.append([ids[j] for j in g.permutation(pool)[:cfgd["n_chunks"]]] if B > 1 else ids)
    queries.append(g.integers(0, 256, cfgd["q"]).tolist())
for _ in range(2):
    eng.prefill_batch(policy, ratio, chunk_lists, queries, use_graph=False)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("profile_step")
eng.prefill_batch(policy, ratio, chunk_lists, queries, use_graph=False)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("done")
