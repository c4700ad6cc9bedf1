"""Greedy decode over the fused table after one Llama-3-8B fused prefill:
ms per generated token, eager loop (host argmax per token) vs the replayed CUDA
graph with the device argmax (qcf_decode_advance). Decode is a weight stream of
~11.8 GB per token (M = 1), so the HBM floor is ~1.8 ms per token."""
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import json
import numpy as np
import torch
import bench

cfgd = dict(bench.CONFIGS["llama3-8b"])
Qm, cfg, w, store, eng, ids, toks = bench.build_engine(cfgd, "bf16", torch.device("cuda"), cfgd["n_chunks"])
q = np.random.default_rng(10_000).integers(0, 256, cfgd["q"]).tolist()
max_new = 33
res = {"max_new": max_new}
for graph in (False, True, False, True):
    eng.decode_graph = graph
    plan, b = eng.prefill("QCFuse", cfgd["ratio"], ids, q, use_graph=False, extra_rows=max_new)
    first = b.logits[0].cpu().numpy()
    next_pos = plan.n_ctx + 1 + len(q)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    toks_out = eng._decode(b.fk, b.fv, next_pos, first, max_new)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) * 1e3
    key = "graph" if graph else "eager"
    res.setdefault(key + "_ms_per_token", []).append(round(dt / max(1, len(toks_out) - 1), 3))
    res[key + "_tokens"] = len(toks_out)
print(json.dumps(res))
