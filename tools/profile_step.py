"""One fused QCFuse prefill at Llama-3-8B shape inside an NVTX range
'profile_step' (for `ncu --nvtx --nvtx-include profile_step/`)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import bench

cfgd = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "llama3-8b"])
policy = sys.argv[2] if len(sys.argv) > 2 else "QCFuse"
Q, cfg, w, store, eng, ids, toks = bench.build_engine(cfgd, "bf16", torch.device("cuda"), cfgd["n_chunks"])
q = np.random.default_rng(10_000).integers(0, 256, cfgd["q"]).tolist()
ratio = cfgd["ratio"] if policy == "QCFuse" else 1.0
for _ in range(2):
    eng.prefill(policy, ratio, ids, q, use_graph=False)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("profile_step")
eng.prefill(policy, ratio, ids, q, use_graph=False)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("done")
