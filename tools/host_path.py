"""Where fuse()'s host-side time goes (Llama-3-8B shape, one request): wall time of
plan / buffers / staging / graph launch / D2H around the device TTFT."""
import sys, time, json
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import bench

cfgd = dict(bench.CONFIGS["llama3-8b"])
Q, cfg, w, store, eng, ids, toks = bench.build_engine(cfgd, "bf16", "cuda", 12)
ids1 = ids[:cfgd["n_chunks"]]
q = [int(x) for x in np.random.default_rng(5).integers(0, 256, cfgd["q"])]
for _ in range(5):
    eng.fuse(q, ids1, 0.15)
torch.cuda.synchronize()
res = {}
T = lambda: time.perf_counter() * 1e3  # noqa: E731
acc = {k: [] for k in ("plan", "buffers", "stage", "replay_launch", "gpu_wait", "d2h", "fuse_total")}
for it in range(20):
    t0 = T()
    plans = [eng._plan("QCFuse", 0.15, ids1, q)]
    t1 = T()
    b = eng._buffers(plans, 0)
    t2 = T()
    eng._stage(plans, b, [q])
    t3 = T()
    b.uses += 1
    b.graph.replay()
    t4 = T()
    torch.cuda.current_stream().synchronize()
    t5 = T()
    lg = b.logits[0].cpu().numpy(); sel = b.rc_pos[:plans[0].n_sel].cpu().numpy()
    t6 = T()
    t7 = T(); eng.fuse(q, ids1, 0.15); t8 = T()
    for k, v in zip(acc, (t1 - t0, t2 - t1, t3 - t2, t4 - t3, t5 - t4, t6 - t5, t8 - t7)):
        acc[k].append(v)
print(json.dumps({k: round(float(np.median(v)), 3) for k, v in acc.items()}))
