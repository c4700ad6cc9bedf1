"""TTFT of one request with the assembly forked onto a second stream
(concurrent with the probe) vs strictly serial, same graph-replay harness."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import json
import statistics
import numpy as np
import torch
import bench

cfgd = dict(bench.CONFIGS["llama3-8b"])
Qm, cfg, w, store, eng, ids, toks = bench.build_engine(cfgd, "bf16", torch.device("cuda"), cfgd["n_chunks"])
q = np.random.default_rng(10_000).integers(0, 256, cfgd["q"]).tolist()
out = {}
for conc in (True, False, True, False):
    eng.concurrent = conc
    eng._bufs.clear()
    plan, b = eng.prefill("QCFuse", cfgd["ratio"], ids, q)
    for _ in range(3):
        b.graph.replay()
    ts = []
    for _ in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        b.graph.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    out.setdefault("concurrent" if conc else "serial", []).append(round(statistics.median(ts), 3))
print(json.dumps(out))
