"""TTFT of one request (graph replay, median of 20) for the assembly schedules:
serial (main stream, before the probe), pipelined on a side stream with layer
ranges of 1/2/4/8 (critical layer during the probe, the rest with the recompute),
and `concurrent` (every range at once, overlapping the probe)."""
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
modes = [("serial", False, 4, False)] + [(f"pipelined/{g}", True, g, False) for g in (1, 2, 4, 8)] + \
        [("concurrent/4", True, 4, True), ("serial", False, 4, False)]
for name, pipe, g, conc in modes:
    eng.pipeline_asm, eng.asm_group, eng.concurrent = pipe, g, conc
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
    out.setdefault(name, []).append(round(statistics.median(ts), 3))
print(json.dumps(out))
