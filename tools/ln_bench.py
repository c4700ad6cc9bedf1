"""qcf_add_layernorm at the fused-path shapes: achieved HBM GB/s (x+delta read,
x+out written)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import json
import torch
from paper_2604_08585_b200 import _lib

s = torch.cuda.current_stream().cuda_stream
d = 4096
for m in (32, 256, 800, 6400):
    x = torch.randn(m, d, device="cuda")
    dl = torch.randn(m, d, device="cuda")
    g = torch.ones(d, device="cuda")
    b = torch.zeros(d, device="cuda")
    o = torch.empty(m, d, device="cuda", dtype=torch.bfloat16)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    f = lambda: _lib.call("qcf_add_layernorm", x.data_ptr(), dl.data_ptr(), m, d, g.data_ptr(), b.data_ptr(), 1e-5,
                          o.data_ptr(), 1, s)
    for _ in range(3):
        f()
    ts = []
    for _ in range(20):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        f()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = sorted(ts)[len(ts) // 2]
    by = m * d * (4 + 4 + 4 + 2)
    print(json.dumps({"kernel": "add_layernorm", "m": m, "d": d, "us": round(ms * 1e3, 1),
                      "GBps": round(by / ms / 1e6, 1), "note": "L2 flushed before each launch"}))
