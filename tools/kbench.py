"""Micro-timings of the small per-row kernels in isolation (CUDA events)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2604_08585_b200 import _lib

s = torch.cuda.current_stream().cuda_stream
def t(f, it=50):
    for _ in range(3): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it * 1e3
d = 4096
for m in (32, 800, 5153):
    x = torch.randn(m, d, device="cuda"); g = torch.ones(d, device="cuda"); b = torch.zeros(d, device="cuda")
    o = torch.empty(m, d, device="cuda", dtype=torch.bfloat16)
    us = t(lambda: _lib.call("qcf_layernorm", x.data_ptr(), m, d, g.data_ptr(), b.data_ptr(), 1e-5, o.data_ptr(), 1, s))
    print(f"layernorm m={m}: {us:.1f} us  ({(m*d*6)/us/1e3:.0f} GB/s)")
    qkv = torch.randn(m, 3 * d, device="cuda")
    pos = torch.arange(m, dtype=torch.int32, device="cuda")
    from paper_2604_08585_b200.model import RopeTable
    rope = RopeTable(128, 10000.0, "cuda", 8192)
    qo = torch.empty(m, 32, 128, device="cuda", dtype=torch.bfloat16)
    kt = torch.empty(m, 32, 128, device="cuda", dtype=torch.bfloat16); vt = torch.empty_like(kt)
    us = t(lambda: _lib.call("qcf_rope_qkv_scatter", qkv.data_ptr(), m, 32, 32, 128, pos.data_ptr(), pos.data_ptr(),
                             rope.cos.data_ptr(), rope.sin.data_ptr(), rope.n_pos, qo.data_ptr(), kt.data_ptr(), vt.data_ptr(), 1, s))
    print(f"rope m={m}: {us:.1f} us ({(m*3*d*(4+2))/us/1e3:.0f} GB/s)")
