"""Launch-gap check: a CUDA graph of 400 dependent small kernels (add_rows),
timed with and without Programmatic Dependent Launch (QCF_PDL env)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2604_08585_b200 import _lib
x = torch.zeros(4096 * 16, device="cuda"); d = torch.ones_like(x)
side = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=side):
    for _ in range(400):
        _lib.call("qcf_add_rows", x.data_ptr(), d.data_ptr(), x.numel(), side.cuda_stream)
g.replay(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
print("us per kernel:", e0.elapsed_time(e1) * 1e3 / 400, "x[0] =", x[0].item())
