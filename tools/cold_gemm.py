"""Cold-L2 qcf_gemm_ws timings vs M for a weight matrix (DRAM-streaming efficiency)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import os
from paper_2604_08585_b200 import _lib
from paper_2604_08585_b200.model import tile64
LAY = int(os.environ.get("QCF_TILED", "1"))  # 1 = tile-major weights (production layout)
n, k = int(sys.argv[1]), int(sys.argv[2])
if len(sys.argv) > 3:
    os.environ.setdefault("QCF_MS", sys.argv[3])
s = torch.cuda.current_stream().cuda_stream
flush = torch.empty(512 * 1024 * 1024 // 4, device="cuda")
b = (torch.randn(n, k, device="cuda") * 0.05).bfloat16()
b = tile64(b) if LAY else b
MS = [int(x) for x in os.environ.get("QCF_MS", "32,128,256,384,512,800,1024,1536").split(",")]
for m in MS:
    a = (torch.randn(m, k, device="cuda") * 0.5).bfloat16()
    c = torch.empty(m, n, device="cuda")
    ws = torch.zeros(max(int(_lib.lib.qcf_gemm_workspace(m, n, k)), 16), dtype=torch.uint8, device="cuda")
    f = lambda: _lib.call("qcf_gemm_ws", 1, a.data_ptr(), k, b.data_ptr(), k, c.data_ptr(), n, m, n, k, 0, 0, LAY,
                          ws.data_ptr(), ws.numel(), s)
    f(); torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(int(2e7))
        e0.record(); f(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    t = sorted(ts)[2]
    print(f"M={m:5d} N={n} K={k}: {t:7.1f} us  weights {n*k*2/t/1e3:6.0f} GB/s  {2*m*n*k/t/1e6:7.1f} TF")
