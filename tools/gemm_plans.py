"""TFLOP/s of every tcgen05 GEMM tile plan at the fused-path shapes (CUDA events; +8 = stream-K on;
tile-major weights as in production). Plans: 1 = 2-CTA 256x256, 2 = 1-CTA
128x256, 3 = 128x128, 4 = 128x64, 6 = 2-CTA 256x128, 0 = the auto choice
(QCF_PLANS=0,1,6 selects)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import json
import torch
from paper_2604_08585_b200 import _lib
from paper_2604_08585_b200.model import tile64

S = torch.cuda.current_stream().cuda_stream
FLUSH = __import__("os").environ.get("QCF_FLUSH", "0") == "1"
flush = torch.ones(64 << 20, dtype=torch.float32, device="cuda") if FLUSH else None
ms = [int(x) for x in sys.argv[1:]] or [800, 6400]
for m in ms:
    for n, k, epi in [(12288, 4096, 0), (4096, 4096, 0), (14336, 4096, 1), (4096, 14336, 0)]:
        a = (torch.randn(m, k, device="cuda") * 0.5).bfloat16()
        b = tile64((torch.randn(n, k, device="cuda") * 0.05).bfloat16())
        out_dt = 1 if epi == 1 else 0
        c = torch.empty(m, n, device="cuda", dtype=torch.bfloat16 if epi == 1 else torch.float32)
        row = {"m": m, "n": n, "k": k}
        ws = torch.zeros(int(_lib.lib.qcf_gemm_workspace(m, n, k)), dtype=torch.uint8, device="cuda")
        plans = [int(x) for x in __import__("os").environ.get("QCF_PLANS", "0,8,1,9,2,3,4,6").split(",")]
        for plan in plans:
            _lib.call("qcf_set_gemm_plan", plan)
            f = lambda: _lib.call("qcf_gemm_ws", 1, a.data_ptr(), k, b.data_ptr(), k, c.data_ptr(), n, m, n, k, epi,
                                  out_dt, 1, ws.data_ptr(), ws.numel(), S)
            for _ in range(3):
                f()
            torch.cuda.synchronize()
            if FLUSH:  # cold L2 per launch (a 256 MB READ between launches -- clean lines, no write-back
                # traffic during the timed launch -- outside the events)
                ms_ = 0.0
                for _ in range(10):
                    flush.sum()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    f()
                    e1.record()
                    torch.cuda.synchronize()
                    ms_ += e0.elapsed_time(e1) / 10
            else:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(20):
                    f()
                e1.record()
                torch.cuda.synchronize()
                ms_ = e0.elapsed_time(e1) / 20
            row[f"plan{plan}_us"] = round(ms_ * 1e3, 1)
            row[f"plan{plan}_tflops"] = round(2 * m * n * k / ms_ / 1e9, 1)
        _lib.call("qcf_set_gemm_plan", 0)
        print(json.dumps(row), flush=True)
