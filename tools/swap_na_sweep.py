"""M=800 swapped-GEMM activation tile count sweep, cold weights (L2 flushed before
every launch) as in the fused step: python tools/swap_na_sweep.py (QCF_SWAP_NA is
read once per process, so tools/swap_na_sweep.sh runs one process per setting)."""
import sys, os, json
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2604_08585_b200 import _lib
from paper_2604_08585_b200.model import tile64
s = torch.cuda.current_stream().cuda_stream
flush = torch.empty(512 * 1024 * 1024 // 4, device="cuda")
m = int(os.environ.get("QCF_M", "800"))
res = {"na": os.environ.get("QCF_SWAP_NA", "auto"), "m": m}
for n, k, epi, name in [(12288, 4096, 0, "qkv"), (4096, 4096, 2, "wo"), (14336, 4096, 1, "w1"), (4096, 14336, 2, "w2")]:
    a = (torch.randn(m, k, device="cuda") * 0.5).bfloat16()
    b = tile64((torch.randn(n, k, device="cuda") * 0.05).bfloat16())
    out_dt = _lib.QCF_BF16 if epi == 1 else _lib.QCF_F32
    c = torch.zeros(m, n, device="cuda", dtype=torch.bfloat16 if epi == 1 else torch.float32)
    ws = torch.zeros(max(int(_lib.lib.qcf_gemm_workspace(m, n, k)), 16), dtype=torch.uint8, device="cuda")
    f = lambda: _lib.call("qcf_gemm_ws", _lib.QCF_BF16, a.data_ptr(), k, b.data_ptr(), k, c.data_ptr(), n, m, n, k,
                          epi, out_dt, 1, ws.data_ptr(), ws.numel(), s)
    f(); torch.cuda.synchronize()
    ts = []
    for _ in range(7):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(int(2e6))
        e0.record(); f(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    us = ts[len(ts) // 2]
    res[name + "_us"] = round(us, 1)
    res[name + "_tflops"] = round(2.0 * m * n * k / us / 1e6, 1)
print(json.dumps(res), flush=True)
