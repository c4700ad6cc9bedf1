"""Run one qcf_gemm_ws shape a few times (for ncu)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import os
from paper_2604_08585_b200 import _lib
from paper_2604_08585_b200.model import tile64
LAY = int(os.environ.get("QCF_TILED", "1"))  # 1 = tile-major weights (production layout)
m, n, k, epi = (int(x) for x in sys.argv[1:5])
_lib.call("qcf_set_gemm_plan", int(os.environ.get("QCF_PLAN", "0")))
if epi == 9:  # fused QKV + RoPE + KV scatter (n = 3*H*D)
    from paper_2604_08585_b200.model import RopeTable
    D = 128; H = n // (3 * D)
    a = (torch.randn(m, k, device="cuda") * 0.5).bfloat16()
    w = (torch.randn(n, k, device="cuda") * 0.05).bfloat16()
    w = tile64(w) if LAY else w
    pos = torch.arange(m, dtype=torch.int32, device="cuda")
    rope = RopeTable(D, 10000.0, "cuda", 8192)
    q = torch.empty(m, H, D, device="cuda", dtype=torch.bfloat16); kt = torch.empty_like(q); vt = torch.empty_like(q)
    s = torch.cuda.current_stream().cuda_stream
    wsq = torch.zeros(int(_lib.lib.qcf_gemm_workspace(m, n, k)), dtype=torch.uint8, device="cuda")
    for _ in range(4):
        _lib.call("qcf_gemm_qkv_rope", a.data_ptr(), k, w.data_ptr(), k, LAY, m, k, H, H, D, pos.data_ptr(), pos.data_ptr(),
                  rope.cs32.data_ptr(), rope.n_pos, q.data_ptr(), kt.data_ptr(), vt.data_ptr(), wsq.data_ptr(), wsq.numel(), s)
    torch.cuda.synchronize()
    sys.exit(0)
a = (torch.randn(m, k, device="cuda") * 0.5).bfloat16()
b = (torch.randn(n, k, device="cuda") * 0.05).bfloat16()
b = tile64(b) if LAY else b
out_dt = _lib.QCF_BF16 if epi == 1 else _lib.QCF_F32
c = torch.zeros(m, n, device="cuda", dtype=torch.bfloat16 if epi == 1 else torch.float32)
ws = torch.zeros(max(int(_lib.lib.qcf_gemm_workspace(m, n, k)), 16), dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for _ in range(4):
    _lib.call("qcf_gemm_ws", _lib.QCF_BF16, a.data_ptr(), k, b.data_ptr(), k, c.data_ptr(), n, m, n, k, epi, out_dt, LAY,
              ws.data_ptr(), ws.numel(), s)
torch.cuda.synchronize()
