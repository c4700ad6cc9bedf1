"""Swapped vs normal 2-CTA GEMM: bit-equality of the fp32 results and the time of
the fused QKV + RoPE launch at the single request's shape (plans 0 / 1 / 7)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import json
import torch
from paper_2604_08585_b200 import _lib
from paper_2604_08585_b200.model import tile64, RopeTable

S = torch.cuda.current_stream().cuda_stream
call = _lib.call
for m, n, k in [(800, 4096, 4096), (512, 4096, 1024)]:
    a = (torch.randn(m, k, device="cuda") * 0.5).bfloat16()
    b = tile64((torch.randn(n, k, device="cuda") * 0.05).bfloat16())
    res = {}
    for plan in (1, 4, 7):
        call("qcf_set_gemm_plan", plan)
        c = torch.empty(m, n, device="cuda")
        call("qcf_gemm_ws", 1, a.data_ptr(), k, b.data_ptr(), k, c.data_ptr(), n, m, n, k, 0, 0, 1, None, 0, S)
        res[plan] = c
    torch.cuda.synchronize()
    call("qcf_set_gemm_plan", 0)
    print(json.dumps({"m": m, "n": n, "k": k, "pair_eq_one": bool(torch.equal(res[1], res[4])),
                      "swap_eq_pair": bool(torch.equal(res[7], res[1])),
                      "swap_diff_max": (res[7] - res[1]).abs().max().item(),
                      "swap_ndiff": int((res[7] != res[1]).sum().item())}))
m, H, D, K = 800, 32, 128, 4096
N = 3 * H * D
a = (torch.randn(m, K, device="cuda") * 0.5).bfloat16()
w = tile64((torch.randn(N, K, device="cuda") * 0.05).bfloat16())
pos = torch.sort(torch.randperm(6000, device="cuda")[:m]).values.int()
rope = RopeTable(D, 500000.0, "cuda", 8192)
q = torch.empty(m, H, D, device="cuda", dtype=torch.bfloat16)
kt = torch.zeros(6000, H, D, device="cuda", dtype=torch.bfloat16)  # unwritten rows stay 0 (not NaN garbage)
vt = torch.zeros_like(kt)
row = {"shape": "qkv_rope 800x12288x4096"}
outs = {}
for plan in (0, 1, 7, 0):
    call("qcf_set_gemm_plan", plan)
    f = lambda: call("qcf_gemm_qkv_rope", a.data_ptr(), K, w.data_ptr(), K, 1, m, K, H, H, D, pos.data_ptr(),
                     pos.data_ptr(), rope.cs32.data_ptr(), rope.n_pos, q.data_ptr(), kt.data_ptr(), vt.data_ptr(),
                     None, 0, S)
    for _ in range(3):
        f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(20):
        f()
    e1.record()
    torch.cuda.synchronize()
    row[f"plan{plan}_us"] = round(e0.elapsed_time(e1) / 20 * 1e3, 1)
    outs[plan] = (q.clone(), kt[:m].clone(), vt[:m].clone())
call("qcf_set_gemm_plan", 0)
row["rope_swap_eq_pair"] = [bool(torch.equal(x, y)) for x, y in zip(outs[7], outs[1])]
row["rope_swap_ndiff"] = [int((x != y).sum().item()) for x, y in zip(outs[7], outs[1])]
written = torch.zeros(m, dtype=torch.bool, device="cuda")
written[pos[pos < m].long()] = True
row["k_ndiff_written_rows"] = int((outs[7][1][written] != outs[1][1][written]).sum().item())
print(json.dumps(row))
