"""Compare an attention kernel knob with the single-tile kernel (v1) on small cases
(python tools/attn_debug.py <knob>): max |diff| and the rows above 2e-2."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2604_08585_b200 import _lib
S = torch.cuda.current_stream().cuda_stream
D = 128
knob = int(sys.argv[1]) if len(sys.argv) > 1 else 9


def run(ver, q, k, v, kmax, m, n, H, Hkv, n_req):
    out = torch.zeros_like(q)
    _lib.call("qcf_set_attention_kernel", ver)
    _lib.call("qcf_attention_batched", 1, q.data_ptr(), k.data_ptr(), v.data_ptr(), kmax.data_ptr(), m, n_req, H, Hkv,
              D, n, out.data_ptr(), S)
    torch.cuda.synchronize()
    _lib.call("qcf_set_attention_kernel", 0)
    return out


for (m, n, H, note, kfn) in [(128, 128, 1, "1 q tile, 1 key tile", lambda m, n: torch.full((1, m), n - 1)),
                             (256, 128, 1, "2 q tiles, 1 key tile", lambda m, n: torch.full((1, m), n - 1)),
                             (256, 384, 1, "2 q tiles, 3 key tiles", lambda m, n: torch.full((1, m), n - 1)),
                             (256, 640, 2, "2 q tiles, 5 key tiles, 2 heads", lambda m, n: torch.full((1, m), n - 1)),
                             (384, 640, 1, "3 q tiles causal-ish", lambda m, n: torch.sort(torch.randint(0, n, (1, m))).values),
                             (800, 5153, 2, "recompute shape", lambda m, n: torch.sort(torch.randint(0, n, (1, m))).values)]:
    torch.manual_seed(0)
    q = torch.randn(1, m, H, D, device="cuda").bfloat16()
    k = torch.randn(1, n, H, D, device="cuda").bfloat16()
    v = torch.randn(1, n, H, D, device="cuda").bfloat16()
    kmax = kfn(m, n).int().cuda().contiguous()
    a = run(1, q, k, v, kmax, m, n, H, H, 1)
    b = run(knob, q, k, v, kmax, m, n, H, H, 1)
    err = (a.float() - b.float()).abs()
    rows_bad = (err.amax(dim=(0, 2, 3)) > 2e-2).nonzero().flatten().tolist()
    print(note, "max err", err.max().item(), "bad rows", rows_bad[:10], len(rows_bad), flush=True)
