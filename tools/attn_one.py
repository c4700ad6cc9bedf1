"""One attention launch at the single-request fused shape (for ncu): argv[1] =
knob (0 auto + workspace, 1, 2, 3)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2604_08585_b200 import _lib
sys.argv += ["0"] * 2
ver = int(sys.argv[1])
m, n_keys, H, D, n_req = 800, 5153, 32, 128, int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "0" else 1
g = torch.Generator().manual_seed(0)
rows = [torch.cat([torch.sort(torch.randperm(5120, generator=g)[:768] + 1).values, torch.arange(5121, 5153)])
        for _ in range(n_req)]
kmax = torch.stack(rows).int().cuda().contiguous()
q = torch.randn(n_req, m, H, D, device="cuda").bfloat16()
k = torch.randn(n_req, n_keys, H, D, device="cuda").bfloat16()
v = torch.randn(n_req, n_keys, H, D, device="cuda").bfloat16()
out = torch.empty_like(q)
nb = int(_lib.lib.qcf_attention_workspace(m, n_req, H, n_keys))
ws = torch.empty(max(nb, 16), dtype=torch.uint8, device="cuda")
_lib.call("qcf_set_attention_kernel", ver)
S = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    _lib.call("qcf_attention_batched_ws", 1, q.data_ptr(), k.data_ptr(), v.data_ptr(), kmax.data_ptr(), m, n_req, H, H,
              D, n_keys, out.data_ptr(), ws.data_ptr() if ver == 0 else None, nb if ver == 0 else 0, S)
torch.cuda.synchronize()
