"""tcgen05 attention kernels at the fused-path shapes (CUDA events): 1 = one
tile per CTA, 2 = ping-pong pairs with half-row softmax threads, 3 = ping-pong
with full-row threads, 4 = two CTAs per SM over 64-key tiles, 8 = two softmax
groups on alternate key tiles with three S buffers (0 = auto).
QCF_ATTN_PAIR=0/1 forces adjacent/mirrored pairing.
FLOPs counted on the exact visible keys: 4*H*D*sum(kmax+1)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import json
import torch
from paper_2604_08585_b200 import _lib

S = torch.cuda.current_stream().cuda_stream
D = 128


def bench(m, n_keys, H, Hkv, n_req, kmax, it=20):
    q = torch.randn(n_req, m, H, D, device="cuda").bfloat16()
    k = torch.randn(n_req, n_keys, Hkv, D, device="cuda").bfloat16()
    v = torch.randn(n_req, n_keys, Hkv, D, device="cuda").bfloat16()
    out = torch.empty_like(q)
    flops = 4.0 * H * D * float((kmax.long() + 1).sum())
    res = {}
    nb = int(_lib.lib.qcf_attention_workspace(m, n_req, H, n_keys))
    ws = torch.empty(max(nb, 16), dtype=torch.uint8, device="cuda")
    res["auto_split"] = int(_lib.lib.qcf_attention_split(m, n_req, H, n_keys))
    order = [int(x) for x in __import__("os").environ.get("QCF_ATTN_ORDER", "1,4,8,0").split(",")]
    for ver in order:   # 0 = auto with workspace (split-KV for one-wave grids)
        _lib.call("qcf_set_attention_kernel", ver)
        f = lambda: _lib.call("qcf_attention_batched_ws", 1, q.data_ptr(), k.data_ptr(), v.data_ptr(),
                              kmax.data_ptr(), m, n_req, H, Hkv, D, n_keys, out.data_ptr(),
                              ws.data_ptr() if ver == 0 else None, nb if ver == 0 else 0, S)
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(it):
            f()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / it
        res[f"v{ver}_us"] = round(ms * 1e3, 1)
        res[f"v{ver}_tflops"] = round(flops / ms / 1e9, 1)
    _lib.call("qcf_set_attention_kernel", 0)
    return res


def sel_kmax(n_ctx, n_sel, q, n_req, seed=0):
    g = torch.Generator().manual_seed(seed)
    rows = []
    for r in range(n_req):
        s = torch.sort(torch.randperm(n_ctx, generator=g)[:n_sel] + 1).values
        rows.append(torch.cat([s, torch.arange(n_ctx + 1, n_ctx + 1 + q)]))
    return torch.stack(rows).int().cuda().contiguous()


for name, n_req, H, Hkv in [("llama batch8", 8, 32, 32), ("llama single", 1, 32, 32), ("llama-gqa batch8", 8, 32, 8)]:
    km = sel_kmax(5120, 768, 32, n_req)
    print(json.dumps({"shape": name, "m": 800, "keys": 5153, **bench(800, 5153, H, Hkv, n_req, km)}), flush=True)
km = torch.arange(5152, dtype=torch.int32, device="cuda")[None].contiguous()
print(json.dumps({"shape": "full prefill causal", "m": 5152, "keys": 5153, **bench(5152, 5153, 32, 32, 1, km)}), flush=True)
km = (torch.arange(32, dtype=torch.int32) + 5121)[None].cuda().contiguous()
print(json.dumps({"shape": "query rows only (FullReuse)", "m": 32, "keys": 5153, **bench(32, 5153, 32, 32, 1, km)}),
      flush=True)
km = (torch.arange(32, dtype=torch.int32) + 261)[None].cuda().contiguous()   # probe: q rows over the anchor prefix
print(json.dumps({"shape": "probe rows (anchor prefix)", "m": 32, "keys": 293, **bench(32, 293, 32, 32, 1, km)}),
      flush=True)
km = (torch.arange(32, dtype=torch.int32) + 261)[None].repeat(8, 1).cuda().contiguous()
print(json.dumps({"shape": "probe rows batch8", "m": 32, "keys": 293, **bench(32, 293, 32, 32, 8, km)}), flush=True)
km = sel_kmax(32768, 4916, 32, 1)
print(json.dumps({"shape": "mistral 32k single", "m": 4948, "keys": 32801, **bench(4948, 32801, 32, 8, 1, km, it=5)}),
      flush=True)
