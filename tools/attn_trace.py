"""Per-CTA timeline of the single-tile tcgen05 attention kernel (measurement
build: `make trace` -> tools/bin/libqcf_trace.so, compiled with QCF_ATTN_TRACE).
Prints per-CTA setup (entry -> first S ready), main loop (per key tile), epilogue,
and the idle gap between consecutive CTAs on one SM."""
import os
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
os.environ["QCFUSE_B200_LIB"] = str(ROOT / "tools/bin" / os.environ.get("QCF_TRACE_LIB", "libqcf_trace.so"))

sys.path.insert(0, str(ROOT))
import ctypes
import json
import numpy as np
import torch
from paper_2604_08585_b200 import _lib

S = torch.cuda.current_stream().cuda_stream
D = 128


def sel_kmax(n_ctx, n_sel, q, n_req, seed=0):
    g = torch.Generator().manual_seed(seed)
    rows = []
    for r in range(n_req):
        s = torch.sort(torch.randperm(n_ctx, generator=g)[:n_sel] + 1).values
        rows.append(torch.cat([s, torch.arange(n_ctx + 1, n_ctx + 1 + q)]))
    return torch.stack(rows).int().cuda().contiguous()


def run(name, m, n_keys, H, Hkv, n_req, kmax):
    q = torch.randn(n_req, m, H, D, device="cuda").bfloat16()
    k = torch.randn(n_req, n_keys, Hkv, D, device="cuda").bfloat16()
    v = torch.randn(n_req, n_keys, Hkv, D, device="cuda").bfloat16()
    out = torch.empty_like(q)
    n_cta = H * ((m + 127) // 128) * n_req
    buf = torch.zeros(n_cta * 8, dtype=torch.int64, device="cuda")
    _lib.call("qcf_set_attention_kernel", int(os.environ.get("QCF_TRACE_KNOB", "1")))
    f = lambda: _lib.call("qcf_attention_batched", 1, q.data_ptr(), k.data_ptr(), v.data_ptr(), kmax.data_ptr(), m,
                          n_req, H, Hkv, D, n_keys, out.data_ptr(), S)
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    buf2 = torch.zeros(64 * 8, dtype=torch.int64, device="cuda")
    _lib.lib.qcf_debug_set_attn_trace(ctypes.c_void_p(buf.data_ptr()))
    _lib.lib.qcf_debug_set_attn_trace2(ctypes.c_void_p(buf2.data_ptr()))
    f()
    torch.cuda.synchronize()
    _lib.lib.qcf_debug_set_attn_trace(ctypes.c_void_p(0))
    _lib.lib.qcf_debug_set_attn_trace2(ctypes.c_void_p(0))
    c = buf2.view(64, 8).cpu().numpy().astype(np.int64)
    nj = int((c[:, 0] > 0).sum())
    if nj > 12:
        js = range(4, min(nj - 2, 14))
        d = lambda a, b: [int(c[j, b] - c[j, a]) for j in js]
        print(json.dumps({"cta0_key_tiles": nj, "clk_per_tile": [int(c[j + 1, 0] - c[j, 0]) for j in js],
                          "s_wait_to_exp_end": d(0, 3), "pv_p_seen_to_v_ready": d(7, 1),
                          "pv_v_ready_to_mmas_issued": d(1, 2), "pv_mmas_to_commits": d(2, 6),
                          "exp_end_to_arrive": d(3, 4),
                          "arrive_to_next_s": [int(c[j + 1, 0] - c[j, 4]) for j in js],
                          "p_seen_by_mma_to_pv_issued": d(7, 6),
                          "p_arrive_to_p_seen_by_mma": d(4, 7),
                          "p_arrive_to_pv_issued": [int(c[j, 6] - c[j, 4]) for j in js],
                          "s_issued_to_s_seen": [int(c[j, 0] - c[j, 5]) for j in js],
                          "s_issue_gap": [int(c[j + 1, 5] - c[j, 5]) for j in js]}), flush=True)
        t0 = c[10, 4]
        names = {0: "softmax sees S", 3: "exp end", 4: "softmax arrive P", 7: "MMA sees P", 1: "V ready",
                 2: "PV MMAs issued", 6: "PV committed", 5: "S committed"}
        ev = sorted((int(c[j, k] - t0), f"{names[k]}({j})") for j in range(9, 14) for k in names)
        print(json.dumps({"timeline_rel_arrive10": ev}), flush=True)
    _lib.call("qcf_set_attention_kernel", 0)
    t = buf.view(n_cta, 8).cpu().numpy().astype(np.int64)
    sm, t1, t2, t3, t4, t5, t6, nt = (t[:, i] for i in range(8))
    span = (t6.max() - t1.min()) / 1e3
    gaps = []
    for s_ in np.unique(sm):
        idx = np.where(sm == s_)[0]
        idx = idx[np.argsort(t1[idx])]
        gaps += list((t1[idx[1:]] - t6[idx[:-1]]) / 1e3)
    main = (t4 - t3) / 1e3
    res = {"shape": name, "ctas": int(n_cta), "span_us": round(float(span), 1),
           "cta_us_mean": round(float(((t6 - t1) / 1e3).mean()), 2),
           "setup_us_mean": round(float(((t3 - t1) / 1e3).mean()), 2),
           "setup_to_sync_us": round(float(((t2 - t1) / 1e3).mean()), 2),
           "first_s_after_sync_us": round(float(((t3 - t2) / 1e3).mean()), 2),
           "main_us_mean": round(float(main.mean()), 2),
           "ns_per_key_tile": round(float(((t4 - t3) / np.maximum(nt - 1, 1)).mean()), 1),
           "epi_us_mean": round(float(((t6 - t4) / 1e3).mean()), 2),
           "epi_wait_pv_us": round(float(((t5 - t4) / 1e3).mean()), 2),
           "gap_us_mean": round(float(np.mean(gaps)), 2) if gaps else 0.0,
           "key_tiles_mean": round(float(nt.mean()), 1),
           "busy_frac": round(float(((t6 - t1) / 1e3).sum() / (span * len(np.unique(sm)))), 3)}
    print(json.dumps(res), flush=True)


run("llama batch8", 800, 5153, 32, 32, 8, sel_kmax(5120, 768, 32, 8))
run("llama single", 800, 5153, 32, 32, 1, sel_kmax(5120, 768, 32, 1))
run("llama-gqa batch8", 800, 5153, 32, 8, 8, sel_kmax(5120, 768, 32, 8))
