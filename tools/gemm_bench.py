"""Time qcf_gemm (tcgen05) on the fused-path shapes; prints TFLOP/s per shape."""
import sys, json
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import os
from paper_2604_08585_b200 import _lib
from paper_2604_08585_b200.model import tile64
LAY = int(os.environ.get("QCF_TILED", "1"))  # 1 = tile-major weights (production layout)

SHAPES = [  # (m, n, k, epi, name)
    (800, 12288, 4096, 0, "qkv M=800"), (800, 4096, 4096, 2, "wo M=800"),
    (800, 14336, 4096, 1, "w1 M=800"), (800, 4096, 14336, 2, "w2 M=800"),
    (32, 12288, 4096, 0, "qkv M=32"), (32, 14336, 4096, 1, "w1 M=32"), (32, 4096, 14336, 2, "w2 M=32"),
    (5153, 12288, 4096, 0, "qkv M=5153"), (5153, 14336, 4096, 1, "w1 M=5153"),
    (8192, 8192, 8192, 0, "square 8192"),
]
res = []
s = torch.cuda.current_stream().cuda_stream
for m, n, k, epi, name in SHAPES:
    a = (torch.randn(m, k, device="cuda") * 0.5).bfloat16()
    b = (torch.randn(n, k, device="cuda") * 0.05).bfloat16()
    b = tile64(b) if LAY else b
    out_dt = _lib.QCF_BF16 if epi == 1 else _lib.QCF_F32
    c = torch.zeros(m, n, device="cuda", dtype=torch.bfloat16 if epi == 1 else torch.float32)
    ws = torch.zeros(max(int(_lib.lib.qcf_gemm_workspace(m, n, k)), 16), dtype=torch.uint8, device="cuda")
    f = lambda: _lib.call("qcf_gemm_ws", _lib.QCF_BF16, a.data_ptr(), k, b.data_ptr(), k, c.data_ptr(), n, m, n, k, epi, out_dt, LAY, ws.data_ptr(), ws.numel(), s)
    for _ in range(3): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    it = 20
    # graph-captured so host launch cost does not hide the device time
    side = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        sc = side.cuda_stream
        for _ in range(it):
            _lib.call("qcf_gemm_ws", _lib.QCF_BF16, a.data_ptr(), k, b.data_ptr(), k, c.data_ptr(), n, m, n, k, epi,
                      out_dt, LAY, ws.data_ptr(), ws.numel(), sc)
    g.replay(); torch.cuda.synchronize()
    e0.record()
    g.replay()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / it
    # cold-L2 variant: flush L2 (256 MB write) before each call
    flush = torch.empty(256 * 1024 * 1024 // 4, device="cuda")
    cold = []
    for _ in range(5):
        flush.fill_(1.0)
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(int(2e7))
        c0.record(); f(); c1.record(); torch.cuda.synchronize()
        cold.append(c0.elapsed_time(c1))
    cold_ms = sorted(cold)[len(cold) // 2]
    tf = 2 * m * n * k / ms / 1e9
    # torch reference speed for context
    bt = b.t()
    g = lambda: torch.matmul(a, bt)
    for _ in range(3): g()
    torch.cuda.synchronize(); e0.record()
    for _ in range(it): g()
    e1.record(); torch.cuda.synchronize()
    tms = e0.elapsed_time(e1) / it
    res.append({"shape": name, "ms": round(ms, 4), "tflops": round(tf, 1), "cold_ms": round(cold_ms, 4),
                "cold_hbm_gbs": round((n * k * 2 + m * k * 2) / cold_ms / 1e6, 0), "cublas_ms": round(tms, 4),
                "cublas_tflops": round(2 * m * n * k / tms / 1e9, 1)})
    print(json.dumps(res[-1]), flush=True)
