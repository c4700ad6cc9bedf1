"""Benchmark: QCFuse fused-prefill TTFT and requests/s at Llama-3-8B shape.

Contract (one JSON line from rank 0):
  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
A step = one fused prefill (assemble → probe → score → Top-N → selective
recompute + query rows → first-token logits) of one RAG request of
BASELINE.json configs[1]: random-init Llama-3-8B shape (L32 H32 D128 F14336,
reference architecture: LayerNorm, ReLU FFN, tied byte vocab 259), 10 chunks ×
512 tokens precomputed into the HBM chunk pool, 32-token query, 15% recompute.
`value` = requests/s over all ranks (device-resident inputs, CUDA-graph
replay); `e2e` = the same through the public `FusionEngine.fuse()` call with
host query tokens in and host logits/selection out. Under torchrun each rank
serves its own requests (weak scaling); results are gathered to rank 0 over
NCCL once per step. `--impl reference` times the CPU oracle port on a bounded
layer sample (rank 0 only).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    "llama3-8b": dict(n_layers=32, n_heads=32, d_model=4096, d_head=128, d_ff=14336,
                      n_chunks=10, chunk_len=512, q=32, ratio=0.15),
    "tiny": dict(n_layers=4, n_heads=4, d_model=256, d_head=64, d_ff=1024,
                 n_chunks=4, chunk_len=128, q=16, ratio=0.15),
}
METRIC = "fused-prefill TTFT (ms) and requests/s, Llama-3-8B shape, 1/2/4/8 B200"


def peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "_fallback": True}


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
            time.sleep(0.15)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.12)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU baseline: the oracle port on a bounded layer sample
# ---------------------------------------------------------------------------
def cpu_sample(cfgd: dict, chunk_kv_host, chunk_tokens, anchors, query, sample_layers: int) -> dict:
    """Time the oracle's fused path at full width over `sample_layers` layers
    and extrapolate each phase to the full stack (labelled as such)."""
    from oracle import qcfuse_oracle as O
    L = cfgd["n_layers"]
    oc = O.Config(n_layers=max(4, sample_layers), n_heads=cfgd["n_heads"], d_model=cfgd["d_model"],
                  d_head=cfgd["d_head"], d_ff=cfgd["d_ff"], seed=1234,
                  critical_layer=2 if max(4, sample_layers) >= 4 else None)
    w = O.init_weights(oc, layers=sample_layers)
    chunks = [O.Chunk(np.asarray(t), [O.KV(k[li], v[li], np.arange(k.shape[1])) for li in range(sample_layers)],
                      np.zeros(len(t), np.float32), np.asarray(a)) for t, (k, v), a in
              zip(chunk_tokens, chunk_kv_host, anchors)]
    t = {}
    t0 = time.perf_counter()
    # BOS row: computed once per engine in the reference (fusion.py:226), not per request
    bos = [O.KV(np.zeros((1, oc.n_heads, oc.d_head), np.float32), np.zeros((1, oc.n_heads, oc.d_head), np.float32),
                np.zeros(1, np.int64)) for _ in range(sample_layers)]
    fused = O.assemble(w, chunks, bos)
    t["assemble"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    pr = O.probe(w, chunks, fused, query, "anchors", bos, layers=sample_layers)
    t["probe"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    scores = O.score_against_keys(pr.queries[-1], fused.keys[sample_layers - 1][1:], oc.d_head)
    t["score"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    sel = O.select_topn(scores, cfgd["ratio"])
    t["select"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    upd = O.recompute(w, fused, sel)
    t["recompute"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    O.query_forward(w, upd, query)
    t["query_forward"] = time.perf_counter() - t0
    c = math.ceil(L / 2)
    scale = {"assemble": L / sample_layers, "probe": (c - 1) / sample_layers, "score": 1.0,
             "select": 1.0, "recompute": L / sample_layers, "query_forward": L / sample_layers}
    total = sum(t[k] * scale[k] for k in t)
    return {"phases_s": t, "sample_s": sum(t.values()), "extrapolated_request_s": total}


def cpu_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ---------------------------------------------------------------------------
def build_engine(cfgd, dtype, device):
    import torch
    import paper_2604_08585_b200 as Q
    cfg = Q.ModelConfig(n_layers=cfgd["n_layers"], n_heads=cfgd["n_heads"], d_model=cfgd["d_model"],
                        d_head=cfgd["d_head"], d_ff=cfgd["d_ff"], seed=1234)
    w = Q.init_weights(cfg, dtype=dtype, device=device)
    store = Q.ChunkStore(tempfile.mkdtemp(prefix="qcf-bench-"), cfg, dtype=dtype, device=device,
                         persist=False)
    toks = [np.random.default_rng(i).integers(0, 256, cfgd["chunk_len"]) for i in range(cfgd["n_chunks"])]
    ids = [store.precompute(w, t, 0.05, f"chunk{i}").chunk_id for i, t in enumerate(toks)]
    eng = Q.FusionEngine(w, store)
    torch.cuda.synchronize()
    return Q, cfg, w, store, eng, ids, toks


def phase_profile(eng, ids, query, policy, ratio):
    """Instrumented eager pass: CUDA events around every C-ABI launch."""
    import torch
    from paper_2604_08585_b200 import _lib
    _lib.profiler = _lib.Profiler()
    try:
        # park the GPU on a spin kernel so every launch below is queued before it
        # runs: the event pairs then bracket device time only, not host launch gaps
        torch.cuda._sleep(int(4e8))
        plan, b = eng.prefill(policy, ratio, ids, query, use_graph=False)
        torch.cuda.synchronize()
        recs = _lib.profiler.summary()
    finally:
        _lib.profiler = None
    return plan, b, recs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="llama3-8b", choices=sorted(CONFIGS))
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "f32"])
    ap.add_argument("--ratio", type=float, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-full", action="store_true", help="skip the full-prefill comparison")
    args = ap.parse_args()
    cfgd = dict(CONFIGS[args.config])
    if args.ratio is not None:
        cfgd["ratio"] = args.ratio
    args.warmup = max(args.warmup, 3)

    rank, world, local = (int(os.environ.get(k, d)) for k, d in (("RANK", 0), ("WORLD_SIZE", 1),
                                                                   ("LOCAL_RANK", 0)))
    if args.impl == "reference":
        return run_reference(args, cfgd, rank)

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=device)
    from paper_2604_08585_b200 import _lib
    from paper_2604_08585_b200.dist import gather_rows, max_over_ranks

    Q, cfg, w, store, eng, ids, chunk_toks = build_engine(cfgd, args.dtype, device)
    q = cfgd["q"]
    ratio = cfgd["ratio"]
    n_req = args.warmup + args.steps
    queries = [np.random.default_rng(10_000 + rank * 100_000 + r).integers(0, 256, q) for r in range(n_req)]
    qdev = torch.as_tensor(np.stack(queries).astype(np.int32), device=device)

    # graph capture + per-request query swap (inputs resident in HBM)
    plan, b = eng.prefill("QCFuse", ratio, ids, queries[0].tolist(), use_graph=True)
    n_ctx = plan.n_ctx
    qslice = slice(1 + n_ctx, 1 + n_ctx + q)
    stream = torch.cuda.current_stream()
    launches_per_step = None

    def step(i):
        b.tok[qslice].copy_(qdev[i], non_blocking=True)
        b.graph.replay()

    # count our kernels in one eager pass of the same plan (== graph nodes)
    c0 = _lib.launch_count
    eng._launch(plan, b)
    launches_per_step = _lib.launch_count - c0

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        for i in range(args.steps):
            step(args.warmup + i)
            if world > 1:
                res = torch.cat([b.logits[0], b.rc_pos[:plan.n_sel].float()])[None]
                gather_rows(res, world, world, rank)
        ev1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    dev_ms = ev0.elapsed_time(ev1)
    dev_ms = max_over_ranks(dev_ms, device)
    ms_per_step = dev_ms / args.steps
    value = world * args.steps / (dev_ms / 1e3)

    # ---- e2e through the public API (host tokens in, host logits out)
    e2e_times = []
    for i in range(args.warmup + args.steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        logits, sel = eng.fuse(queries[i].tolist(), ids, ratio)
        e1.record(stream)
        torch.cuda.synchronize()
        if i >= args.warmup:
            e2e_times.append(e0.elapsed_time(e1))
    e2e_ms = max_over_ranks(float(np.mean(e2e_times)), device)
    h2d = len(ids) * 32 + 4 * (1 + n_ctx + q) + 4 * plan.anchor_rows.size
    d2h = 4 * cfg.vocab_size + 4 * plan.n_sel

    # ---- instrumented pass: per-phase + dominant kernel (GEMM) roofline
    _, _, recs = phase_profile(eng, ids, queries[0].tolist(), "QCFuse", ratio)
    phases: dict[str, float] = {}
    gemm_flops = gemm_ms = 0.0
    n_gemm = 0
    gemm_shapes: dict[str, list] = {}
    for name, a, ms in recs:
        phases[name] = phases.get(name, 0.0) + ms
        if name in ("qcf_gemm", "qcf_gemm_ws", "qcf_gemm_qkv_rope"):
            if name == "qcf_gemm_qkv_rope":
                m_, k_, n_ = a[4], a[5], (a[6] + 2 * a[7]) * a[8]
            else:
                m_, n_, k_ = a[7], a[8], a[9]
            gemm_flops += 2.0 * m_ * n_ * k_
            gemm_ms += ms
            n_gemm += 1
            g = gemm_shapes.setdefault(f"{m_}x{n_}x{k_}", [0, 0.0, 2.0 * m_ * n_ * k_])
            g[0] += 1
            g[1] += ms
        if name == "qcf_attention":
            g = gemm_shapes.setdefault(f"attn m={a[5]} keys={a[9]}", [0, 0.0, 0.0])
            g[0] += 1
            g[1] += ms
    kernel_detail = {k: {"launches": v[0], "ms": round(v[1], 4),
                         "tflops": round(v[2] * v[0] / (v[1] / 1e3) / 1e12, 1) if v[2] else None}
                     for k, v in sorted(gemm_shapes.items(), key=lambda x: -x[1][1])}
    pk = peaks()
    achieved = gemm_flops / (gemm_ms / 1e3) / 1e12 if gemm_ms else None
    traffic = None
    tf = ROOT / "profiles" / "gemm_traffic.json"
    if tf.exists():
        try:
            traffic = json.loads(tf.read_text()).get("bytes_per_launch")
        except Exception:
            traffic = None
    roofline = {"bound": "tensor", "kernel": "qcf_gemm* family (tcgen05 bf16: 2-CTA/1-CTA/split-K, fused QKV+RoPE)",
                "achieved": achieved,
                "peak": pk["bf16_tflops"], "unit": "TFLOP/s",
                "frac": (achieved / pk["bf16_tflops"]) if achieved else None, "traffic": traffic,
                "launches_per_step": n_gemm, "share_of_step": gemm_ms / sum(phases.values()),
                "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst)" if not pk.get("_fallback")
                else "fallback"}

    # ---- full prefill on the same box (the TTFT denominator)
    full_ms = None
    if not args.no_full:
        fplan, fb = eng.prefill("FullCompute", 1.0, ids, queries[0].tolist(), use_graph=True)
        torch.cuda.synchronize()
        for _ in range(2):
            fb.graph.replay()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        nf = 3
        for _ in range(nf):
            fb.graph.replay()
        f1.record(stream)
        torch.cuda.synchronize()
        full_ms = f0.elapsed_time(f1) / nf
        del fb.graph
        eng._bufs.clear()

    # ---- CPU baseline (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_block(cfgd, store, ids, queries[0], sample_layers=2)

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": "requests/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "ttft_ms": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": args.dtype, "data": "synthetic (random-init weights, seeded byte tokens)",
            "config": {"workload": f"{args.config}: {cfgd['n_chunks']}x{cfgd['chunk_len']}-token chunks, "
                                   f"q={q}, recompute {ratio:.0%}, QCFuse",
                       "model": f"Llama-3-8B shape (L{cfg.n_layers} H{cfg.n_heads} D{cfg.d_head} "
                                f"F{cfg.d_ff}, reference arch)" if args.config == "llama3-8b" else args.config,
                       "n_ctx": n_ctx, "n_selected": plan.n_sel, "anchors": int(plan.anchor_rows.size - 1),
                       "requests_per_step_per_gpu": 1, "parallelism": f"replicas x{world} (request sharding)",
                       "l2": "inputs larger than L2 (11.8 GB weights + 2.7 GB chunk pool streamed per step)"},
            "e2e": {"value": world * 1e3 / e2e_ms, "unit": "requests/s", "ttft_ms": e2e_ms,
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": launches_per_step * args.steps,
            "roofline": roofline,
            "phases_ms": {k: round(v, 4) for k, v in sorted(phases.items(), key=lambda x: -x[1])},
            "kernels": kernel_detail,
            "full_prefill_ms": full_ms,
            "fused_over_full": (ms_per_step / full_ms) if full_ms else None,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


def cpu_baseline_block(cfgd, store, ids, query, sample_layers):
    recs = [store.get_record(c) for c in ids]
    kv = [(r.k[:sample_layers].float().cpu().numpy(), r.v[:sample_layers].float().cpu().numpy()) for r in recs]
    toks = [r.token_ids for r in recs]
    anchors = [r.anchor_indices for r in recs]
    t0 = time.perf_counter()
    res = cpu_sample(cfgd, kv, toks, anchors, query, sample_layers)
    return {"value": 1.0 / res["extrapolated_request_s"], "unit": "requests/s", "cores": cpu_cores(),
            "kind": "port",
            "sample": f"oracle numpy port, full Llama-3-8B width, {sample_layers} of {cfgd['n_layers']} layers "
                      f"of the fused path (10x512 ctx, q32, r .15), per-phase times extrapolated to "
                      f"{cfgd['n_layers']} layers (probe to c-1); BLAS threads = all host cores",
            "sample_seconds": round(res["sample_s"], 3),
            "extrapolated_request_s": round(res["extrapolated_request_s"], 3),
            "phases_s": {k: round(v, 4) for k, v in res["phases_s"].items()},
            "wall_s": round(time.perf_counter() - t0, 2)}


def run_reference(args, cfgd, rank):
    """CPU oracle port timed on the host (BASELINE.md §2 plan); rank 0 only."""
    if rank != 0:
        return
    from oracle import qcfuse_oracle as O
    L = cfgd["n_layers"]
    sample_layers = 1
    # chunk KV for the sample layers from the oracle itself (no GPU on this arm)
    oc = O.Config(n_layers=4, n_heads=cfgd["n_heads"], d_model=cfgd["d_model"], d_head=cfgd["d_head"],
                  d_ff=cfgd["d_ff"], seed=1234)
    w1 = O.init_weights(oc, layers=sample_layers)
    toks = [np.random.default_rng(i).integers(0, 256, cfgd["chunk_len"]) for i in range(cfgd["n_chunks"])]
    kv, anchors = [], []
    for t in toks:
        tr = O.forward(w1, t, np.arange(t.size), None, layers=sample_layers)
        k = np.stack([x.keys for x in tr.kv])
        v = np.stack([x.values for x in tr.kv])
        norms = np.linalg.norm(k[0], axis=2).mean(axis=1)
        kv.append((k, v))
        anchors.append(O.extract_anchors(norms, 0.05))
    times = []
    for i in range(args.warmup + args.steps):
        qt = np.random.default_rng(10_000 + i).integers(0, 256, cfgd["q"])
        r = cpu_sample(cfgd, kv, toks, anchors, qt, sample_layers)
        if i >= args.warmup:
            times.append(r["extrapolated_request_s"])
    per = float(np.mean(times))
    out = {"metric": METRIC, "impl": "reference", "value": 1.0 / per, "unit": "requests/s", "n_gpus": 1,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": per * 1e3, "ttft_ms": per * 1e3,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
           "data": "synthetic", "config": {"workload": f"{args.config}: {cfgd['n_chunks']}x{cfgd['chunk_len']}, "
                                                       f"q={cfgd['q']}, recompute {cfgd['ratio']:.0%}, QCFuse"},
           "cpu_baseline": {"value": 1.0 / per, "unit": "requests/s", "cores": cpu_cores(), "kind": "port",
                            "sample": f"oracle numpy port, full width, {sample_layers} of {L} layers per phase, "
                                      f"extrapolated to {L} layers"},
           "e2e": {"value": 1.0 / per, "unit": "requests/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
