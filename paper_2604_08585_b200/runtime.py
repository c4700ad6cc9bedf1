"""The decoder layer stack as a sequence of C-ABI kernel launches.

One executor serves every hot-path forward of the reference:
  * selective recompute + query rows (fusion.py:446-490 fused with 536-540),
  * the anchor probe (fusion.py:269-311 → model.py:403-424),
  * chunk precompute / full prefill (model.py:391-400), decode steps (433-465).
Each is "M rows at positions `pos`, writing their fresh K/V into table rows
`dst`, attending to table rows 0..kmax[i]" (model.py:345-388 with the mask of
fusion.py:467). Launches only — no host synchronisation — so a whole request
can be captured into a CUDA graph.
"""

from __future__ import annotations

import os
import threading
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import EPI_ADD_F32, EPI_RELU, EPI_STORE, QCF_F32, call
from .model import ModelWeights, RopeTable, cuda_stream


@dataclass
class Scratch:
    """Per-M activations (fixed addresses once allocated; graph friendly)."""
    cap: int
    x: torch.Tensor      # f32 [cap, d] residual stream
    a: torch.Tensor      # dt  [cap, d] LN output (GEMM A operand)
    qkv: torch.Tensor    # f32 [cap, (H+2Hkv)D]
    q: torch.Tensor      # dt  [cap, H, D] rotated queries
    o: torch.Tensor      # dt  [cap, H*D] attention output
    hid: torch.Tensor    # dt  [cap, F]   relu(W1 x)
    ws: torch.Tensor     # u8  GEMM workspace: stream-K flags/partials + skinny split-K partials
    delta: torch.Tensor  # f32 [cap, d] projection output awaiting its residual add
    pending: bool = False  # delta not yet added into x (launch-sequencing state)


class Executor:
    def __init__(self, weights: ModelWeights, rope: RopeTable | None = None):
        self.w = weights
        self.cfg = weights.config
        self.rope = rope or RopeTable(self.cfg.d_head, self.cfg.rope_theta, weights.device)
        self._scratch: dict[int, Scratch] = {}
        self._aws: dict[tuple, torch.Tensor] = {}
        # the scratch / workspaces are shared by every engine on these weights: one
        # request at a time runs through them (the reference engine is re-entrant,
        # fusion.py:211-216, so concurrent Python threads must be safe)
        self.lock = threading.RLock()
        self.residual_in_epilogue = os.environ.get("QCF_RESID_EPI", "1") == "1"
        # fused QKV+RoPE epilogue: bf16 on a tcgen05 device, head dim a multiple of 32
        self.fused_qkv = (weights.dtype == "bf16" and self.cfg.d_head % 32 == 0
                          and torch.cuda.is_available() and bool(_lib.lib.qcf_tc_available()))

    # ------------------------------------------------------------------
    def scratch(self, m: int, key=None) -> Scratch:
        """Scratch with capacity >= m; `key` separates independent users (graphs)."""
        k = key if key is not None else "default"
        s = self._scratch.get(k)
        if s is None or s.cap < m:
            cfg, dev, dt = self.cfg, self.w.device, self.w.torch_dtype
            cap = max(m, 16)
            H, Hkv, D = cfg.n_heads, cfg.n_kv_heads, cfg.d_head
            d, F = cfg.d_model, cfg.d_ff
            ws_bytes = max(int(_lib.lib.qcf_gemm_workspace(cap, n, k))
                           for n, k in (((H + 2 * Hkv) * D, d), (d, H * D), (F, d), (d, F)))
            s = Scratch(cap,
                        torch.empty(cap, cfg.d_model, dtype=torch.float32, device=dev),
                        torch.empty(cap, cfg.d_model, dtype=dt, device=dev),
                        torch.empty(cap, (H + 2 * Hkv) * D, dtype=torch.float32, device=dev),
                        torch.empty(cap, H, D, dtype=dt, device=dev),
                        torch.empty(cap, H * D, dtype=dt, device=dev),
                        torch.empty(cap, cfg.d_ff, dtype=dt, device=dev),
                        # zero-filled once: the stream-K flag words must start at 0 (qcf_gemm_ws)
                        torch.zeros(max(ws_bytes, 16), dtype=torch.uint8, device=dev),
                        torch.empty(cap, cfg.d_model, dtype=torch.float32, device=dev))
            self._scratch[k] = s
        return s

    def _attn_ws(self, m_per_req: int, n_req: int, n_keys: int) -> torch.Tensor | None:
        """Split-KV workspace of the attention (only for grids far below one wave)."""
        if self.w.dtype != "bf16":
            return None
        n = int(_lib.lib.qcf_attention_workspace(m_per_req, n_req, self.cfg.n_heads, n_keys))
        if n == 0:
            return None
        t = self._aws.get((m_per_req, n_req, n_keys))
        if t is None:
            t = torch.empty(n, dtype=torch.uint8, device=self.w.device)
            self._aws[(m_per_req, n_req, n_keys)] = t
        return t

    # ------------------------------------------------------------------
    def embed(self, sc: Scratch, m: int, tokens: torch.Tensor, rows: torch.Tensor | None = None,
              row_base: int = 0, stream=None) -> None:
        call("qcf_embed", tokens.data_ptr(), rows.data_ptr() if rows is not None else None,
             row_base, m, self.w.emb.data_ptr(), self.cfg.d_model, sc.x.data_ptr(),
             cuda_stream(stream))
        sc.pending = False

    def _norm(self, sc: Scratch, m: int, g, b, s) -> None:
        """a = LN(x), first folding a pending projection output into x
        (the residual adds of model.py:375-376, fused into the LayerNorm)."""
        call("qcf_add_layernorm", sc.x.data_ptr(), sc.delta.data_ptr() if sc.pending else None, m,
             self.cfg.d_model, g.data_ptr(), b.data_ptr(), self.cfg.ln_eps, sc.a.data_ptr(),
             self.w.qcf_dtype, s)
        sc.pending = False

    def flush(self, sc: Scratch, m: int, stream=None) -> None:
        """Make x current (apply a pending residual add)."""
        if sc.pending:
            call("qcf_add_rows", sc.x.data_ptr(), sc.delta.data_ptr(), m * self.cfg.d_model,
                 cuda_stream(stream))
            sc.pending = False

    def gemm(self, sc: Scratch, a, lda, b, ldb, c, ldc, m, n, k, epi, out_dt, s) -> None:
        """qcf_gemm_ws: tcgen05 (2-CTA / 1-CTA / split-K skinny) for bf16, FFMA for f32."""
        call("qcf_gemm_ws", self.w.qcf_dtype, a.data_ptr(), lda, b.data_ptr(), ldb, c.data_ptr(), ldc,
             m, n, k, epi, out_dt, self.w.b_layout, sc.ws.data_ptr(), sc.ws.numel(), s)

    def _project(self, sc: Scratch, a, lda, w, m: int, k: int, s) -> None:
        """x += a @ w (model.py:375-376). The residual add runs in the GEMM
        epilogue (read-modify-write of x, one f32 add per element: the same
        arithmetic as adding it later), so the LayerNorm that follows reads x
        alone (6 instead of 14 bytes per element) -- residual_in_epilogue
        (default; QCF_RESID_EPI=0 turns it off). The swapped kernel's epilogue
        issues all 32 residual loads of a row group before its stores (they were
        serialised: W_o at M = 800 took 119 us). A/B on one box (r2s3,
        profiles/r2s3_resid_epi_ab.txt, two pairs): LayerNorm 4.39 -> 3.0-3.2 ms
        per batch and 1.10 -> 0.95 ms per request, 88.4/89.3 -> 89.8/89.4 req/s,
        TTFT 13.50/13.48 -> 13.42/13.44 ms. Off: the projection goes to `delta`
        and the add folds into the next LayerNorm."""
        d = self.cfg.d_model
        if self.residual_in_epilogue:
            self.gemm(sc, a, lda, w, lda, sc.x, d, m, d, k, EPI_ADD_F32, QCF_F32, s)
        else:
            self.gemm(sc, a, lda, w, lda, sc.delta, d, m, d, k, EPI_STORE, QCF_F32, s)
            sc.pending = True

    def layer(self, li: int, sc: Scratch, m: int, pos: torch.Tensor, dst: torch.Tensor,
              kmax: torch.Tensor, tab_k: torch.Tensor, tab_v: torch.Tensor,
              q_only: bool = False, q_out: torch.Tensor | None = None, stream=None,
              n_req: int = 1) -> None:
        """One decoder layer (model.py:359-376) over m rows.

        tab_k/tab_v: [n_rows, Hkv, D] views of THIS layer's table. With q_only
        the layer stops after LN1 → QKV → RoPE (the probe's critical-layer Q).
        n_req > 1: a homogeneous batch — rows are n_req blocks of m/n_req, the
        table n_req blocks of n_rows/n_req; `dst` indexes the whole table,
        `kmax` is relative to the row's own block."""
        cfg, w = self.cfg, self.w
        lw = w.layers[li]
        d, H, Hkv, D, F = cfg.d_model, cfg.n_heads, cfg.n_kv_heads, cfg.d_head, cfg.d_ff
        dt = w.qcf_dtype
        s = cuda_stream(stream)
        nq = (H + 2 * Hkv) * D
        self._norm(sc, m, lw.ln1_g, lw.ln1_b, s)
        qdst = q_out if q_out is not None else sc.q
        if self.fused_qkv:
            # bf16: projection + RoPE + KV scatter in one tcgen05 kernel epilogue (M <= 256:
            # cluster split-K weight streaming with the rotation applied in the reduction)
            call("qcf_gemm_qkv_rope", sc.a.data_ptr(), d, lw.wqkv.data_ptr(), d, self.w.b_layout, m, d, H, Hkv, D,
                 pos.data_ptr(), dst.data_ptr(), self.rope.cs32.data_ptr(),
                 self.rope.n_pos, qdst.data_ptr(), tab_k.data_ptr(), tab_v.data_ptr(), sc.ws.data_ptr(), sc.ws.numel(), s)
        else:
            self.gemm(sc, sc.a, d, lw.wqkv, d, sc.qkv, nq, m, nq, d, EPI_STORE, QCF_F32, s)
            call("qcf_rope_qkv_scatter", sc.qkv.data_ptr(), m, H, Hkv, D, pos.data_ptr(),
                 dst.data_ptr(), self.rope.cos.data_ptr(), self.rope.sin.data_ptr(), self.rope.n_pos,
                 qdst.data_ptr(), tab_k.data_ptr(), tab_v.data_ptr(), dt, s)
        if q_only:
            return
        aws = self._attn_ws(m // n_req, n_req, tab_k.shape[0] // n_req)
        call("qcf_attention_batched_ws", dt, qdst.data_ptr(), tab_k.data_ptr(), tab_v.data_ptr(),
             kmax.data_ptr(), m // n_req, n_req, H, Hkv, D, tab_k.shape[0] // n_req, sc.o.data_ptr(),
             aws.data_ptr() if aws is not None else None, aws.numel() if aws is not None else 0, s)
        self._project(sc, sc.o, H * D, lw.wo, m, H * D, s)
        self._norm(sc, m, lw.ln2_g, lw.ln2_b, s)
        self.gemm(sc, sc.a, d, lw.w1, d, sc.hid, F, m, F, d, EPI_RELU, dt, s)
        self._project(sc, sc.hid, F, lw.w2, m, F, s)

    def stack(self, sc: Scratch, m: int, pos, dst, kmax, tab_k: torch.Tensor, tab_v: torch.Tensor,
              layers: range | None = None, q_store: torch.Tensor | None = None, stream=None,
              n_req: int = 1, before_layer=None) -> None:
        """Run layers over m rows. tab_k/tab_v: [L, n_rows, Hkv, D].
        q_store (optional) [L, m, H, D] receives each layer's rotated Q.
        before_layer(li) (optional) runs before layer li is enqueued (stream waits)."""
        layers = range(self.cfg.n_layers) if layers is None else layers
        for li in layers:
            if before_layer is not None:
                before_layer(li)
            self.layer(li, sc, m, pos, dst, kmax, tab_k[li], tab_v[li],
                       q_out=q_store[li] if q_store is not None else None, stream=stream, n_req=n_req)
        self.flush(sc, m, stream)

    def lm_head(self, sc: Scratch, rows: torch.Tensor, out: torch.Tensor, stream=None) -> None:
        """logits[r] = LN_f(x[rows[r]]) @ embᵀ (model.py:384-385)."""
        cfg = self.cfg
        call("qcf_lm_head", sc.x.data_ptr(), rows.data_ptr(), rows.numel(), cfg.d_model,
             self.w.ln_f_gain.data_ptr(), self.w.ln_f_bias.data_ptr(), cfg.ln_eps,
             self.w.emb.data_ptr(), cfg.vocab_size, out.data_ptr(), cuda_stream(stream))

    # ------------------------------------------------------------------
    def new_table(self, n_rows: int, n_layers: int | None = None) -> tuple[torch.Tensor, torch.Tensor]:
        cfg = self.cfg
        shape = (cfg.n_layers if n_layers is None else n_layers, n_rows, cfg.n_kv_heads, cfg.d_head)
        return (torch.empty(shape, dtype=self.w.torch_dtype, device=self.w.device),
                torch.empty(shape, dtype=self.w.torch_dtype, device=self.w.device))

    def forward_full_batch(self, tokens: torch.Tensor, stream=None, layers: range | None = None):
        """forward_full of B equal-length sequences at once: tokens [B][m] ->
        tables [L][B*m][Hkv][D] (sequence b owns rows b*m..), one layer stack
        with the batched attention (n_req = B). Every row's arithmetic is the
        one forward_full does for it alone (per-row GEMM accumulation order and
        attention are independent of the batch)."""
        B, m = tokens.shape
        self.rope.ensure(m + 1)
        dev = self.w.device
        tk, tv = self.new_table(B * m, None if layers is None else len(layers))
        ar = torch.arange(m, dtype=torch.int32, device=dev)
        pos = ar.repeat(B)
        dst = torch.arange(B * m, dtype=torch.int32, device=dev)
        sc = self.scratch(B * m, key=("full_batch", B * m))
        self.embed(sc, B * m, tokens.reshape(-1), stream=stream)
        self.stack(sc, B * m, pos, dst, pos, tk, tv, stream=stream, n_req=B, layers=layers)
        return tk, tv

    def forward_full(self, tokens: torch.Tensor, start: int = 0, tab=None, want_logits_rows=None,
                     stream=None, layers: range | None = None):
        """Full causal forward of `tokens` at positions start.. (model.py:391-400).
        Returns (table K, table V, x scratch). Table row i = token i.
        `layers` = range(n) runs layers 1..n only (tables hold n layers)."""
        m = tokens.numel()
        self.rope.ensure(start + m + 1)
        dev = self.w.device
        tk, tv = tab if tab is not None else self.new_table(m, None if layers is None else len(layers))
        ar = torch.arange(m, dtype=torch.int32, device=dev)
        pos = ar + start
        sc = self.scratch(m, key=("full", m))
        self.embed(sc, m, tokens, stream=stream)
        self.stack(sc, m, pos, ar, ar, tk, tv, stream=stream, layers=layers)
        return tk, tv, sc
