"""B200-native QCFuse fusion engine behind the reference's `FusionEngine` API
(fusion.py:211-563).

Hot path (`FusionEngine.fuse` / `run("QCFuse", …)`), all on one CUDA stream,
no host synchronisation between kernels:

  K1 qcf_assemble          fused table = [BOS | R(off_c)·K_c …], V copied     fusion.py:234-263
  K2 qcf_assemble_rot      probe past = [BOS | R(off_c)·anchor rows] for layers < c, from the
                           chunks' HBM-resident anchor copies; K1 runs concurrently on a
                           forked stream (both are HBM-bound, no data dependence) and joins
                           before K4                                           fusion.py:281-303
  K3 layer stack (q rows)  LN→QKV→RoPE→attn→Wo→LN→FFN for layers 1..c-1, then
                           layer c's LN→Wq→RoPE = Q_c                          fusion.py:305-311
  K4 qcf_score             softmax over context keys, mean over (h,t)         fusion.py:313-326
  K5 qcf_topn              stable Top-N, ties → lower index, ascending        fusion.py:148-158
  K6 layer stack (N+q rows) selected rows re-embedded, K/V scattered into the
                           fused table in place, location-aware attention;
                           the query rows ride in the same pass              fusion.py:446-490, 536-540
     qcf_lm_head           LN_f + tied lm-head on the last query row         fusion.py:540

The reference-shaped objects (`FusedContext.layer_kv`, `QueryProbe.queries`,
`SelectionResult.indices`, `RunResult.first_logits` …) materialise host numpy
lazily, only when a caller reads them.
"""

from __future__ import annotations

import ctypes
import functools
import math
import os
import time
import weakref
from collections import OrderedDict
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import ChunkDesc, call
from .model import (BOS_ID, EOS_ID, ModelWeights, byte_tokens, cuda_stream, render_tokens)
from .pipeline import CostModel, ScheduleTrace, layer_times, policy_schedule, schedule_events
from .runtime import Executor
from .store import ChunkStore, HostLayerKV

POLICIES = ("FullCompute", "FullReuse", "Random", "EPIC", "CacheBlend",
            "KVShare", "QCLast", "QCAll", "QCFuse")
PROBE_ANCHORS = "anchors"
PROBE_FULL = "full"
PROBE_NONE = "none"

_EXECUTORS: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


def _executor_for(weights: ModelWeights) -> Executor:
    ex = _EXECUTORS.get(weights)
    if ex is None:
        ex = Executor(weights)
        _EXECUTORS[weights] = ex
    return ex


def _serialized(fn):
    """Run an engine method under its executor's lock (shared device buffers)."""
    @functools.wraps(fn)
    def wrapper(self, *args, **kwargs):
        with self.ex.lock:
            return fn(self, *args, **kwargs)
    return wrapper


class _DescView:
    """Byte-offset view of a device descriptor array (for per-request launches)."""

    def __init__(self, t: torch.Tensor, offset: int):
        self._p = t.data_ptr() + offset

    def data_ptr(self) -> int:
        return self._p


def _view_rows(t: torch.Tensor, row0: int) -> _DescView:
    """Pointer to row `row0` of layer 0 of a [L][rows][Hkv][D] table."""
    return _DescView(t, row0 * t.stride(1) * t.element_size())


def _i32(a, device) -> torch.Tensor:
    return torch.as_tensor(np.ascontiguousarray(np.asarray(a, dtype=np.int32)), device=device)


# ---------------------------------------------------------------------------
# result types (fusion.py:62-138)
# ---------------------------------------------------------------------------

class _LazyLayers:
    """Sequence of HostLayerKV over a device table, copied per layer on access."""

    def __init__(self, k: torch.Tensor, v: torch.Tensor, n_rows: int):
        self._k, self._v, self._n = k, v, n_rows
        self._cache: dict[int, HostLayerKV] = {}

    def __len__(self):
        return self._k.shape[0]

    def __getitem__(self, li):
        if isinstance(li, slice):
            return [self[i] for i in range(len(self))[li]]
        if li < 0:
            li += len(self)
        if li not in self._cache:
            self._cache[li] = HostLayerKV(self._k[li, :self._n].float().cpu().numpy(),
                                          self._v[li, :self._n].float().cpu().numpy(), 0)
        return self._cache[li]

    def __iter__(self):
        return (self[i] for i in range(len(self)))


@dataclass
class FusedContext:
    chunk_ids: list[str]
    token_ids: np.ndarray
    offsets: list[int]
    n_ctx: int
    chunk_index: np.ndarray
    k: torch.Tensor            # [L][cap][Hkv][D] device table (rows 0..n_ctx valid)
    v: torch.Tensor
    _layers: _LazyLayers | None = field(default=None, repr=False)

    @property
    def layer_kv(self) -> _LazyLayers:
        if self._layers is None:
            self._layers = _LazyLayers(self.k, self.v, self.n_ctx + 1)
        return self._layers

    def key_positions(self) -> np.ndarray:
        return np.arange(0, self.n_ctx + 1, dtype=np.int64)

    def copy_kv(self) -> list[HostLayerKV]:
        return [kv.copy() for kv in self.layer_kv]

    def clone(self, extra_rows: int = 0) -> "FusedContext":
        L, cap, Hkv, D = self.k.shape
        rows = max(cap, self.n_ctx + 1 + extra_rows)
        k = torch.empty((L, rows, Hkv, D), dtype=self.k.dtype, device=self.k.device)
        v = torch.empty_like(k)
        k[:, :self.n_ctx + 1].copy_(self.k[:, :self.n_ctx + 1])
        v[:, :self.n_ctx + 1].copy_(self.v[:, :self.n_ctx + 1])
        return FusedContext(list(self.chunk_ids), self.token_ids, list(self.offsets), self.n_ctx,
                            self.chunk_index, k, v)


@dataclass
class QueryProbe:
    query_tokens: np.ndarray
    positions: np.ndarray
    q_store: torch.Tensor              # [layers_run][q][H][D] rotated queries
    prefix_positions: np.ndarray
    _crit_tab: tuple | None = field(default=None, repr=False)   # (k, v, n_prefix) at layer c
    _crit_layer: int = 0
    _queries: list | None = field(default=None, repr=False)

    @property
    def queries(self) -> list[np.ndarray]:
        if self._queries is None:
            self._queries = [self.q_store[i].float().cpu().numpy() for i in range(self.q_store.shape[0])]
        return self._queries

    @property
    def critical_attention(self) -> np.ndarray:
        """[H, q, n_prefix] probe attention over the prefix at the critical layer
        (fusion.py:308-311). Diagnostic field; computed on demand on the device."""
        tk, tv, n_pre = self._crit_tab
        q = self.q_store[self._crit_layer - 1].float()            # [q, H, D]
        nq, H, D = q.shape
        keys = tk[: n_pre + nq].float()                            # [n, Hkv, D]
        rep = H // keys.shape[1]
        keys = keys.repeat_interleave(rep, dim=1)
        s = torch.einsum("mhd,nhd->hmn", q, keys) / math.sqrt(D)
        mask = torch.ones(nq, n_pre + nq, dtype=torch.bool, device=q.device)
        mask[:, n_pre:] = torch.tril(torch.ones(nq, nq, dtype=torch.bool, device=q.device))
        s = s.masked_fill(~mask[None], float("-inf"))
        return torch.softmax(s, dim=-1)[:, :, :n_pre].cpu().numpy()


@dataclass
class SelectionResult:
    policy: str
    ratio: float
    indices: np.ndarray
    scores: np.ndarray

    @property
    def n_selected(self) -> int:
        return int(self.indices.size)


@dataclass
class RecomputeTrace:
    updated_indices: np.ndarray
    fetch_seconds: list[float]
    compute_seconds: list[float]
    events: list[dict] = field(default_factory=list)


@dataclass
class OracleComparison:
    logit_div_max: float
    logit_kl: float
    token_match: float
    overlap: float


@dataclass
class RunResult:
    policy: str
    ratio: float
    answer_tokens: list[int]
    answer_text: str
    first_logits: np.ndarray
    selection: SelectionResult
    trace: RecomputeTrace
    schedule: ScheduleTrace
    ttft_sim: float
    comparison: OracleComparison | None = None
    timings_ms: dict = field(default_factory=dict)


@dataclass
class RunOptions:
    max_new: int = 32
    query_agg: str = "mean"
    selection_seed: int = 0
    epic_per_chunk: bool = False
    qcall_layer_average: bool = False
    # float64 SIMT scoring (the fp32 parity scoring mode) or tcgen05 bf16 scoring
    # (speed mode); None = precise for f32 weights, tensor cores for bf16
    score_precise: bool | None = None


# ---------------------------------------------------------------------------
# module-level ops (fusion.py:141-208)
# ---------------------------------------------------------------------------

def n_select(ratio: float, n_ctx: int) -> int:
    """N = ceil(ratio * n_ctx) in Python double (fusion.py:155)."""
    if not (0.0 <= ratio <= 1.0):
        raise ValueError("ratio must be in [0, 1]")
    return math.ceil(ratio * n_ctx)


def topn_device(scores: torch.Tensor, n: int, base: int = 1, out: torch.Tensor | None = None,
                stream=None) -> torch.Tensor:
    """Ascending (base-offset) indices of the n largest scores, ties → lower
    index, via the `qcf_topn` kernel."""
    m = scores.numel()
    out = out if out is not None else torch.empty(max(n, 1), dtype=torch.int32, device=scores.device)
    call("qcf_topn", scores.data_ptr(), m, n, base, out.data_ptr(), None, 0, cuda_stream(stream))
    return out[:n]


def _topn_f64(scores, n: int) -> np.ndarray:
    """Ascending 1-based positions of the n largest float64 scores on the
    device (`qcf_topn_f64`): the order of np.argsort(-float64, stable) --
    ties and ±0 toward the lower index, NaN last -- with no float32 rounding."""
    s = np.ascontiguousarray(np.asarray(scores, dtype=np.float64).reshape(-1))
    n = int(n)
    if not (0 <= n <= s.size):
        raise ValueError("n must be in [0, len(scores)]")
    if n == 0:
        return np.zeros(0, np.int64)
    ts = torch.as_tensor(s, device="cuda")
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    call("qcf_topn_f64", ts.data_ptr(), s.size, n, 1, out.data_ptr(), cuda_stream())
    return out.cpu().numpy().astype(np.int64)


def top_n_positions(scores, n: int) -> np.ndarray:
    """fusion.py:141-145 on the device (float64 keys)."""
    return _topn_f64(scores, n)


def select_topn(scores, ratio: float, policy: str = "QCFuse") -> SelectionResult:
    """fusion.py:148-158: N = ceil(ratio·n_ctx), float64 ranking, ties toward
    the lower index, ascending output; scores returned as float32 like the
    reference's SelectionResult."""
    if not (0.0 <= ratio <= 1.0):
        raise ValueError("ratio must be in [0, 1]")
    s = np.asarray(scores, dtype=np.float64)
    n = n_select(ratio, s.size)
    return SelectionResult(policy, ratio, _topn_f64(s, n), s.astype(np.float32))


def epic_select(n_ctx: int, ratio: float, chunk_spans=None) -> SelectionResult:
    """Static prefix selection (fusion.py:161-177); host-side index list."""
    if not (0.0 <= ratio <= 1.0):
        raise ValueError("ratio must be in [0, 1]")
    if chunk_spans is None:
        idx = np.arange(1, math.ceil(ratio * n_ctx) + 1, dtype=np.int64)
    else:
        picks = []
        for start, length in chunk_spans:
            picks.extend(range(start, start + math.ceil(ratio * length)))
        idx = np.asarray(sorted(picks), dtype=np.int64)
    return SelectionResult("EPIC", ratio, idx, np.zeros(n_ctx, np.float32))


def _splitmix_next_below(state: int, n: int) -> tuple[int, int]:
    m = (1 << 64) - 1
    state = (state + 0x9E3779B97F4A7C15) & m
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    return state, (z ^ (z >> 31)) % n


def random_select(seed: int, n_ctx: int, ratio: float) -> SelectionResult:
    """Seeded Fisher-Yates over 1..n_ctx (fusion.py:180-191)."""
    if not (0.0 <= ratio <= 1.0):
        raise ValueError("ratio must be in [0, 1]")
    n = math.ceil(ratio * n_ctx)
    arr = list(range(1, n_ctx + 1))
    st = seed & ((1 << 64) - 1)
    for i in range(n_ctx - 1, 0, -1):
        st, j = _splitmix_next_below(st, i + 1)
        arr[i], arr[j] = arr[j], arr[i]
    return SelectionResult("Random", ratio, np.asarray(sorted(arr[:n]), dtype=np.int64),
                           np.zeros(n_ctx, np.float32))


def sparse_attention(q, positions, keys, values, visible) -> np.ndarray:
    """Attention of scattered rows over a KV table (fusion.py:194-208) on the
    device, for ANY visibility mask: prefix masks (row i sees keys 0..kmax[i],
    what the fused path produces) run on the location-aware kernel, other masks
    on `qcf_attention_masked` with the mask packed to bits. Same errors as the
    reference (ValueError on a shape mismatch or a row with no visible key)."""
    q = np.asarray(q, np.float32)
    keys = np.asarray(keys, np.float32)
    values = np.asarray(values, np.float32)
    visible = np.asarray(visible, bool)
    if visible.shape != (q.shape[0], keys.shape[0]):
        raise ValueError("visibility mask shape mismatch")
    if not visible.any(axis=1).all():
        raise ValueError("every query row needs at least one visible key")
    m, H, D = q.shape
    n = keys.shape[0]
    kmax = n - 1 - np.argmax(visible[:, ::-1], axis=1)
    prefix = np.arange(n)[None, :] <= kmax[:, None]
    dev = torch.device("cuda")
    tq = torch.as_tensor(q, device=dev)
    tk = torch.as_tensor(keys, device=dev)
    tv = torch.as_tensor(values, device=dev)
    out = torch.empty_like(tq)
    if np.array_equal(prefix, visible):
        call("qcf_attention", _lib.QCF_F32, tq.data_ptr(), tk.data_ptr(), tv.data_ptr(),
             _i32(kmax, dev).data_ptr(), m, H, keys.shape[1], D, n, out.data_ptr(), cuda_stream())
    else:
        words = (n + 31) // 32
        bits = np.zeros((m, words * 32), bool)
        bits[:, :n] = visible
        packed = np.packbits(bits.reshape(m, words, 4, 8), axis=3, bitorder="little").reshape(m, words * 4)
        mask = torch.as_tensor(np.ascontiguousarray(packed).view(np.uint32), device=dev)
        call("qcf_attention_masked", _lib.QCF_F32, tq.data_ptr(), tk.data_ptr(), tv.data_ptr(),
             _i32(kmax, dev).data_ptr(), mask.data_ptr(), words, m, H, keys.shape[1], D, n, out.data_ptr(),
             cuda_stream())
    return out.cpu().numpy()


# ---------------------------------------------------------------------------
# request plan + device buffers of the fused fast path
# ---------------------------------------------------------------------------

@dataclass
class _Plan:
    """One request's host-side plan (chunk records, offsets, probe rows)."""
    chunk_ids: list[str]
    records: list
    offsets: list[int]
    n_ctx: int
    q: int
    n_sel: int
    anchor_rows: np.ndarray      # [1 + A] fused rows of the probe prefix
    policy: str

    def shape_key(self):
        return (tuple(r.n_tokens for r in self.records), self.q, self.n_sel, self.anchor_rows.size, self.policy)


class _Bufs:
    """Device buffers for a batch of B requests (fixed addresses -> graph
    replay). Request b owns rows [b*R, (b+1)*R) of every layer's fused table,
    [b*P, (b+1)*P) of the probe table, [b*Q, (b+1)*Q) of the probe rows and
    [b*Mr, (b+1)*Mr) of the recompute rows; positions/kmax are per request.

    Ragged batches (requests with different chunk lengths, query lengths or
    selection sizes) share ONE layer stack: every request's block
    is padded to the batch maximum (R, P, Q, Mr = S + Q with S the largest
    selection), a request's recompute rows are laid out [selected | pad |
    query | pad], and the pad rows run at position 0 attending to BOS only and
    write their K/V into the block's spare last row, which no real row ever
    sees. A homogeneous batch has no pad rows and the exact layout it always
    had."""

    def __init__(self, eng: "FusionEngine", plans: list["_Plan"], extra_rows: int = 0):
        cfg, dev = eng.config, eng.device
        L, H, Hkv, D = cfg.n_layers, cfg.n_heads, cfg.n_kv_heads, cfg.d_head
        dt = eng.weights.torch_dtype
        c = cfg.critical_layer
        B = self.B = len(plans)
        self.n_ctx_r = [p.n_ctx for p in plans]
        self.q_r = [p.q for p in plans]
        self.n_sel_r = [p.n_sel for p in plans]
        self.n_pre_r = [int(p.anchor_rows.size) for p in plans]
        self.n_ch_r = [len(p.records) for p in plans]
        self.ragged = len({p.shape_key() for p in plans}) > 1
        spare = 1 if self.ragged else 0
        self.R = R = max(1 + n + q for n, q in zip(self.n_ctx_r, self.q_r)) + extra_rows + spare
        self.P = P = max(a + q for a, q in zip(self.n_pre_r, self.q_r)) + spare
        self.Q = Q = max(self.q_r)
        self.S = S = max(self.n_sel_r)
        self.Mr = Mr = S + Q
        self.n_ctx_max = n_ctx_max = max(self.n_ctx_r)
        self.n_pre = self.n_pre_r[0]
        self.rows = R
        dsz = ctypes.sizeof(ChunkDesc)
        self.desc_off = [dsz * sum(self.n_ch_r[:r]) for r in range(B)]       # bytes into desc / adesc
        self.delta_off = [4 * sum(self.n_ch_r[:r]) for r in range(B)]        # bytes into adelta
        n_desc = sum(self.n_ch_r)
        self.fk = torch.empty((L, B * R, Hkv, D), dtype=dt, device=dev)
        self.fv = torch.empty_like(self.fk)
        self.desc = torch.empty(n_desc * dsz, dtype=torch.uint8, device=dev)
        self.tok = torch.empty(B * R, dtype=torch.int32, device=dev)
        self.anchor_rows = torch.empty(max(sum(self.n_pre_r), 1), dtype=torch.int32, device=dev)
        # probe prefix straight from each chunk's anchor rows (K rotated by the chunk offset)
        self.adesc = torch.empty(n_desc * dsz, dtype=torch.uint8, device=dev)
        self.adelta = torch.empty(n_desc, dtype=torch.int32, device=dev)
        self.max_delta = n_ctx_max
        self.pk = torch.empty((c, B * P, Hkv, D), dtype=dt, device=dev)
        self.pv = torch.empty_like(self.pk)
        p_pos, p_kmax, p_dst, p_tok = (np.zeros(B * Q, np.int32) for _ in range(4))
        rc_pos, rc_dst = np.zeros(B * Mr, np.int32), np.zeros(B * Mr, np.int32)
        for r in range(B):
            n, q, a = self.n_ctx_r[r], self.q_r[r], self.n_pre_r[r]
            sl = slice(r * Q, (r + 1) * Q)
            i = np.arange(Q)
            live = i < q
            p_pos[sl] = np.where(live, n + 1 + i, 0)                 # probe positions n_ctx+1..
            p_kmax[sl] = np.where(live, a + i, 0)                    # rows in the request's probe table
            p_dst[sl] = r * P + np.where(live, a + i, P - 1)
            p_tok[sl] = r * R + np.where(live, n + 1 + i, R - 1)
            pos = np.zeros(Mr, np.int32)                            # [selected | pad | query | pad]
            dst = np.full(Mr, r * R + R - 1, np.int32)
            pos[S:S + q] = n + 1 + np.arange(q)
            dst[S:S + q] = r * R + n + 1 + np.arange(q)
            rc_pos[r * Mr:(r + 1) * Mr] = pos
            rc_dst[r * Mr:(r + 1) * Mr] = dst
        t32 = lambda a: torch.as_tensor(a, device=dev)  # noqa: E731
        self.p_pos, self.p_kmax, self.p_dst, self.p_tok = t32(p_pos), t32(p_kmax), t32(p_dst), t32(p_tok)
        self.qc = torch.empty((1, B * Q, H, D), dtype=dt, device=dev)
        self.scores = torch.empty(B * n_ctx_max, dtype=torch.float32, device=dev)
        self.score_ws = torch.empty(int(_lib.lib.qcf_score_batched_workspace(n_ctx_max, Q, B, H, Hkv)),
                                    dtype=torch.uint8, device=dev)
        self.rc_pos = t32(rc_pos)   # per-request positions == kmax (selected slots filled by Top-N)
        self.skip_words = (R + 31) // 32   # per-request bitmap of the recompute rows (assembly skips them)
        self.skip_bm = torch.empty(B * self.skip_words, dtype=torch.int32, device=dev)
        self.rc_dst = t32(rc_dst)   # rows in the batch table
        self.last_row = t32(np.asarray([r * Mr + S + self.q_r[r] - 1 for r in range(B)], np.int32))
        self.logits = torch.empty((B, cfg.vocab_size), dtype=torch.float32, device=dev)
        self.sc_probe = eng.ex.scratch(B * Q, key=("probe", id(self)))
        self.sc_rc = eng.ex.scratch(B * Mr, key=("rc", id(self)))
        self.fp32 = eng.fp32_scoring and plans[0].policy == "QCFuse" and S > 0
        if self.fp32:
            # fp32 scoring mode: float32 probe prefix, Q_c and fused critical-layer keys
            f32 = torch.float32
            self.pk32 = torch.empty((c, B * P, Hkv, D), dtype=f32, device=dev)
            self.pv32 = torch.empty_like(self.pk32)
            self.qc32 = torch.empty((B * Q, H, D), dtype=f32, device=dev)
            self.kc32 = torch.empty((B * (1 + n_ctx_max), Hkv, D), dtype=f32, device=dev)
            self.adesc32 = torch.empty_like(self.adesc)
            self.kdesc32 = torch.empty_like(self.desc)
            self.sc_probe32 = eng.ex32.scratch(B * Q, key=("probe32", id(self)))
        self.graph: torch.cuda.CUDAGraph | None = None
        self.rope_key: tuple | None = None   # RoPE table pointers the graph baked in
        self.uses = 0
        self.h_staged: list[torch.Tensor] | None = None   # pinned host mirrors of staged()
        self.h_done: torch.cuda.Event | None = None

    def selection(self, r: int) -> torch.Tensor:
        """Request r's selected positions (device, ascending)."""
        return self.rc_pos[r * self.Mr: r * self.Mr + self.n_sel_r[r]]

    def staged(self) -> list[torch.Tensor]:
        """The device tensors a batch's host inputs are staged into (swapped
        between graph replays)."""
        extra = [self.adesc32, self.kdesc32] if self.fp32 else []
        return [self.desc, self.tok, self.anchor_rows, self.adesc, self.adelta] + extra


class FusionEngine:
    """B200 engine with the reference's FusionEngine surface (fusion.py:211-563)."""

    def __init__(self, weights: ModelWeights, store: ChunkStore, cost: CostModel | None = None,
                 options: RunOptions | None = None):
        if store.dtype != weights.dtype:
            raise ValueError("store pool dtype must match the weights dtype")
        self.weights = weights
        self.config = weights.config
        self.store = store
        self.cost = cost or CostModel(tier=store.tier)
        self.options = options or RunOptions()
        self.device = weights.device
        self.ex = _executor_for(weights)
        # BOS row computed once at position 0 (fusion.py:226-227)
        bos = torch.tensor([BOS_ID], dtype=torch.int32, device=self.device)
        bk, bv, _ = self.ex.forward_full(bos, 0)
        self._bos_k, self._bos_v = bk[:, 0].contiguous(), bv[:, 0].contiguous()
        # fp32 scoring mode (SURVEY §7 hard parts): a bf16 engine whose store keeps
        # float32 critical-layer keys and anchor rows, and whose weights carry
        # float32 copies of layers 1..c: the probe (FFMA GEMMs, float64 RoPE) and
        # the float64 scoring run in float32 end to end, so the selected index set
        # is the reference's bit for bit; the recompute stays bf16 on tcgen05
        self.fp32_scoring = getattr(store, "keep_f32_probe", False)
        self.ex32 = None
        if self.fp32_scoring:
            if weights.probe32 is None:
                raise ValueError("store is in fp32 scoring mode: build the weights with scoring='fp32'")
            self.ex32 = _executor_for(weights.probe32)
            c = self.config.critical_layer
            bk32, bv32, _ = self.ex32.forward_full(bos, 0, layers=range(c))
            self._bos_k32, self._bos_v32 = bk32[:, 0].contiguous(), bv32[:, 0].contiguous()
        self._bufs: "OrderedDict[tuple, _Bufs]" = OrderedDict()
        self.max_shapes = int(os.environ.get("QCF_MAX_SHAPES", "8"))
        self._oracle_cache: dict = {}
        # assembly || probe on two streams (see _launch); measured neutral on B200 at the
        # Llama-3-8B shape (tools/concurrency_check.py: both phases are HBM-bound), off by default
        # True: the whole assembly may also overlap the probe (both HBM-bound); QCF_ASM_CONCURRENT=1
        self.concurrent = os.environ.get("QCF_ASM_CONCURRENT", "0") == "1"
        self.asm_skip = os.environ.get("QCF_ASM_SKIP", "1") != "0"
        self.asm_group = int(os.environ.get("QCF_ASM_GROUP", "4"))   # layers per side-stream assembly launch
        # False: assembly on the main stream, in order (instrumented passes; QCF_PIPELINE_ASM=0)
        self.pipeline_asm = os.environ.get("QCF_PIPELINE_ASM", "1") != "0"
        self.decode_graph = True  # greedy decode as a replayed CUDA graph (False: eager loop)
        self._decode_graphs: dict = {}
        self._aux: torch.cuda.Stream | None = None

    # ------------------------------------------------------------------
    # planning helpers
    # ------------------------------------------------------------------
    def _records(self, chunk_ids):
        if not chunk_ids:
            raise ValueError("chunk list must be non-empty")
        recs = [self.store.get_record(cid) for cid in chunk_ids]
        offs, pos = [], 1
        for r in recs:
            offs.append(pos)
            pos += r.n_tokens
        L = self.config.n_layers
        for r in recs:   # fetch accounting of assemble_context (store.py:402-403)
            nb = 2 * r.n_tokens * self.config.n_kv_heads * self.config.d_head * 4
            self.store.manifest.layers_fetched += L
            self.store.manifest.bytes_fetched += L * nb
        return recs, offs, pos - 1

    def _desc_bytes(self, recs, offs) -> torch.Tensor:
        arr = (ChunkDesc * len(recs))()
        for i, (r, o) in enumerate(zip(recs, offs)):
            arr[i].k = r.k.data_ptr()
            arr[i].v = r.v.data_ptr()
            arr[i].layer_stride = r.k.stride(0)
            arr[i].n_tok = r.n_tokens
            arr[i].offset = o
        return torch.frombuffer(bytearray(arr), dtype=torch.uint8)

    def _anchor_desc_bytes(self, recs, offs) -> torch.Tensor:
        """Descriptors of each chunk's HBM-resident anchor rows, landing at
        consecutive probe-prefix rows after BOS (zero-anchor chunks occupy no rows)."""
        arr = (ChunkDesc * len(recs))()
        row = 1
        for i, r in enumerate(recs):
            ak, av = self.store.anchor_kv(r)
            na = int(r.anchor_indices.size)
            arr[i].k = ak.data_ptr()
            arr[i].v = av.data_ptr()
            arr[i].layer_stride = ak.stride(0) if na else 0
            arr[i].n_tok = na
            arr[i].offset = row
            row += na
        return torch.frombuffer(bytearray(arr), dtype=torch.uint8)

    def _anchor_desc32_bytes(self, recs) -> torch.Tensor:
        """Descriptors of the float32 anchor rows (layers 1..c) of each chunk."""
        arr = (ChunkDesc * len(recs))()
        row = 1
        for i, r in enumerate(recs):
            na = int(r.anchor_indices.size)
            arr[i].k = r.anchor_k32.data_ptr()
            arr[i].v = r.anchor_v32.data_ptr()
            arr[i].layer_stride = r.anchor_k32.stride(0) if na else 0
            arr[i].n_tok = na
            arr[i].offset = row
            row += na
        return torch.frombuffer(bytearray(arr), dtype=torch.uint8)

    def _kcrit32_desc_bytes(self, recs, offs) -> torch.Tensor:
        """Descriptors of the float32 critical-layer keys (one layer, K only)."""
        arr = (ChunkDesc * len(recs))()
        for i, (r, o) in enumerate(zip(recs, offs)):
            arr[i].k = r.k_crit32.data_ptr()
            arr[i].v = r.k_crit32.data_ptr()
            arr[i].layer_stride = 0
            arr[i].n_tok = r.n_tokens
            arr[i].offset = o
        return torch.frombuffer(bytearray(arr), dtype=torch.uint8)

    def _assemble_range(self, recs, n_ctx, fk, fv, desc_dev, layer0, n_layers, stream=None, layer_stride=None,
                        skip_ptr: int | None = None):
        """Layers [layer0, layer0 + n_layers) of assemble_context (fusion.py:234-263).
        skip_ptr: device bitmap of fused rows the recompute rewrites in every layer
        (the selection); those rows are neither read nor written."""
        cfg = self.config
        self.ex.rope.ensure(n_ctx + 2)
        args = (desc_dev.data_ptr(), len(recs), n_ctx, self._bos_k.data_ptr(),
                self._bos_v.data_ptr(), fk.data_ptr(), fv.data_ptr(),
                fk.stride(0) if layer_stride is None else layer_stride, layer0, n_layers,
                cfg.n_kv_heads, cfg.d_head, self.ex.rope.cos.data_ptr(), self.ex.rope.sin.data_ptr(),
                self.ex.rope.n_pos, self.weights.qcf_dtype)
        if skip_ptr is None:
            call("qcf_assemble_range", *args, cuda_stream(stream))
        else:
            call("qcf_assemble_range_skip", *args, skip_ptr, cuda_stream(stream))

    def _assemble_into(self, recs, offs, n_ctx, fk, fv, desc_dev, stream=None, layer_stride=None):
        cfg = self.config
        self.ex.rope.ensure(n_ctx + 2)
        call("qcf_assemble", desc_dev.data_ptr(), len(recs), n_ctx, self._bos_k.data_ptr(),
             self._bos_v.data_ptr(), fk.data_ptr(), fv.data_ptr(),
             fk.stride(0) if layer_stride is None else layer_stride, cfg.n_layers,
             cfg.n_kv_heads, cfg.d_head, self.ex.rope.cos.data_ptr(), self.ex.rope.sin.data_ptr(),
             self.ex.rope.n_pos, self.weights.qcf_dtype, cuda_stream(stream))

    @staticmethod
    def _anchor_rows(recs, offs, mode, n_ctx) -> np.ndarray:
        if mode == PROBE_FULL:
            return np.arange(0, n_ctx + 1, dtype=np.int64)
        rows = [np.zeros(1, np.int64)]
        if mode == PROBE_ANCHORS:
            for r, o in zip(recs, offs):
                if r.anchor_indices.size:
                    rows.append(o + r.anchor_indices)
        elif mode != PROBE_NONE:
            raise ValueError(f"unknown probe mode: {mode}")
        return np.concatenate(rows)

    # ------------------------------------------------------------------
    # context assembly (fusion.py:234-263)
    # ------------------------------------------------------------------
    @_serialized
    def assemble_context(self, chunk_ids: list[str], extra_rows: int = 0) -> FusedContext:
        recs, offs, n_ctx = self._records(chunk_ids)
        cfg = self.config
        fk = torch.empty((cfg.n_layers, 1 + n_ctx + extra_rows, cfg.n_kv_heads, cfg.d_head),
                         dtype=self.weights.torch_dtype, device=self.device)
        fv = torch.empty_like(fk)
        desc = self._desc_bytes(recs, offs).to(self.device)
        self._assemble_into(recs, offs, n_ctx, fk, fv, desc)
        token_ids = np.concatenate([r.token_ids for r in recs])
        chunk_index = np.concatenate([np.full(r.n_tokens, i, np.int64) for i, r in enumerate(recs)])
        return FusedContext(list(chunk_ids), token_ids, offs, n_ctx, chunk_index, fk, fv)

    # ------------------------------------------------------------------
    # probing and scoring (fusion.py:269-329)
    # ------------------------------------------------------------------
    @_serialized
    def probe_query(self, query_tokens, fused: FusedContext, mode: str = PROBE_ANCHORS,
                    layers: int | None = None) -> QueryProbe:
        toks = np.asarray(query_tokens, dtype=np.int64)
        if toks.size == 0:
            raise ValueError("query must be non-empty")
        cfg = self.config
        recs = [self.store.get_record(cid) for cid in fused.chunk_ids]
        rows = self._anchor_rows(recs, fused.offsets, mode, fused.n_ctx)
        n_layers = cfg.n_layers if layers is None else layers
        q = toks.size
        n_pre = rows.size
        dev = self.device
        dt = self.weights.torch_dtype
        pk = torch.empty((n_layers, n_pre + q, cfg.n_kv_heads, cfg.d_head), dtype=dt, device=dev)
        pv = torch.empty_like(pk)
        s = cuda_stream()
        call("qcf_gather_rows", fused.k.data_ptr(), fused.v.data_ptr(), fused.k.stride(0),
             _i32(rows, dev).data_ptr(), n_pre, pk.data_ptr(), pv.data_ptr(), pk.stride(0), n_layers,
             cfg.n_kv_heads * cfg.d_head, self.weights.qcf_dtype, s)
        ar = torch.arange(q, dtype=torch.int32, device=dev)
        pos = ar + (fused.n_ctx + 1)
        dst = ar + n_pre
        self.ex.rope.ensure(fused.n_ctx + q + 2)
        sc = self.ex.scratch(q, key="probe_api")
        self.ex.embed(sc, q, _i32(toks, dev))
        q_store = torch.empty((n_layers, q, cfg.n_heads, cfg.d_head), dtype=dt, device=dev)
        self.ex.stack(sc, q, pos, dst, dst, pk, pv, layers=range(n_layers), q_store=q_store)
        positions = np.arange(1 + fused.n_ctx, 1 + fused.n_ctx + q, dtype=np.int64)
        c = cfg.critical_layer
        crit = (pk[c - 1], pv[c - 1], n_pre) if n_layers >= c else None
        return QueryProbe(toks, positions, q_store, fused.key_positions()[rows] if mode != PROBE_FULL
                          else fused.key_positions(), crit, c)

    @property
    def score_precise(self) -> bool:
        p = self.options.score_precise
        return (self.weights.dtype == "f32") if p is None else bool(p)

    def _score_dev(self, q_c: torch.Tensor, k_ctx: torch.Tensor, n_ctx: int, out: torch.Tensor,
                   ws: torch.Tensor, stream=None, n_req: int = 1, k_req_stride: int | None = None) -> None:
        """qcf_score_batched: q_c [n_req*q][H][D]; request r's context keys at
        k_ctx + r*k_req_stride elements (rows of Hkv*D); out [n_req][n_ctx]."""
        cfg = self.config
        nq = q_c.shape[0] // n_req
        stride = k_req_stride if k_req_stride is not None else n_ctx * cfg.n_kv_heads * cfg.d_head
        call("qcf_score_batched", self.weights.qcf_dtype, q_c.data_ptr(), k_ctx.data_ptr(), stride, n_ctx,
             nq, n_req, cfg.n_heads, cfg.n_kv_heads, cfg.d_head, 1.0 / math.sqrt(cfg.d_head),
             1 if self.options.query_agg == "last" else 0, 1 if self.score_precise else 0,
             out.data_ptr(), ws.data_ptr(), ws.numel(), cuda_stream(stream))

    @_serialized
    def score_against_keys(self, probe: QueryProbe, fused: FusedContext, layer: int) -> np.ndarray:
        if self.options.query_agg not in ("mean", "last"):
            raise ValueError(f"unknown query_agg: {self.options.query_agg}")
        q_c = probe.q_store[layer - 1]
        if q_c.shape[1] != self.config.n_heads or q_c.shape[2] != fused.k.shape[3]:
            raise ValueError("probe and fused context disagree on head shape")
        out = torch.empty(fused.n_ctx, dtype=torch.float32, device=self.device)
        ws = torch.empty(int(_lib.lib.qcf_score_batched_workspace(fused.n_ctx, q_c.shape[0], 1, self.config.n_heads,
                                                                  self.config.n_kv_heads)),
                         dtype=torch.uint8, device=self.device)
        self._score_dev(q_c, fused.k[layer - 1, 1:], fused.n_ctx, out, ws)
        return out.cpu().numpy()

    def score_critical(self, probe: QueryProbe, fused: FusedContext) -> np.ndarray:
        return self.score_against_keys(probe, fused, self.config.critical_layer)

    @_serialized
    def oracle_importance(self, context_tokens, query_tokens) -> np.ndarray:
        """Critical-layer importance from a full GPU forward over
        [BOS | context | query] (fusion.py:331-346)."""
        return self.importance_at(context_tokens, query_tokens, self.config.critical_layer)

    @_serialized
    def importance_at(self, context_tokens, query_tokens, layer: int) -> np.ndarray:
        """oracle_importance at any layer (the full forward runs layers 1..layer)."""
        ctx = np.asarray(context_tokens, np.int64)
        qt = np.asarray(query_tokens, np.int64)
        toks = _i32(np.concatenate([[BOS_ID], ctx, qt]), self.device)
        c = int(layer)
        m = toks.numel()
        cfg = self.config
        q_store = torch.empty((c, m, cfg.n_heads, cfg.d_head), dtype=self.weights.torch_dtype, device=self.device)
        tk, tv = self.ex.new_table(m)
        ar = torch.arange(m, dtype=torch.int32, device=self.device)
        self.ex.rope.ensure(m + 1)
        sc = self.ex.scratch(m, key="oracle")
        self.ex.embed(sc, m, toks)
        self.ex.stack(sc, m, ar, ar, ar, tk, tv, layers=range(c), q_store=q_store)
        out = torch.empty(ctx.size, dtype=torch.float32, device=self.device)
        ws = torch.empty(int(_lib.lib.qcf_score_batched_workspace(ctx.size, qt.size, 1, cfg.n_heads,
                                                                  cfg.n_kv_heads)),
                         dtype=torch.uint8, device=self.device)
        self._score_dev(q_store[c - 1, 1 + ctx.size:].contiguous(), tk[c - 1, 1:1 + ctx.size],
                        ctx.size, out, ws)
        return out.cpu().numpy()

    # ------------------------------------------------------------------
    # selection policies (fusion.py:352-440)
    # ------------------------------------------------------------------
    def qcfuse_select(self, query_tokens, fused: FusedContext, ratio: float) -> SelectionResult:
        if self.fp32_scoring:   # the float32 probe + scoring of the fast path (bit-exact selection)
            return self._qcfuse_select_fp32(query_tokens, fused, ratio)
        probe = self.probe_query(query_tokens, fused, PROBE_ANCHORS, layers=self.config.critical_layer)
        return select_topn(self.score_critical(probe, fused), ratio, "QCFuse")

    @_serialized
    def _qcfuse_select_fp32(self, query_tokens, fused: FusedContext, ratio: float) -> SelectionResult:
        """fusion.py:394-397 in the fp32 scoring mode: the same K2-K5 launches the
        fast path runs (float32 anchor prefix and probe, float32 K_c, float64
        scoring, Top-N), on a one-request buffer set."""
        qt = [int(t) for t in np.asarray(query_tokens, np.int64)]
        if not qt:
            raise ValueError("query must be non-empty")
        n_select(ratio, fused.n_ctx)   # ratio validation (ValueError)
        plans = [self._plan("QCFuse", ratio, fused.chunk_ids, qt)]
        b = self._buffers(plans)
        self._stage(plans, b, [qt])
        self.ex32.rope.ensure(b.rows + 2)
        n = plans[0].n_sel
        if n:
            self._probe_score_fp32(plans, b)
            self._topn_all(b, cuda_stream())
            idx = b.selection(0).cpu().numpy().astype(np.int64)
        else:
            idx = np.zeros(0, np.int64)
        scores = b.scores[:fused.n_ctx].cpu().numpy().copy() if n else np.zeros(fused.n_ctx, np.float32)
        return SelectionResult("QCFuse", ratio, idx, scores)

    def qclast_select(self, query_tokens, fused, ratio) -> SelectionResult:
        probe = self.probe_query(query_tokens, fused, PROBE_NONE)
        return select_topn(self.score_against_keys(probe, fused, self.config.n_layers), ratio, "QCLast")

    def qcall_select(self, query_tokens, fused, ratio) -> SelectionResult:
        probe = self.probe_query(query_tokens, fused, PROBE_FULL)
        if self.options.qcall_layer_average:
            scores = np.mean([self.score_against_keys(probe, fused, li)
                              for li in range(1, self.config.n_layers + 1)], axis=0)
        else:
            scores = self.score_critical(probe, fused)
        return select_topn(scores, ratio, "QCAll")

    @_serialized
    def select(self, policy: str, ratio: float, fused: FusedContext, query_tokens) -> SelectionResult:
        if policy not in POLICIES:
            raise ValueError(f"unknown policy: {policy}")
        n = fused.n_ctx
        if policy == "FullCompute":
            return SelectionResult(policy, 1.0, np.arange(1, n + 1, dtype=np.int64), np.zeros(n, np.float32))
        if policy == "FullReuse":
            return SelectionResult(policy, 0.0, np.zeros(0, np.int64), np.zeros(n, np.float32))
        if policy == "Random":
            return random_select(self.options.selection_seed, n, ratio)
        if policy == "EPIC":
            spans = None
            if self.options.epic_per_chunk:
                spans = [(off, (fused.offsets + [n + 1])[i + 1] - off) for i, off in enumerate(fused.offsets)]
            return epic_select(n, ratio, spans)
        if policy == "QCLast":
            return self.qclast_select(query_tokens, fused, ratio)
        if policy == "QCAll":
            return self.qcall_select(query_tokens, fused, ratio)
        if policy == "CacheBlend":
            return self.cacheblend_select(fused, ratio)
        if policy == "KVShare":
            return self.kvshare_select(fused, ratio)
        return self.qcfuse_select(query_tokens, fused, ratio)

    # ---- layer-1 deviation baselines (fusion.py:352-392) on the device
    @_serialized
    def _layer1_recompute_pass(self, fused: FusedContext, want_attention: bool = False):
        """Layer 1 recomputed for every context token from raw embeddings
        (fusion.py:352-373): returns (new K [n][Hkv][D], new V, received
        attention [n] or None). The reference's full attention weights are
        reduced on the device to what KVShare consumes: their mean over heads
        and rows for each context column (fusion.py:390)."""
        cfg, dev, n = self.config, self.device, fused.n_ctx
        tk = fused.k[0, :n + 1].clone()
        tv = fused.v[0, :n + 1].clone()
        pos = torch.arange(1, n + 1, dtype=torch.int32, device=dev)
        tok = _i32(np.concatenate([[BOS_ID], fused.token_ids]), dev)
        sc = self.ex.scratch(n, key="layer1")
        self.ex.embed(sc, n, tok, rows=pos)
        self.ex.rope.ensure(n + 2)
        q = torch.empty((n, cfg.n_heads, cfg.d_head), dtype=self.weights.torch_dtype, device=dev)
        self.ex.layer(0, sc, n, pos, pos, pos, tk, tv, q_only=True, q_out=q)
        received = None
        if want_attention:
            out = torch.empty(n + 1, dtype=torch.float32, device=dev)
            per_row = 8 * (cfg.n_heads * (n + 1) + 2 * cfg.n_heads)
            ws = torch.empty(8 * (n + 1) + 256 + per_row * min(n, max(1, (256 << 20) // per_row)),
                             dtype=torch.uint8, device=dev)
            scale = 1.0 / float(np.float32(math.sqrt(cfg.d_head)))   # model.py:334 divides by float32(sqrt(D))
            call("qcf_received_attention", self.weights.qcf_dtype, q.data_ptr(), tk.data_ptr(), n + 1, n,
                 cfg.n_heads, cfg.n_kv_heads, cfg.d_head, scale, pos.data_ptr(), out.data_ptr(), ws.data_ptr(),
                 ws.numel(), cuda_stream())
            received = out[1:]
        return tk[1:], tv[1:], received

    def _kv_deviation(self, fused: FusedContext, new_k: torch.Tensor, new_v: torch.Tensor) -> torch.Tensor:
        """fusion.py:375-380 on the device (qcf_kv_deviation)."""
        cfg, n = self.config, fused.n_ctx
        out = torch.empty(n, dtype=torch.float32, device=self.device)
        call("qcf_kv_deviation", self.weights.qcf_dtype, fused.k[0, 1:n + 1].data_ptr(),
             fused.v[0, 1:n + 1].data_ptr(), new_k.data_ptr(), new_v.data_ptr(), n, cfg.n_kv_heads, cfg.d_head,
             out.data_ptr(), cuda_stream())
        return out

    def cacheblend_select(self, fused: FusedContext, ratio: float) -> SelectionResult:
        """fusion.py:382-386: Top-N of the layer-1 KV deviation."""
        k, v, _ = self._layer1_recompute_pass(fused)
        return select_topn(self._kv_deviation(fused, k, v).cpu().numpy(), ratio, "CacheBlend")

    def kvshare_select(self, fused: FusedContext, ratio: float) -> SelectionResult:
        """fusion.py:388-392: Top-N of deviation x received attention."""
        k, v, received = self._layer1_recompute_pass(fused, want_attention=True)
        dev = self._kv_deviation(fused, k, v).cpu().numpy()
        return select_topn(dev * received.cpu().numpy().astype(np.float32), ratio, "KVShare")

    # ------------------------------------------------------------------
    # recomputation (fusion.py:446-490)
    # ------------------------------------------------------------------
    @_serialized
    def recompute_selected(self, fused: FusedContext, selection: SelectionResult):
        cfg = self.config
        sel = np.asarray(selection.indices, dtype=np.int64)
        if sel.size and (sel.min() < 1 or sel.max() > fused.n_ctx):
            raise ValueError("selection indices out of context range")
        new = fused.clone()
        fetch, compute = layer_times(sel.size, fused.n_ctx, cfg, self.cost)
        if sel.size:
            dev = self.device
            pos = _i32(sel, dev)
            tok = _i32(np.concatenate([[BOS_ID], fused.token_ids]), dev)
            sc = self.ex.scratch(sel.size, key="recompute_api")
            self.ex.embed(sc, sel.size, tok, rows=pos)
            self.ex.rope.ensure(fused.n_ctx + 2)
            self.ex.stack(sc, sel.size, pos, pos, pos, new.k, new.v)
            fetch_s, compute_s = [fetch] * cfg.n_layers, [compute] * cfg.n_layers
        else:
            fetch_s, compute_s = [fetch] * cfg.n_layers, [0.0] * cfg.n_layers
        return new, RecomputeTrace(sel, fetch_s, compute_s)

    # ------------------------------------------------------------------
    # the fused fast path
    # ------------------------------------------------------------------
    def _plan(self, policy, ratio, chunk_ids, query_tokens) -> _Plan:
        recs, offs, n_ctx = self._records(chunk_ids)
        q = len(query_tokens)
        if policy == "QCFuse":
            n_sel = n_select(ratio, n_ctx)
            rows = self._anchor_rows(recs, offs, PROBE_ANCHORS, n_ctx)
        elif policy == "FullCompute":
            n_sel, rows = n_ctx, np.zeros(1, np.int64)
        elif policy == "FullReuse":
            n_sel, rows = 0, np.zeros(1, np.int64)
        else:
            raise ValueError(f"fast path covers QCFuse/FullCompute/FullReuse, not {policy}")
        return _Plan(list(chunk_ids), recs, offs, n_ctx, q, n_sel, rows, policy)

    def _buffers(self, plans: list[_Plan], extra_rows: int = 0) -> _Bufs:
        """Per-shape buffers + graph, least-recently-used first out: at most
        `max_shapes` shapes stay resident (each holds a full fused table)."""
        key = (tuple(p.shape_key() for p in plans), extra_rows)
        b = self._bufs.pop(key, None)
        if b is None:
            while len(self._bufs) >= max(1, self.max_shapes):
                self._evict(next(iter(self._bufs)))
            b = _Bufs(self, plans, extra_rows)
        self._bufs[key] = b      # most recently used last
        return b

    def _evict(self, key) -> None:
        b = self._bufs.pop(key)
        b.graph = None
        for k in (("probe", id(b)), ("rc", id(b))):
            self.ex._scratch.pop(k, None)

    def _stage(self, plans: list[_Plan], b: _Bufs, queries, stream=None) -> dict:
        """Host -> device copies of the batch's inputs (chunk descriptors,
        token tables, probe rows). Returns the byte counts."""
        descs, toks, rows, adescs, adeltas, a32, k32 = [], [], [], [], [], [], []
        for plan, qt in zip(plans, queries):
            descs.append(self._desc_bytes(plan.records, plan.offsets))
            adescs.append(self._anchor_desc_bytes(plan.records, plan.offsets))
            if b.fp32:
                a32.append(self._anchor_desc32_bytes(plan.records))
                k32.append(self._kcrit32_desc_bytes(plan.records, plan.offsets))
            adeltas.append(np.asarray(plan.offsets, np.int32))
            t = np.zeros(b.R, np.int32)
            body = np.concatenate([[BOS_ID], *[r.token_ids for r in plan.records], np.asarray(qt, np.int64)])
            t[:body.size] = body
            toks.append(t)
            rows.append(plan.anchor_rows.astype(np.int32))
        desc = torch.cat(descs)
        tok = np.concatenate(toks)
        rows = np.concatenate(rows)
        adesc = torch.cat(adescs)
        adelta = np.concatenate(adeltas)
        host = [desc, torch.from_numpy(tok), torch.from_numpy(rows), adesc, torch.from_numpy(adelta)]
        dev = [b.desc, b.tok, b.anchor_rows[:rows.size], b.adesc, b.adelta]
        if b.fp32:
            host += [torch.cat(a32), torch.cat(k32)]
            dev += [b.adesc32, b.kdesc32]
        if b.h_staged is None:   # persistent pinned staging buffers (no per-call pinned allocation)
            b.h_staged = [torch.empty(t.numel() * t.element_size(), dtype=torch.uint8, pin_memory=True)
                          for t in host]
            b.h_done = torch.cuda.Event()
        b.h_done.synchronize()   # the previous batch's H2D copies out of these buffers have finished
        s = stream or torch.cuda.current_stream()
        with torch.cuda.stream(s):
            for h, pinned, d in zip(host, b.h_staged, dev):
                view = pinned.view(h.dtype)[:h.numel()]
                view.copy_(h.reshape(-1))
                d.copy_(view, non_blocking=True)
            b.h_done.record(s)
        return {"h2d": sum(h.numel() * h.element_size() for h in host)}

    def _launch(self, plans: list[_Plan], b: _Bufs, stream=None) -> None:
        """Every kernel of one (batched) fused prefill, in order (module docstring).
        Ragged batches run the same launches over the padded blocks (_Bufs);
        only scoring and Top-N go request by request there."""
        cfg, ex, plan = self.config, self.ex, plans[0]
        c, B, Q = cfg.critical_layer, b.B, b.Q
        s = cuda_stream(stream)
        row_elems = cfg.n_kv_heads * cfg.d_head
        esz = b.fk.element_size()
        probe = plan.policy == "QCFuse" and b.S > 0
        main = stream or torch.cuda.current_stream()
        # K1 (assembly, HBM-bound on the chunk pool) runs on a side stream, layer range
        # by layer range: the critical layer first (scoring reads it, overlapping the
        # probe), the others once the recompute starts, each range joined by the
        # recompute right before its layer -- so the copy overlaps the tensor-bound
        # recompute instead of preceding it (graph capture records the fork/join).
        # `concurrent`: start every range at once (overlaps the HBM-bound probe).
        layer_ready: dict[int, torch.cuda.Event] = {}
        pending: list[tuple[int, int]] = []
        aux = None
        last = None

        def enqueue(rngs, skip: bool = False) -> None:
            nonlocal last
            for l0, nl in rngs:
                for r in range(B):   # request r's slice of the batch table, layers [l0, l0+nl)
                    sp = b.skip_bm.data_ptr() + 4 * r * b.skip_words if skip else None
                    self._assemble_range(plans[r].records, plans[r].n_ctx, _view_rows(b.fk, r * b.R),
                                         _view_rows(b.fv, r * b.R), _DescView(b.desc, b.desc_off[r]), l0, nl, aux,
                                         layer_stride=b.fk.stride(0), skip_ptr=sp)
                e = torch.cuda.Event()
                e.record(aux)
                last = e
                for l in range(l0, l0 + nl):
                    layer_ready[l] = e

        if sum(b.n_ch_r) > 0:
            if self._aux is None:
                self._aux = torch.cuda.Stream(device=self.device)
            aux = self._aux if self.pipeline_asm else main
            ev = torch.cuda.Event()
            ev.record(main)
            aux.wait_event(ev)
            L, g = cfg.n_layers, max(1, self.asm_group)
            first = [(c - 1, 1)] if probe else []
            lo = 0
            while lo < L:
                hi = min(L, lo + g)
                if probe and lo <= c - 1 < hi:   # split around the critical layer
                    if lo < c - 1:
                        pending.append((lo, c - 1 - lo))
                    if c < hi:
                        pending.append((c, hi - c))
                else:
                    pending.append((lo, hi - lo))
                lo = hi
            enqueue(first)
            if self.concurrent or not probe:
                enqueue(pending)
                pending = []

        def wait_layer(li: int) -> None:
            e = layer_ready.pop(li, None)
            if e is not None:
                main.wait_event(e)
        if probe and b.fp32:
            self._probe_score_fp32(plans, b, stream)
        elif probe:
            for r in range(B):   # K2: probe prefix rows of request r from the chunks' anchor rows
                call("qcf_assemble_rot", b.adesc.data_ptr() + b.desc_off[r], b.n_ch_r[r], b.n_pre_r[r] - 1,
                     self._bos_k.data_ptr(), self._bos_v.data_ptr(), b.pk.data_ptr() + r * b.P * row_elems * esz,
                     b.pv.data_ptr() + r * b.P * row_elems * esz, b.pk.stride(0), c, cfg.n_kv_heads, cfg.d_head,
                     self.ex.rope.cos.data_ptr(), self.ex.rope.sin.data_ptr(), self.ex.rope.n_pos,
                     b.adelta.data_ptr() + b.delta_off[r], b.max_delta, self.weights.qcf_dtype, s)
            # K3: probe layers 1..c-1 + layer c's Q, all B*Q rows at once
            ex.embed(b.sc_probe, B * Q, b.tok, rows=b.p_tok, stream=stream)
            for li in range(c - 1):
                ex.layer(li, b.sc_probe, B * Q, b.p_pos, b.p_dst, b.p_kmax, b.pk[li], b.pv[li], stream=stream,
                         n_req=B)
            ex.layer(c - 1, b.sc_probe, B * Q, b.p_pos, b.p_dst, b.p_kmax, b.pk[c - 1], b.pv[c - 1],
                     q_only=True, q_out=b.qc[0], stream=stream, n_req=B)
            wait_layer(c - 1)
            # K4: scoring (request r's keys at rows r*R+1.. of layer c)
            if not b.ragged:
                self._score_dev(b.qc[0], b.fk[c - 1, 1:], b.n_ctx_max, b.scores, b.score_ws, stream, n_req=B,
                                k_req_stride=b.R * row_elems)
            else:
                for r in range(B):
                    self._score_dev(b.qc[0, r * Q: r * Q + b.q_r[r]], b.fk[c - 1, r * b.R + 1:], b.n_ctx_r[r],
                                    b.scores[r * b.n_ctx_max:], b.score_ws, stream)
        if probe:
            self._topn_all(b, s)
        elif plan.policy == "FullCompute":
            for r in range(B):
                call("qcf_iota", b.n_sel_r[r], 1, b.rc_pos.data_ptr() + r * b.Mr * 4, s)
                call("qcf_iota", b.n_sel_r[r], 1 + r * b.R, b.rc_dst.data_ptr() + r * b.Mr * 4, s)
        if pending:   # the remaining layers' assembly starts with the recompute
            # the selection is known now: the rows the recompute rewrites in every layer
            # are left out of the copy (QCF_ASM_SKIP=0 copies them too)
            skip = probe and self.asm_skip
            if skip:
                call("qcf_rows_bitmap", b.rc_pos.data_ptr(), b.Mr, B, b.Mr, b.skip_bm.data_ptr(), b.skip_words, s)
            ev = torch.cuda.Event()
            ev.record(main)
            aux.wait_event(ev)
            enqueue(pending, skip=skip)
        m = B * b.Mr   # K6: recompute + query rows of the whole batch
        ex.embed(b.sc_rc, m, b.tok, rows=b.rc_dst, stream=stream)
        ex.stack(b.sc_rc, m, b.rc_pos, b.rc_dst, b.rc_pos, b.fk, b.fv, stream=stream, n_req=B,
                 before_layer=wait_layer)
        if last is not None:   # join the side stream (every range is complete by now anyway)
            main.wait_event(last)
        ex.lm_head(b.sc_rc, b.last_row, b.logits, stream=stream)

    @staticmethod
    def _topn_all(b: _Bufs, s) -> None:
        """K5: Top-N of every request (ascending positions -> rc_pos, table rows
        -> rc_dst): one launch for a homogeneous batch; per request otherwise
        (its own context length and N; rc_dst = positions + the block's base)."""
        if not b.ragged:
            call("qcf_topn_batched", b.scores.data_ptr(), b.n_ctx_max, b.B, b.S, 1, b.rc_pos.data_ptr(), b.Mr,
                 b.rc_dst.data_ptr(), b.R, s)
            return
        for r in range(b.B):
            if b.n_sel_r[r] == 0:
                continue
            pos = b.rc_pos.data_ptr() + r * b.Mr * 4
            call("qcf_topn_batched", b.scores.data_ptr() + r * b.n_ctx_max * 4, b.n_ctx_r[r], 1, b.n_sel_r[r], 1,
                 pos, b.n_sel_r[r], None, 0, s)
            call("qcf_iota_add", pos, b.n_sel_r[r], r * b.R, b.rc_dst.data_ptr() + r * b.Mr * 4, s)

    def _probe_score_fp32(self, plans: list[_Plan], b: _Bufs, stream=None) -> None:
        """K2-K4 of the fp32 scoring mode: the probe prefix from the float32
        anchor rows (fusion.py:281-303), the probe's layers 1..c-1 plus layer c's
        Q on the float32 weights (FFMA GEMMs, float64 RoPE; model.py:345-388),
        the float32 fused critical-layer keys assembled from each chunk's float32
        K_c (fusion.py:234-263), and the float64 scoring of fusion.py:313-326."""
        cfg, ex32 = self.config, self.ex32
        c, B, Q = cfg.critical_layer, b.B, b.Q
        s = cuda_stream(stream)
        row_elems = cfg.n_kv_heads * cfg.d_head
        rope = ex32.rope
        kstride = (1 + b.n_ctx_max) * row_elems
        for r in range(B):
            call("qcf_assemble_rot", b.adesc32.data_ptr() + b.desc_off[r], b.n_ch_r[r], b.n_pre_r[r] - 1,
                 self._bos_k32.data_ptr(), self._bos_v32.data_ptr(), b.pk32.data_ptr() + r * b.P * row_elems * 4,
                 b.pv32.data_ptr() + r * b.P * row_elems * 4, b.pk32.stride(0), c, cfg.n_kv_heads, cfg.d_head,
                 rope.cos.data_ptr(), rope.sin.data_ptr(), rope.n_pos, b.adelta.data_ptr() + b.delta_off[r],
                 b.max_delta, _lib.QCF_F32, s)
            call("qcf_assemble", b.kdesc32.data_ptr() + b.desc_off[r], b.n_ch_r[r], b.n_ctx_r[r],
                 self._bos_k32[c - 1].data_ptr(), None, b.kc32.data_ptr() + r * kstride * 4, None, kstride, 1,
                 cfg.n_kv_heads, cfg.d_head, rope.cos.data_ptr(), rope.sin.data_ptr(), rope.n_pos, _lib.QCF_F32, s)
        sc = b.sc_probe32
        ex32.embed(sc, B * Q, b.tok, rows=b.p_tok, stream=stream)
        for li in range(c - 1):
            ex32.layer(li, sc, B * Q, b.p_pos, b.p_dst, b.p_kmax, b.pk32[li], b.pv32[li], stream=stream, n_req=B)
        ex32.layer(c - 1, sc, B * Q, b.p_pos, b.p_dst, b.p_kmax, b.pk32[c - 1], b.pv32[c - 1],
                   q_only=True, q_out=b.qc32, stream=stream, n_req=B)
        agg = 1 if self.options.query_agg == "last" else 0
        scale = 1.0 / math.sqrt(cfg.d_head)
        groups = [(0, B, b.n_ctx_max, Q)] if not b.ragged else [(r, 1, b.n_ctx_r[r], b.q_r[r]) for r in range(B)]
        for r0, nr, n_ctx, q in groups:
            call("qcf_score_batched", _lib.QCF_F32, b.qc32[r0 * Q:].data_ptr(),
                 b.kc32[r0 * (1 + b.n_ctx_max) + 1:].data_ptr(), kstride, n_ctx, q, nr, cfg.n_heads,
                 cfg.n_kv_heads, cfg.d_head, scale, agg, 1, b.scores[r0 * b.n_ctx_max:].data_ptr(),
                 b.score_ws.data_ptr(), b.score_ws.numel(), s)

    # ------------------------------------------------------------------
    # host-pool variant: layer-pipelined chunk-KV streaming
    # ------------------------------------------------------------------
    def _launch_host(self, plans: list[_Plan], b: _Bufs, n_slots: int = 3) -> None:
        """The fused prefill when the chunk pool lives in pinned host memory.

        Probe prefix: `qcf_assemble_rot` from the HBM-resident anchor rows
        (K rotated by the chunk offset, fusion.py:281-303). Scoring: the
        critical-layer fused K from the HBM-resident critical keys. Recompute:
        layer l's chunk K/V are copied host->device on a copy stream into one
        of `n_slots` staging buffers while layer l-1 recomputes; layer l is
        assembled from the slot (`qcf_assemble`, n_layers = 1) right before
        its recompute (fusion.py:468-483 consumes layer l only at step l).
        Same kernels and arithmetic as the HBM path: bit-identical results."""
        cfg, ex, plan = self.config, self.ex, plans[0]
        c, q, n_ctx, n_sel, B, L = cfg.critical_layer, plan.q, plan.n_ctx, plan.n_sel, b.B, cfg.n_layers
        dev, dt = self.device, self.weights.torch_dtype
        main = torch.cuda.current_stream()
        s = cuda_stream(main)
        row_elems = cfg.n_kv_heads * cfg.d_head
        esz = b.fk.element_size()
        self.ex.rope.ensure(b.rows + 2)
        rope = self.ex.rope
        bos_k, bos_v = self._bos_k, self._bos_v     # [L][Hkv][D]
        recs_all = [r for pl in plans for r in pl.records]
        n_ch = len(plan.records)

        def descs(fields) -> torch.Tensor:
            arr = (ChunkDesc * len(fields))()
            for i, (k, v, lstride, n_tok, off) in enumerate(fields):
                arr[i].k, arr[i].v, arr[i].layer_stride, arr[i].n_tok, arr[i].offset = k, v, lstride, n_tok, off
            return torch.frombuffer(bytearray(arr), dtype=torch.uint8).to(dev)

        keep = []   # device descriptor arrays must outlive the launches
        if b.fp32:   # fp32 scoring: its inputs (float32 anchors, K_c) are HBM-resident
            self._probe_score_fp32(plans, b)
            call("qcf_topn_batched", b.scores.data_ptr(), n_ctx, B, n_sel, 1, b.rc_pos.data_ptr(), b.Mr,
                 b.rc_dst.data_ptr(), b.R, s)
        elif plan.policy == "QCFuse" and n_sel > 0:
            for r, pl in enumerate(plans):
                # probe prefix rows [BOS | anchors of chunk 0 | ...] of layers < c, K rotated by off_c
                fields, deltas, row = [], [], 1
                for rec, off in zip(pl.records, pl.offsets):
                    na = rec.anchor_indices.size
                    if na:
                        fields.append((rec.anchor_k.data_ptr(), rec.anchor_v.data_ptr(), na * row_elems, na, row))
                        deltas.append(off)
                        row += na
                if fields:
                    d_desc, d_delta = descs(fields), _i32(deltas, dev)
                    keep += [d_desc, d_delta]
                    call("qcf_assemble_rot", d_desc.data_ptr(), len(fields), row - 1, bos_k.data_ptr(),
                         bos_v.data_ptr(), b.pk.data_ptr() + r * b.P * row_elems * esz,
                         b.pv.data_ptr() + r * b.P * row_elems * esz, b.pk.stride(0), c, cfg.n_kv_heads,
                         cfg.d_head, rope.cos.data_ptr(), rope.sin.data_ptr(), rope.n_pos, d_delta.data_ptr(),
                         max(deltas), self.weights.qcf_dtype, s)
                # critical-layer fused K (V slot filled with K; layer c-1 is re-assembled before its recompute)
                d_desc = descs([(rec.k_crit.data_ptr(), rec.k_crit.data_ptr(), 0, rec.n_tokens, off)
                                for rec, off in zip(pl.records, pl.offsets)])
                keep.append(d_desc)
                lay = (c - 1) * b.fk.stride(0) * esz
                call("qcf_assemble", d_desc.data_ptr(), n_ch, n_ctx, bos_k[c - 1].data_ptr(), bos_v[c - 1].data_ptr(),
                     b.fk.data_ptr() + lay + r * b.R * row_elems * esz, b.fv.data_ptr() + lay + r * b.R * row_elems * esz,
                     b.fk.stride(0), 1, cfg.n_kv_heads, cfg.d_head, rope.cos.data_ptr(), rope.sin.data_ptr(),
                     rope.n_pos, self.weights.qcf_dtype, s)
            ex.embed(b.sc_probe, B * q, b.tok, rows=b.p_tok)
            for li in range(c - 1):
                ex.layer(li, b.sc_probe, B * q, b.p_pos, b.p_dst, b.p_kmax, b.pk[li], b.pv[li], n_req=B)
            ex.layer(c - 1, b.sc_probe, B * q, b.p_pos, b.p_dst, b.p_kmax, b.pk[c - 1], b.pv[c - 1],
                     q_only=True, q_out=b.qc[0], n_req=B)
            self._score_dev(b.qc[0], b.fk[c - 1, 1:], n_ctx, b.scores, b.score_ws, None, n_req=B,
                            k_req_stride=b.R * row_elems)
            call("qcf_topn_batched", b.scores.data_ptr(), n_ctx, B, n_sel, 1, b.rc_pos.data_ptr(), b.Mr,
                 b.rc_dst.data_ptr(), b.R, s)
        elif plan.policy == "FullCompute":
            for r in range(B):
                call("qcf_iota", n_sel, 1, b.rc_pos.data_ptr() + r * b.Mr * 4, s)
                call("qcf_iota", n_sel, 1 + r * b.R, b.rc_dst.data_ptr() + r * b.Mr * 4, s)

        # ---- layer-pipelined streaming of the chunk KV + recompute
        S_tot = sum(r.n_tokens for r in recs_all)
        if not hasattr(self, "_copy_stream"):
            self._copy_stream = torch.cuda.Stream(device=dev)
        cs = self._copy_stream
        slots = self._host_slots(n_slots, S_tot, row_elems, dt)
        staged = [torch.cuda.Event() for _ in range(L)]
        freed = [torch.cuda.Event() for _ in range(L)]
        slot_descs = []
        for si in range(n_slots):   # per slot: descriptors of every request's chunks (fused rows = offsets)
            per_req, base = [], 0
            for pl in plans:
                fields = []
                for rec, off in zip(pl.records, pl.offsets):
                    fields.append((slots[si][0][base:].data_ptr(), slots[si][1][base:].data_ptr(), 0, rec.n_tokens, off))
                    base += rec.n_tokens
                per_req.append(descs(fields))
            slot_descs.append(per_req)

        def fetch(li):
            si = li % n_slots
            with torch.cuda.stream(cs):
                if li >= n_slots:
                    cs.wait_event(freed[li - n_slots])
                base = 0
                for rec in recs_all:
                    n = rec.n_tokens
                    slots[si][0][base:base + n].copy_(rec.k[li].view(n, row_elems), non_blocking=True)
                    slots[si][1][base:base + n].copy_(rec.v[li].view(n, row_elems), non_blocking=True)
                    base += n
                staged[li].record(cs)

        # the previous call's last assemblies (main stream) may still read these
        # slots: the copy stream starts only after everything enqueued so far
        cs.wait_stream(main)
        for li in range(min(n_slots, L)):
            fetch(li)
        m = B * b.Mr
        ex.embed(b.sc_rc, m, b.tok, rows=b.rc_dst)
        for li in range(L):
            main.wait_event(staged[li])
            lay = li * b.fk.stride(0) * esz
            for r in range(B):
                call("qcf_assemble", slot_descs[li % n_slots][r].data_ptr(), n_ch, n_ctx, bos_k[li].data_ptr(),
                     bos_v[li].data_ptr(), b.fk.data_ptr() + lay + r * b.R * row_elems * esz,
                     b.fv.data_ptr() + lay + r * b.R * row_elems * esz, b.fk.stride(0), 1, cfg.n_kv_heads,
                     cfg.d_head, rope.cos.data_ptr(), rope.sin.data_ptr(), rope.n_pos, self.weights.qcf_dtype, s)
            freed[li].record(main)
            if li + n_slots < L:
                fetch(li + n_slots)
            ex.layer(li, b.sc_rc, m, b.rc_pos, b.rc_dst, b.rc_pos, b.fk[li], b.fv[li], n_req=B)
        ex.flush(b.sc_rc, m)
        ex.lm_head(b.sc_rc, b.last_row, b.logits)
        main.wait_stream(cs)
        b._keep = keep + slot_descs   # alive until the next launch into these buffers

    def _host_slots(self, n_slots, rows, row_elems, dt):
        key = (n_slots, rows, row_elems, dt)
        sl = getattr(self, "_slots", None)
        if sl is None or sl[0] != key:
            bufs = [(torch.empty((rows, row_elems), dtype=dt, device=self.device),
                     torch.empty((rows, row_elems), dtype=dt, device=self.device)) for _ in range(n_slots)]
            self._slots = (key, bufs)
        return self._slots[1]

    @_serialized
    def prefill_batch(self, policy: str, ratio: float, chunk_lists, queries, use_graph: bool = True,
                      extra_rows: int = 0, stream=None):
        """Device-side fused prefill of a batch of requests (any mix of chunk
        lengths, query lengths and selection sizes: ragged batches are padded,
        see _Bufs) up to first-token logits. Returns (plans, buffers): logits
        b.logits[r], selection of request r in b.selection(r)."""
        plans = [self._plan(policy, ratio, ids, qt) for ids, qt in zip(chunk_lists, queries)]
        if not plans:
            raise ValueError("empty batch")
        b = self._buffers(plans, extra_rows)
        self._stage(plans, b, queries, stream)
        self.ex.rope.ensure(b.rows + 2)
        if self.ex32 is not None:
            self.ex32.rope.ensure(b.rows + 2)
        if any(r.on_host for pl in plans for r in pl.records):
            if not all(r.on_host for pl in plans for r in pl.records):
                raise ValueError("a batch must draw all its chunks from one pool placement")
            if b.ragged:
                raise NotImplementedError("host-pool batches need requests of one shape")
            self._launch_host(plans, b)   # eager: two streams, per-layer events
            return plans, b
        b.uses += 1
        if not use_graph or (b.ragged and b.uses < 2):
            # a ragged batch composition is captured only once it repeats (a serving
            # loop's compositions mostly do not; capture costs more than one launch)
            self._launch(plans, b, stream)
            return plans, b
        rope_key = tuple((r.cos.data_ptr(), r.sin.data_ptr(), r.cs32.data_ptr(), r.n_pos)
                         for r in (self.ex.rope, self.ex32.rope if self.ex32 is not None else None) if r is not None)
        if b.graph is not None and b.rope_key != rope_key:
            b.graph = None      # the RoPE table grew (moved) since capture: re-capture
        if b.graph is None:
            s = stream or torch.cuda.current_stream()
            side = torch.cuda.Stream(device=self.device)
            side.wait_stream(s)
            with torch.cuda.stream(side):
                self._launch(plans, b, side)       # warm-up (lazy attributes, workspaces)
            s.wait_stream(side)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=side):
                self._launch(plans, b, side)
            s.wait_stream(side)
            b.graph = g
            b.rope_key = rope_key
        b.graph.replay()
        return plans, b

    def prefill(self, policy: str, ratio: float, chunk_ids, query_tokens, use_graph: bool = True,
                extra_rows: int = 0, stream=None):
        """Single-request prefill (a batch of one). Returns (plan, buffers);
        logits in b.logits[0], selection in b.rc_pos[:n_sel]."""
        plans, b = self.prefill_batch(policy, ratio, [chunk_ids], [query_tokens], use_graph, extra_rows, stream)
        return plans[0], b

    @_serialized
    def fuse_batch(self, queries, chunk_lists, ratio: float = 0.15):
        """Batched north-star entry (BASELINE config 3): one fused prefill for
        a batch of RAG requests (ragged allowed). Returns (logits [B][V] numpy,
        list of selected-position arrays)."""
        qts = [byte_tokens(q) if isinstance(q, (str, bytes)) else list(q) for q in queries]
        if not qts or any(not q for q in qts):
            raise ValueError("query must be non-empty")
        plans, b = self.prefill_batch("QCFuse", ratio, chunk_lists, qts)
        pos = b.rc_pos.view(b.B, b.Mr).cpu().numpy().astype(np.int64)
        return b.logits.cpu().numpy(), [pos[r, :b.n_sel_r[r]] for r in range(b.B)]

    @_serialized
    def fuse(self, query, chunk_ids, ratio: float = 0.15):
        """North-star entry: fuse(query, chunks) → (first-token logits [V] f32
        numpy, ascending selected positions). QCFuse policy."""
        qt = byte_tokens(query) if isinstance(query, (str, bytes)) else list(query)
        if not qt:
            raise ValueError("query must be non-empty")
        plan, b = self.prefill("QCFuse", ratio, chunk_ids, qt)
        return b.logits[0].cpu().numpy(), b.rc_pos[:plan.n_sel].cpu().numpy().astype(np.int64)

    # ------------------------------------------------------------------
    # decode (model.py:433-465) over the fused table
    # ------------------------------------------------------------------
    def _decode(self, fk, fv, next_pos: int, first_logits: np.ndarray, max_new: int) -> list[int]:
        if max_new < 1:
            raise ValueError("max_new must be >= 1")
        if self.decode_graph:
            return self._decode_graph(fk, fv, next_pos, first_logits, max_new)
        out, logits = [], first_logits
        dev = self.device
        tok = torch.empty(1, dtype=torch.int32, device=dev)
        pos = torch.empty(1, dtype=torch.int32, device=dev)
        zero = torch.zeros(1, dtype=torch.int32, device=dev)
        lg = torch.empty((1, self.config.vocab_size), dtype=torch.float32, device=dev)
        sc = self.ex.scratch(1, key="decode")
        for step in range(max_new):
            t = int(np.argmax(logits))
            out.append(t)
            if t == EOS_ID or step == max_new - 1:
                break
            tok.fill_(t)
            pos.fill_(next_pos)
            self.ex.rope.ensure(next_pos + 2)
            self.ex.embed(sc, 1, tok)
            self.ex.stack(sc, 1, pos, pos, pos, fk, fv)
            self.ex.lm_head(sc, zero, lg)
            logits = lg[0].cpu().numpy()
            next_pos += 1
        return out

    def _decode_graph(self, fk, fv, next_pos: int, first_logits: np.ndarray, max_new: int) -> list[int]:
        """The same greedy decode with the argmax on the device (`qcf_decode_advance`:
        ties -> lowest index, like np.argmax) and one decode step captured as a CUDA
        graph, replayed max_new - 1 times with no host round trip per token; the
        tokens after the first EOS are discarded (their KV rows land in the table's
        spare rows, as the eager loop's would not)."""
        t0 = int(np.argmax(first_logits))
        if t0 == EOS_ID or max_new == 1:
            return [t0]
        n = max_new - 1
        dev, V = self.device, self.config.vocab_size
        self.ex.rope.ensure(next_pos + n + 2)
        # one captured step per (table, token budget): the graph reads tok / pos /
        # step from device buffers, so later calls on the same table only reset them
        rope = self.ex.rope   # (a grown RoPE table moves: part of the key)
        key = (fk.data_ptr(), fv.data_ptr(), tuple(fk.shape), n, rope.cos.data_ptr(), rope.cs32.data_ptr())
        st = self._decode_graphs.get(key)
        s = torch.cuda.current_stream()
        if st is None:
            st = {"tok": torch.zeros(1, dtype=torch.int32, device=dev),
                  "pos": torch.zeros(1, dtype=torch.int32, device=dev),
                  "step": torch.zeros(1, dtype=torch.int32, device=dev),
                  "log": torch.zeros(n, dtype=torch.int32, device=dev),
                  "zero": torch.zeros(1, dtype=torch.int32, device=dev),
                  "lg": torch.empty((1, V), dtype=torch.float32, device=dev),
                  "sc": self.ex.scratch(1, key=("decode", key)), "graph": None}
        tok, pos, step, log, lg = st["tok"], st["pos"], st["step"], st["log"], st["lg"]
        tok.fill_(t0)
        pos.fill_(next_pos)
        step.zero_()
        log.fill_(-1)

        def one_step(stream) -> None:
            self.ex.embed(st["sc"], 1, tok, stream=stream)
            self.ex.stack(st["sc"], 1, pos, pos, pos, fk, fv, stream=stream)
            self.ex.lm_head(st["sc"], st["zero"], lg, stream=stream)
            call("qcf_decode_advance", lg.data_ptr(), V, tok.data_ptr(), pos.data_ptr(), step.data_ptr(),
                 log.data_ptr(), n, cuda_stream(stream))

        if st["graph"] is None:
            side = torch.cuda.Stream(device=dev)
            side.wait_stream(s)
            with torch.cuda.stream(side):
                one_step(side)                  # step 1, eagerly (lazy attributes, workspaces)
            if n > 1:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=side):
                    one_step(side)
                st["graph"] = g
            s.wait_stream(side)
            reps = n - 1
            if len(self._decode_graphs) >= 4:
                self._decode_graphs.clear()
            self._decode_graphs[key] = st
        else:
            reps = n
        for _ in range(reps):
            st["graph"].replay()
        out = [t0]
        for t in log.cpu().tolist():
            out.append(int(t))
            if t == EOS_ID:
                break
        return out

    # ------------------------------------------------------------------
    # end to end (fusion.py:496-563)
    # ------------------------------------------------------------------
    @_serialized
    def oracle_run(self, context_tokens, query_tokens, max_new: int | None = None) -> dict:
        """Full-computation reference on the GPU (fusion.py:496-517): a full
        prefill over [BOS | context | query], greedy decode, importance."""
        max_new = max_new or self.options.max_new
        key = (np.asarray(context_tokens, np.int64).tobytes(), np.asarray(query_tokens, np.int64).tobytes(),
               max_new)
        if key in self._oracle_cache:
            return self._oracle_cache[key]
        ctx = np.asarray(context_tokens, np.int64)
        qt = np.asarray(query_tokens, np.int64)
        toks = np.concatenate([[BOS_ID], ctx, qt])
        m = toks.size
        tk, tv = self.ex.new_table(m + max_new)
        _, _, sc = self.ex.forward_full(_i32(toks, self.device), 0, tab=(tk, tv))
        lg = torch.empty((1, self.config.vocab_size), dtype=torch.float32, device=self.device)
        self.ex.lm_head(sc, torch.tensor([m - 1], dtype=torch.int32, device=self.device), lg)
        first = lg[0].cpu().numpy()
        answer = self._decode(tk, tv, m, first, max_new)
        res = {"first_logits": first, "answer_tokens": answer,
               "importance": self.oracle_importance(ctx, qt)}
        self._oracle_cache[key] = res
        return res

    @_serialized
    def run(self, policy: str, ratio: float, chunk_ids: list[str], query,
            compare_oracle: bool = False, max_new: int | None = None) -> RunResult:
        if policy not in POLICIES:
            raise ValueError(f"unknown policy: {policy}")
        if not (0.0 <= ratio <= 1.0):
            raise ValueError("ratio must be in [0, 1]")
        max_new = max_new or self.options.max_new
        qt = byte_tokens(query) if isinstance(query, (str, bytes)) else list(query)
        if not qt:
            raise ValueError("query must be non-empty")
        if not chunk_ids:
            raise ValueError("chunk list must be non-empty")
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if policy in ("QCFuse", "FullCompute", "FullReuse") and self.options.query_agg == "mean":
            ev0.record()
            plan, b = self.prefill(policy, ratio, chunk_ids, qt, use_graph=False, extra_rows=max_new)
            ev1.record()
            n_ctx = plan.n_ctx
            sel_idx = b.rc_pos[:plan.n_sel].cpu().numpy().astype(np.int64)
            scores = (b.scores.cpu().numpy() if policy == "QCFuse" and plan.n_sel
                      else np.zeros(n_ctx, np.float32))
            selection = SelectionResult(policy, 1.0 if policy == "FullCompute" else
                                        (0.0 if policy == "FullReuse" else ratio), sel_idx, scores)
            first = b.logits[0].cpu().numpy()
            fk, fv = b.fk, b.fv
            token_ids = np.concatenate([r.token_ids for r in plan.records])
        else:
            ev0.record()
            fused = self.assemble_context(chunk_ids, extra_rows=len(qt) + max_new)
            selection = self.select(policy, ratio, fused, qt)
            upd, _ = self.recompute_selected(fused, selection)
            n_ctx = fused.n_ctx
            fk, fv = upd.k, upd.v
            m = len(qt)
            pos = torch.arange(m, dtype=torch.int32, device=self.device) + (n_ctx + 1)
            sc = self.ex.scratch(m, key="query_api")
            self.ex.embed(sc, m, _i32(qt, self.device))
            self.ex.stack(sc, m, pos, pos, pos, fk, fv)
            lg = torch.empty((1, self.config.vocab_size), dtype=torch.float32, device=self.device)
            self.ex.lm_head(sc, torch.tensor([m - 1], dtype=torch.int32, device=self.device), lg)
            ev1.record()
            first = lg[0].cpu().numpy()
            sel_idx = selection.indices
            token_ids = fused.token_ids
        torch.cuda.synchronize()
        ttft_ms = ev0.elapsed_time(ev1)
        answer = self._decode(fk, fv, n_ctx + 1 + len(qt), first, max_new)
        fetch, compute = layer_times(sel_idx.size, n_ctx, self.config, self.cost)
        trace = RecomputeTrace(sel_idx, [fetch] * self.config.n_layers,
                               [compute if sel_idx.size else 0.0] * self.config.n_layers)
        schedule = policy_schedule(policy, sel_idx.size, n_ctx, len(qt), self.config, self.cost)
        trace.events = schedule_events(schedule)
        comparison = None
        if compare_oracle:
            from . import metrics
            oracle = self.oracle_run(token_ids, qt, max_new)
            div, kl = metrics.logit_divergence(oracle["first_logits"], first)
            match = metrics.token_match_rate(oracle["answer_tokens"], answer, max_new)
            top = top_n_positions(oracle["importance"], sel_idx.size)
            comparison = OracleComparison(div, kl, match, metrics.selection_overlap(sel_idx, top))
        return RunResult(policy, selection.ratio, answer, render_tokens(answer), first, selection,
                         trace, schedule, schedule.ttft + self.cost.decode_gamma, comparison,
                         {"ttft_device_ms": ttft_ms})
