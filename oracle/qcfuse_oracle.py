"""CPU ORACLE — test infrastructure only, never the product path.

A numpy restatement of the reference QCFuse fused-prefill path
(`/root/reference/pkg/src/qcfuse/{model,store,fusion}.py`). Every function
cites the reference file:line whose arithmetic it follows. Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` / `--impl reference`
legs may import this module, and only as a checker / CPU baseline.

Pinning: `tests/test_oracle_golden.py` checks this restatement against the
golden vectors in `tests/golden/` that `tests/golden/make_golden.py` generated
by importing and running the reference itself in the build container, plus
the reference's own known-answer vectors (splitmix64 seed-0, golden logits
`tests/data/golden_logits_ab.json`, select_topn / extract_anchors examples).

Deviations from the reference that do not change the algorithm:
* attention and scoring contract Q·Kᵀ with per-head `np.matmul` (threaded
  BLAS) instead of the unthreaded `np.einsum` (`model.py:334,337`,
  `fusion.py:322`); same products, different summation order (≤1e-6 rel);
* `init_weights` draws the splitmix64 stream tensor by tensor instead of all
  at once (`model.py:240-241` materialises every draw), so Llama-width weights
  fit in RAM; bit-identical because the stream is indexable by global step;
* `layers=` lets callers build only a prefix of the layer stack (the CPU
  baseline times a bounded sample of layers at full width).
"""

from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass, field

import numpy as np

BOS_ID, EOS_ID, PAD_ID, VOCAB = 256, 257, 258, 259
W_LO, W_HI = -0.05, 0.05
_M64 = (1 << 64) - 1
_GAMMA = 0x9E3779B97F4A7C15
_MIX1 = 0xBF58476D1CE4E5B9
_MIX2 = 0x94D049BB133111EB


# --------------------------------------------------------------------------
# deterministic init                               model.py:35-46, 67-69, 225-257
# --------------------------------------------------------------------------

def splitmix64_at(seed: int, steps) -> np.ndarray:
    """Output `steps` of the splitmix64 stream keyed by `seed` (model.py:35-46):
    state_g = seed + (g+1)·γ, then the two xor-shift-multiply mixes."""
    g = np.asarray(steps, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed & _M64) + (g + np.uint64(1)) * np.uint64(_GAMMA)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(_MIX1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(_MIX2)
        return z ^ (z >> np.uint64(31))


def u64_to_unit(u) -> np.ndarray:
    """Top 53 bits × 2⁻⁵³ → float64 in [0,1) (model.py:67-69)."""
    return (np.asarray(u, dtype=np.uint64) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def draw_uniform_f32(seed: int, start: int, count: int) -> np.ndarray:
    """Draws start..start+count of the stream mapped to [-0.05,0.05) in f32
    (model.py:241: LOW + u·(HIGH-LOW) in float64, then cast)."""
    u = u64_to_unit(splitmix64_at(seed, np.arange(start, start + count, dtype=np.uint64)))
    return (W_LO + u * (W_HI - W_LO)).astype(np.float32)


@dataclass(frozen=True)
class Config:
    """Mirror of ModelConfig (model.py:74-118), validated the same way."""
    n_layers: int = 4
    n_heads: int = 2
    d_model: int = 32
    d_head: int = 16
    d_ff: int = 64
    vocab_size: int = VOCAB
    rope_theta: float = 10000.0
    ln_eps: float = 1e-5
    seed: int = 1234
    critical_layer: int | None = None
    # GQA extension (the reference is MHA-only): query head h reads kv head
    # h // (n_heads / n_kv_heads); None = n_heads, which IS the reference
    n_kv_heads: int | None = None

    def __post_init__(self):
        if self.critical_layer is None:                     # model.py:87-89
            object.__setattr__(self, "critical_layer", math.ceil(self.n_layers / 2))
        if self.n_kv_heads is None:
            object.__setattr__(self, "n_kv_heads", self.n_heads)
        if self.n_heads % self.n_kv_heads:
            raise ValueError("n_heads must be a multiple of n_kv_heads")
        if self.d_model != self.n_heads * self.d_head:      # model.py:92-105
            raise ValueError("d_model must equal n_heads * d_head")
        if self.n_layers < 4:
            raise ValueError("n_layers must be >= 4")
        if not (1 < self.critical_layer < self.n_layers):
            raise ValueError("critical_layer must satisfy 1 < c < n_layers")
        if self.d_head % 2:
            raise ValueError("d_head must be even")


@dataclass
class Layer:
    wq: np.ndarray
    wk: np.ndarray
    wv: np.ndarray
    wo: np.ndarray
    w1: np.ndarray
    w2: np.ndarray
    ln1_g: np.ndarray
    ln1_b: np.ndarray
    ln2_g: np.ndarray
    ln2_b: np.ndarray


@dataclass
class Weights:
    cfg: Config
    emb: np.ndarray            # [V, d]; tied lm-head (model.py:384-385)
    layers: list[Layer]
    lnf_g: np.ndarray
    lnf_b: np.ndarray


def weight_shapes(cfg: Config) -> list[tuple[int, int]]:
    """Stream order: embedding, then per layer wq wk wv wo w1 w2 (model.py:232-235);
    GQA: wk/wv are [d, Hkv*D] at the same stream positions."""
    d, f = cfg.d_model, cfg.d_ff
    kvd = cfg.n_kv_heads * cfg.d_head
    shapes = [(cfg.vocab_size, d)]
    for _ in range(cfg.n_layers):
        shapes += [(d, d), (d, kvd), (d, kvd), (d, d), (d, f), (f, d)]
    return shapes


def init_weights(cfg: Config, layers: int | None = None) -> Weights:
    """Bit-exact chunked restatement of init_weights (model.py:225-257)."""
    n_build = cfg.n_layers if layers is None else layers
    shapes = weight_shapes(cfg)
    mats, off = [], 0
    for i, (r, c) in enumerate(shapes):
        if i == 0 or (i - 1) // 6 < n_build:
            mats.append(draw_uniform_f32(cfg.seed, off, r * c).reshape(r, c))
        off += r * c
    d = cfg.d_model
    one, zero = np.ones(d, np.float32), np.zeros(d, np.float32)
    layer_list = []
    for li in range(n_build):
        wq, wk, wv, wo, w1, w2 = mats[1 + 6 * li: 7 + 6 * li]
        layer_list.append(Layer(wq, wk, wv, wo, w1, w2, one.copy(), zero.copy(),
                                one.copy(), zero.copy()))
    return Weights(cfg, mats[0], layer_list, one.copy(), zero.copy())


# --------------------------------------------------------------------------
# model arithmetic                                           model.py:264-424
# --------------------------------------------------------------------------

def inv_freq(d_head: int, theta: float) -> np.ndarray:
    """θ^(−2j/D) in float64 (model.py:264-268)."""
    return theta ** (-2.0 * np.arange(d_head // 2, dtype=np.float64) / d_head)


def rope(x: np.ndarray, positions, theta: float) -> np.ndarray:
    """Interleaved-pair rotation in float64, cast to f32 (model.py:271-286)."""
    ang = np.asarray(positions, np.float64)[:, None] * inv_freq(x.shape[-1], theta)[None]
    c, s = np.cos(ang)[:, None, :], np.sin(ang)[:, None, :]
    x64 = x.astype(np.float64)
    ev, od = x64[..., 0::2], x64[..., 1::2]
    out = np.empty_like(x64)
    out[..., 0::2] = ev * c - od * s
    out[..., 1::2] = ev * s + od * c
    return out.astype(np.float32)


def rope_delta(x: np.ndarray, delta: int, theta: float) -> np.ndarray:
    """Shift every row by the same delta (model.py:289-292)."""
    return rope(x, np.full(x.shape[0], delta, np.int64), theta)


def layer_norm(x, g, b, eps):
    """Biased-variance LayerNorm (model.py:305-308)."""
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    return ((x - mu) / np.sqrt(var + eps)) * g + b


def softmax_rows(s: np.ndarray) -> np.ndarray:
    """Max-subtracted softmax over the last axis, f32 out (model.py:319-323)."""
    e = np.exp(s - s.max(axis=-1, keepdims=True))
    return (e / e.sum(axis=-1, keepdims=True)).astype(np.float32)


def repeat_kv(k: np.ndarray, n_heads: int) -> np.ndarray:
    """GQA: [n, Hkv, D] → [n, H, D], query head h reading kv head h // (H/Hkv)."""
    return k if k.shape[1] == n_heads else np.repeat(k, n_heads // k.shape[1], axis=1)


def attention(q, k, v, mask):
    """Masked SDPA (model.py:326-338): scores divided by float32(√D), -inf
    outside the mask. q [m,H,D], k/v [n,Hkv,D], mask [m,n] → (out [m,H,D], w [H,m,n])."""
    d = q.shape[-1]
    k, v = repeat_kv(k, q.shape[1]), repeat_kv(v, q.shape[1])
    s = np.matmul(q.transpose(1, 0, 2), k.transpose(1, 2, 0)) / np.float32(math.sqrt(d))
    s = np.where(mask[None], s, np.float32(-np.inf))
    w = softmax_rows(s)
    out = np.matmul(w, v.transpose(1, 0, 2)).transpose(1, 0, 2).astype(np.float32)
    return out, w


def ffn(x, lw: Layer):
    """ReLU two-matrix FFN (model.py:341-342)."""
    return np.maximum(x @ lw.w1, np.float32(0.0)) @ lw.w2


@dataclass
class KV:
    keys: np.ndarray       # [n, H, D] post-RoPE
    values: np.ndarray
    positions: np.ndarray  # [n] int64


@dataclass
class Trace:
    logits: np.ndarray
    kv: list[KV]
    attn: list[np.ndarray] | None
    queries: list[np.ndarray] | None


def forward(w: Weights, tokens, positions, past: list[KV] | None = None,
            want_attn=False, want_q=False, layers: int | None = None) -> Trace:
    """Decoder stack (model.py:345-388): LN → QKV → RoPE → attention over
    [past | self] (past fully visible, self causal) → Wo residual → FFN residual;
    then LN_f and the tied lm-head."""
    cfg = w.cfg
    tokens = np.asarray(tokens, np.int64)
    positions = np.asarray(positions, np.int64)
    H, Hkv, D = cfg.n_heads, cfg.n_kv_heads, cfg.d_head
    x = w.emb[tokens]
    n = tokens.size
    self_mask = positions[None, :] <= positions[:, None]
    kvs, attns, qs = [], [], []
    n_layers = len(w.layers) if layers is None else layers
    for li in range(n_layers):
        lw = w.layers[li]
        a = layer_norm(x, lw.ln1_g, lw.ln1_b, cfg.ln_eps)
        q = rope((a @ lw.wq).reshape(n, H, D), positions, cfg.rope_theta)
        k = rope((a @ lw.wk).reshape(n, Hkv, D), positions, cfg.rope_theta)
        v = (a @ lw.wv).reshape(n, Hkv, D)
        if past is not None:
            pk = past[li]
            k_all = np.concatenate([pk.keys, k])
            v_all = np.concatenate([pk.values, v])
            mask = np.concatenate([np.ones((n, pk.keys.shape[0]), bool), self_mask], axis=1)
        else:
            k_all, v_all, mask = k, v, self_mask
        o, aw = attention(q, k_all, v_all, mask)
        x = x + o.reshape(n, -1) @ lw.wo
        x = x + ffn(layer_norm(x, lw.ln2_g, lw.ln2_b, cfg.ln_eps), lw)
        kvs.append(KV(k, v, positions.copy()))
        if want_attn:
            attns.append(aw)
        if want_q:
            qs.append(q)
    x = layer_norm(x, w.lnf_g, w.lnf_b, cfg.ln_eps)
    logits = x @ w.emb.T
    return Trace(logits, kvs, attns if want_attn else None, qs if want_q else None)


def forward_full(w: Weights, tokens, start: int = 0, **kw) -> Trace:
    """model.py:391-400."""
    tokens = np.asarray(tokens, np.int64)
    if tokens.size == 0 or start < 0:
        raise ValueError("bad forward_full input")
    return forward(w, tokens, np.arange(start, start + tokens.size), None, **kw)


def decode_greedy(w: Weights, state: list[KV], first_logits, max_new=32) -> list[int]:
    """Greedy argmax decode (model.py:433-465); ties → lowest id."""
    keys = [s.keys for s in state]
    vals = [s.values for s in state]
    poss = [s.positions for s in state]
    nxt = int(max(int(p.max()) for p in poss if p.size)) + 1
    out, logits = [], first_logits
    for step in range(max_new):
        tok = int(np.argmax(logits))
        out.append(tok)
        if tok == EOS_ID or step == max_new - 1:
            break
        past = [KV(keys[i], vals[i], poss[i]) for i in range(len(keys))]
        tr = forward(w, [tok], [nxt], past)
        for i, kv in enumerate(tr.kv):
            keys[i] = np.concatenate([keys[i], kv.keys])
            vals[i] = np.concatenate([vals[i], kv.values])
            poss[i] = np.concatenate([poss[i], [nxt]])
        logits = tr.logits[-1]
        nxt += 1
    return out


# --------------------------------------------------------------------------
# chunk store (offline precompute)                              store.py:46-69, 315-363
# --------------------------------------------------------------------------

def chunk_hash(tokens) -> str:
    """SHA-256 of little-endian u32 token ids (store.py:52-56)."""
    return hashlib.sha256(np.asarray(tokens, dtype="<u4").tobytes()).hexdigest()


def extract_anchors(norms, ratio: float) -> np.ndarray:
    """Top-⌈ratio·n⌉ norms, ties → lower index, ascending (store.py:59-69)."""
    norms = np.asarray(norms, np.float64)
    if norms.size == 0 or not (0.0 < ratio <= 1.0):
        raise ValueError("bad anchor input")
    count = math.ceil(ratio * norms.size)
    return np.sort(np.argsort(-norms, kind="stable")[:count]).astype(np.int64)


@dataclass
class Chunk:
    tokens: np.ndarray
    kv: list[KV]              # base position 0, no BOS
    key_norms: np.ndarray
    anchors: np.ndarray

    @property
    def n(self) -> int:
        return int(self.tokens.size)


def precompute_chunk(w: Weights, tokens, anchor_ratio=0.05, norm_mode="critical") -> Chunk:
    """forward_full at base 0 without BOS, per-layer key norm (L2 over D,
    mean over heads) at the critical layer, anchors (store.py:338-354)."""
    tokens = np.asarray(tokens, np.int64)
    tr = forward_full(w, tokens, 0)
    per_layer = np.stack([np.linalg.norm(kv.keys, axis=2).mean(axis=1) for kv in tr.kv])
    if norm_mode == "critical":
        norms = per_layer[w.cfg.critical_layer - 1]
    else:
        norms = per_layer.mean(axis=0)
    norms = norms.astype(np.float32)
    return Chunk(tokens, tr.kv, norms, extract_anchors(norms, anchor_ratio))


# --------------------------------------------------------------------------
# fusion hot path                                             fusion.py:141-563
# --------------------------------------------------------------------------

@dataclass
class Fused:
    tokens: np.ndarray          # [n_ctx]
    offsets: list[int]          # offsets[0] == 1
    keys: list[np.ndarray]      # per layer [1+n_ctx, H, D]
    values: list[np.ndarray]
    n_ctx: int


def bos_kv(w: Weights) -> list[KV]:
    """BOS row computed once at position 0 (fusion.py:226-227)."""
    return forward_full(w, [BOS_ID], 0).kv


def assemble(w: Weights, chunks: list[Chunk], bos: list[KV] | None = None) -> Fused:
    """[BOS | R(off_c)·K_c …] per layer, V concatenated (fusion.py:234-263);
    offsets start at 1 and accumulate chunk lengths (fusion.py:241-246)."""
    if not chunks:
        raise ValueError("chunk list must be non-empty")
    bos = bos or bos_kv(w)
    offs, pos = [], 1
    for c in chunks:
        offs.append(pos)
        pos += c.n
    keys, vals = [], []
    for li in range(len(w.layers)):
        kp = [bos[li].keys] + [rope_delta(c.kv[li].keys, o, w.cfg.rope_theta)
                               for c, o in zip(chunks, offs)]
        vp = [bos[li].values] + [c.kv[li].values for c in chunks]
        keys.append(np.concatenate(kp))
        vals.append(np.concatenate(vp))
    return Fused(np.concatenate([c.tokens for c in chunks]), offs, keys, vals, pos - 1)


@dataclass
class Probe:
    queries: list[np.ndarray]
    critical_attention: np.ndarray
    prefix_positions: np.ndarray


def probe(w: Weights, chunks: list[Chunk], fused: Fused, query, mode="anchors",
          bos: list[KV] | None = None, layers: int | None = None) -> Probe:
    """Forward the query over [BOS | anchors re-rotated to their fused
    positions] (fusion.py:269-311); mode "full" uses the whole fused context
    and "none" BOS only. `layers` truncates the stack (QCFuse needs Q_c only)."""
    q = np.asarray(query, np.int64)
    if q.size == 0:
        raise ValueError("query must be non-empty")
    bos = bos or bos_kv(w)
    past = []
    for li in range(len(w.layers)):
        if mode == "full":
            past.append(KV(fused.keys[li], fused.values[li], np.arange(fused.n_ctx + 1)))
            continue
        kp, vp, pp = [bos[li].keys], [bos[li].values], [np.zeros(1, np.int64)]
        if mode == "anchors":
            for c, off in zip(chunks, fused.offsets):
                idx = c.anchors
                if idx.size == 0:
                    continue
                kp.append(rope_delta(c.kv[li].keys[idx], off, w.cfg.rope_theta))
                vp.append(c.kv[li].values[idx])
                pp.append(off + idx)
        elif mode != "none":
            raise ValueError(f"unknown probe mode: {mode}")
        past.append(KV(np.concatenate(kp), np.concatenate(vp), np.concatenate(pp)))
    positions = np.arange(1 + fused.n_ctx, 1 + fused.n_ctx + q.size)
    tr = forward(w, q, positions, past, want_attn=True, want_q=True, layers=layers)
    c = w.cfg.critical_layer
    crit = tr.attn[c - 1] if len(tr.attn) >= c else None
    n_pre = past[0].positions.size
    return Probe(tr.queries, None if crit is None else crit[:, :, :n_pre], past[0].positions)


def score_against_keys(q_c: np.ndarray, k_ctx: np.ndarray, d_head: int, agg="mean") -> np.ndarray:
    """softmax over context keys of (Q·K)·(1/√D), mean over (h,t) or last t
    (fusion.py:313-326, 566-569). q_c [q,H,D], k_ctx [n_ctx,Hkv,D]."""
    scale = 1.0 / math.sqrt(d_head)
    k_ctx = repeat_kv(k_ctx, q_c.shape[1])
    s = np.matmul(q_c.transpose(1, 0, 2), k_ctx.transpose(1, 2, 0)) * scale
    e = np.exp(s - s.max(axis=-1, keepdims=True))
    wts = e / e.sum(axis=-1, keepdims=True)
    if agg == "last":
        wts = wts[:, -1:, :]
    return wts.mean(axis=(0, 1)).astype(np.float32)


def n_select(ratio: float, n_ctx: int) -> int:
    """N = ceil(ratio·n_ctx) in Python double (fusion.py:151-155)."""
    if not (0.0 <= ratio <= 1.0):
        raise ValueError("ratio must be in [0, 1]")
    return math.ceil(ratio * n_ctx)


def select_topn(scores, ratio: float) -> np.ndarray:
    """Stable top-N, ties → lower index, ascending, 1-based (fusion.py:148-158)."""
    s = np.asarray(scores, np.float64)
    n = n_select(ratio, s.size)
    return (np.sort(np.argsort(-s, kind="stable")[:n]) + 1).astype(np.int64)


def recompute(w: Weights, fused: Fused, sel) -> Fused:
    """Selective recompute (fusion.py:446-490): selected rows restart from raw
    embeddings; each layer writes their fresh K/V into rows `sel` before the
    masked attention (key position ≤ row position) over the whole table."""
    cfg = w.cfg
    sel = np.asarray(sel, np.int64)
    keys = [k.copy() for k in fused.keys]
    vals = [v.copy() for v in fused.values]
    if sel.size:
        if sel.min() < 1 or sel.max() > fused.n_ctx:
            raise ValueError("selection indices out of context range")
        H, Hkv, D = cfg.n_heads, cfg.n_kv_heads, cfg.d_head
        x = w.emb[fused.tokens[sel - 1]]
        vis = np.arange(fused.n_ctx + 1)[None, :] <= sel[:, None]
        m = sel.size
        for li, lw in enumerate(w.layers):
            a = layer_norm(x, lw.ln1_g, lw.ln1_b, cfg.ln_eps)
            q = rope((a @ lw.wq).reshape(m, H, D), sel, cfg.rope_theta)
            k = rope((a @ lw.wk).reshape(m, Hkv, D), sel, cfg.rope_theta)
            v = (a @ lw.wv).reshape(m, Hkv, D)
            keys[li][sel] = k
            vals[li][sel] = v
            o, _ = attention(q, keys[li], vals[li], vis)
            x = x + o.reshape(m, -1) @ lw.wo
            x = x + ffn(layer_norm(x, lw.ln2_g, lw.ln2_b, cfg.ln_eps), lw)
    return Fused(fused.tokens, fused.offsets, keys, vals, fused.n_ctx)


def query_forward(w: Weights, fused: Fused, query) -> Trace:
    """Query rows over the updated fused KV (fusion.py:536-540)."""
    q = np.asarray(query, np.int64)
    past = [KV(fused.keys[i], fused.values[i], np.arange(fused.n_ctx + 1))
            for i in range(len(w.layers))]
    return forward(w, q, np.arange(1 + fused.n_ctx, 1 + fused.n_ctx + q.size), past)


@dataclass
class RunOut:
    fused: Fused
    updated: Fused
    probe: Probe | None
    scores: np.ndarray | None
    selection: np.ndarray
    first_logits: np.ndarray
    answer: list[int] = field(default_factory=list)


def run(w: Weights, chunks: list[Chunk], query, ratio: float, policy="QCFuse",
        max_new: int = 0, agg="mean", bos: list[KV] | None = None) -> RunOut:
    """FusionEngine.run up to first-token logits (fusion.py:519-540), plus
    optional greedy decode (fusion.py:542-546). Policies: QCFuse, FullCompute,
    FullReuse."""
    bos = bos or bos_kv(w)
    fused = assemble(w, chunks, bos)
    pr, scores = None, None
    if policy == "QCFuse":
        if not (0.0 <= ratio <= 1.0):
            raise ValueError("ratio must be in [0, 1]")
        pr = probe(w, chunks, fused, query, "anchors", bos, layers=w.cfg.critical_layer)
        c = w.cfg.critical_layer
        scores = score_against_keys(pr.queries[c - 1], fused.keys[c - 1][1:], w.cfg.d_head, agg)
        sel = select_topn(scores, ratio)
    elif policy == "FullCompute":
        sel = np.arange(1, fused.n_ctx + 1, dtype=np.int64)
    elif policy == "FullReuse":
        sel = np.zeros(0, np.int64)
    else:
        raise ValueError(f"unsupported policy in oracle: {policy}")
    upd = recompute(w, fused, sel)
    qt = query_forward(w, upd, query)
    first = qt.logits[-1]
    answer = []
    if max_new:
        pos = np.arange(0, upd.n_ctx + 1)
        qpos = np.arange(1 + upd.n_ctx, 1 + upd.n_ctx + len(query))
        state = [KV(np.concatenate([upd.keys[i], qt.kv[i].keys]),
                    np.concatenate([upd.values[i], qt.kv[i].values]),
                    np.concatenate([pos, qpos])) for i in range(len(w.layers))]
        answer = decode_greedy(w, state, first, max_new)
    return RunOut(fused, upd, pr, scores, sel, first, answer)


def full_prefill_logits(w: Weights, fused: Fused, query) -> np.ndarray:
    """Full computation over [BOS | ctx | query] (fusion.py:496-517 first_logits)."""
    stream = np.concatenate([[BOS_ID], fused.tokens, np.asarray(query, np.int64)])
    return forward_full(w, stream, 0).logits[-1]


# --------------------------------------------------------------------------
# comparison policies                   fusion.py:352-411
# --------------------------------------------------------------------------

def layer1_recompute_pass(w: Weights, fused: Fused):
    """Layer 1 recomputed for every context token from raw embeddings at its
    fused position; attention over [BOS | new context K/V], key pos <= row pos
    (fusion.py:352-373). Returns (new K [n,Hkv,D], new V, weights [H,n,1+n])."""
    cfg = w.cfg
    lw = w.layers[0]
    n = fused.n_ctx
    H, Hkv, D = cfg.n_heads, cfg.n_kv_heads, cfg.d_head
    pos = np.arange(1, n + 1, dtype=np.int64)
    a = layer_norm(w.emb[fused.tokens], lw.ln1_g, lw.ln1_b, cfg.ln_eps)
    q = rope((a @ lw.wq).reshape(n, H, D), pos, cfg.rope_theta)
    k = rope((a @ lw.wk).reshape(n, Hkv, D), pos, cfg.rope_theta)
    v = (a @ lw.wv).reshape(n, Hkv, D)
    keys = fused.keys[0].copy()
    vals = fused.values[0].copy()
    keys[1:], vals[1:] = k, v
    visible = np.arange(n + 1)[None, :] <= pos[:, None]
    _, attn = attention(q, keys, vals, visible)
    return k, v, attn


def kv_deviation(fused: Fused, new_k, new_v) -> np.ndarray:
    """sum_h ||ΔK||_2 + sum_h ||ΔV||_2 per context row, float64 norms -> f32
    (fusion.py:375-380)."""
    dk = np.linalg.norm((new_k - fused.keys[0][1:]).astype(np.float64), axis=2).sum(axis=1)
    dv = np.linalg.norm((new_v - fused.values[0][1:]).astype(np.float64), axis=2).sum(axis=1)
    return (dk + dv).astype(np.float32)


def cacheblend_scores(w: Weights, fused: Fused) -> np.ndarray:
    """CacheBlend ranking: layer-1 KV deviation (fusion.py:382-386)."""
    k, v, _ = layer1_recompute_pass(w, fused)
    return kv_deviation(fused, k, v)


def kvshare_scores(w: Weights, fused: Fused) -> np.ndarray:
    """KVShare ranking: deviation x attention received by each context column,
    mean over heads and rows (fusion.py:388-392)."""
    k, v, attn = layer1_recompute_pass(w, fused)
    received = attn[:, :, 1:].mean(axis=(0, 1))
    return kv_deviation(fused, k, v) * received.astype(np.float32)
