"""Model configuration and device-resident weights.

Mirrors the reference's `ModelConfig` (model.py:74-118, same fields, defaults,
validation and `to_dict`, so store fingerprints agree) and generates the
reference's splitmix64 weights ON THE GPU with `qcf_init_uniform`
(model.py:225-257), bit-identical to the reference's float32 draws; bf16 mode
rounds those float32 values to nearest bf16.

Device layout (chosen for the tcgen05 GEMM, both operands K-major):
  emb            f32  [V][d]            (embedding gather + tied lm-head)
  wqkv           dt   [(H+2Hkv)·D][d]   = [Wq | Wk | Wv]ᵀ
  wo             dt   [d][d]            = Woᵀ
  w1             dt   [F][d]            = W1ᵀ
  w2             dt   [d][F]            = W2ᵀ
  ln*_g / ln*_b  f32  [d]
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import QCF_BF16, QCF_F32, call

BOS_ID = 256
EOS_ID = 257
PAD_ID = 258
VOCAB_SIZE = 259

DTYPES = {"f32": (QCF_F32, torch.float32), "bf16": (QCF_BF16, torch.bfloat16)}


@dataclass(frozen=True)
class ModelConfig:
    """model.py:74-118."""
    n_layers: int = 4
    n_heads: int = 2
    d_model: int = 32
    d_head: int = 16
    d_ff: int = 64
    vocab_size: int = VOCAB_SIZE
    rope_theta: float = 10000.0
    ln_eps: float = 1e-5
    seed: int = 1234
    critical_layer: int | None = None  # 1-based; defaults to ceil(n_layers / 2)
    # GQA extension (not in the reference, which is MHA-only): kv heads shared by
    # n_heads / n_kv_heads query heads; None = n_heads (reference-exact MHA)
    n_kv_heads: int | None = None

    def __post_init__(self):
        if self.critical_layer is None:
            object.__setattr__(self, "critical_layer", math.ceil(self.n_layers / 2))
        if self.n_kv_heads is None:
            object.__setattr__(self, "n_kv_heads", self.n_heads)
        self.validate()

    def validate(self) -> None:
        if self.d_model != self.n_heads * self.d_head:
            raise ValueError("d_model must equal n_heads * d_head")
        if self.n_layers < 4:
            raise ValueError("n_layers must be >= 4")
        if not (1 < self.critical_layer < self.n_layers):
            raise ValueError("critical_layer must satisfy 1 < critical_layer < n_layers")
        if self.vocab_size != VOCAB_SIZE:
            raise ValueError(f"vocab_size must be {VOCAB_SIZE} (256 bytes + BOS/EOS/PAD)")
        if self.d_head % 2 != 0:
            raise ValueError("d_head must be even for rotary pairs")
        if self.rope_theta <= 0 or self.ln_eps <= 0:
            raise ValueError("rope_theta and ln_eps must be positive")
        if self.n_kv_heads < 1 or self.n_heads % self.n_kv_heads != 0:
            raise ValueError("n_heads must be a multiple of n_kv_heads")

    def to_dict(self) -> dict:
        """model.py:108-118; n_kv_heads appears only for GQA so MHA fingerprints
        equal the reference's (store.py:46-49)."""
        out = {k: getattr(self, k) for k in ("n_layers", "n_heads", "d_model", "d_head", "d_ff",
                                             "vocab_size", "rope_theta", "ln_eps", "seed",
                                             "critical_layer")}
        if self.n_kv_heads != self.n_heads:
            out["n_kv_heads"] = self.n_kv_heads
        return out

    @property
    def kv_dim(self) -> int:
        return self.n_kv_heads * self.d_head

    def layer_params(self) -> int:
        d, f = self.d_model, self.d_ff
        return 2 * d * d + 2 * d * self.kv_dim + 2 * d * f


def tokenize(text) -> list[int]:
    """BOS + bytes (model.py:181-185)."""
    data = text.encode("utf-8") if isinstance(text, str) else bytes(text)
    return [BOS_ID] + list(data)


def byte_tokens(text) -> list[int]:
    """Bytes, no BOS (model.py:188-191)."""
    data = text.encode("utf-8") if isinstance(text, str) else bytes(text)
    return list(data)


def render_tokens(token_ids) -> str:
    """Printable rendering (model.py:194-222)."""
    out, buf = [], bytearray()

    def flush():
        if buf:
            out.append(buf.decode("utf-8", errors="backslashreplace"))
            buf.clear()

    for t in token_ids:
        t = int(t)
        if t < 256:
            if 32 <= t < 127 or t in (9, 10):
                buf.append(t)
            else:
                flush()
                out.append(f"\\x{t:02x}")
        else:
            flush()
            out.append({BOS_ID: "<bos>", EOS_ID: "<eos>", PAD_ID: "<pad>"}[t])
    flush()
    return "".join(out)


def cuda_stream(stream: torch.cuda.Stream | None = None):
    s = stream or torch.cuda.current_stream()
    return s.cuda_stream


@dataclass
class DeviceLayer:
    wqkv: torch.Tensor
    wo: torch.Tensor
    w1: torch.Tensor
    w2: torch.Tensor
    ln1_g: torch.Tensor
    ln1_b: torch.Tensor
    ln2_g: torch.Tensor
    ln2_b: torch.Tensor


@dataclass(eq=False)
class ModelWeights:
    """Device-resident weights (the reference's ModelWeights, model.py:136-141)."""
    config: ModelConfig
    dtype: str
    emb: torch.Tensor
    layers: list[DeviceLayer]
    ln_f_gain: torch.Tensor
    ln_f_bias: torch.Tensor
    device: torch.device = field(default_factory=lambda: torch.device("cuda"))
    b_layout: int = _lib.B_ROWMAJOR   # projection weights tile-major (B_TILE64) in bf16 mode
    # fp32 scoring mode: float32 copies of layers 1..c (the probe that produces
    # Q_c runs on them, so selection is the reference's bit for bit)
    probe32: "ModelWeights | None" = None

    @property
    def qcf_dtype(self) -> int:
        return DTYPES[self.dtype][0]

    @property
    def torch_dtype(self) -> torch.dtype:
        return DTYPES[self.dtype][1]

    @property
    def token_embedding(self) -> np.ndarray:
        return self.emb.cpu().numpy()

    @classmethod
    def from_host(cls, config: ModelConfig, token_embedding, layers, dtype="bf16",
                  device="cuda", scoring: str = "native") -> "ModelWeights":
        """From host arrays in the reference layout: layers is a sequence of
        objects with wq wk wv wo w1 w2 ([d_in][d_out]) and ln gains/biases.
        scoring="fp32" (bf16 weights) also keeps float32 copies of layers 1..c."""
        if scoring not in ("native", "fp32"):
            raise ValueError(f"unknown scoring mode: {scoring}")
        probe32 = None
        if scoring == "fp32" and dtype == "bf16":
            probe32 = cls.from_host(config, token_embedding, list(layers)[:config.critical_layer], "f32", device)
        dev = torch.device(device)
        tdt = DTYPES[dtype][1]

        def t(a, dt=tdt):
            return torch.as_tensor(np.ascontiguousarray(a)).to(device=dev, dtype=dt)

        dl = []
        for lw in layers:
            wqkv = np.concatenate([lw.wq, lw.wk, lw.wv], axis=1).T
            dl.append(DeviceLayer(t(wqkv), t(lw.wo.T), t(lw.w1.T), t(lw.w2.T),
                                  t(_get(lw, "ln1_gain", "ln1_g"), torch.float32),
                                  t(_get(lw, "ln1_bias", "ln1_b"), torch.float32),
                                  t(_get(lw, "ln2_gain", "ln2_g"), torch.float32),
                                  t(_get(lw, "ln2_bias", "ln2_b"), torch.float32)))
        d = config.d_model
        ones = torch.ones(d, dtype=torch.float32, device=dev)
        tiled = use_tiled_weights(config, dtype)
        _tile_layers(dl, tiled)
        return cls(config, dtype, t(token_embedding, torch.float32), dl, ones, torch.zeros_like(ones), dev,
                   _lib.B_TILE64 if tiled else _lib.B_ROWMAJOR, probe32)


def tile64(w: torch.Tensor) -> torch.Tensor:
    """[N][K] -> tile-major [N/64][K/64][64][64] (QCF_B_TILE64, include/qcfuse_b200.h)."""
    n, k = w.shape
    return w.view(n // 64, 64, k // 64, 64).permute(0, 2, 1, 3).contiguous().view(n, k)


def untile64(w: torch.Tensor) -> torch.Tensor:
    n, k = w.shape
    return w.view(n // 64, k // 64, 64, 64).permute(0, 2, 1, 3).contiguous().view(n, k)


def use_tiled_weights(config: ModelConfig, dtype: str) -> bool:
    """bf16 on a tcgen05 device with every projection dim a multiple of 64."""
    if dtype != "bf16" or not torch.cuda.is_available() or not _lib.lib.qcf_tc_available():
        return False
    return all(x % 64 == 0 for x in (config.d_model, config.d_ff, config.n_heads * config.d_head, config.kv_dim))


def _tile_layers(layers: list, on: bool) -> None:
    if not on:
        return
    for lw in layers:
        lw.wqkv, lw.wo, lw.w1, lw.w2 = tile64(lw.wqkv), tile64(lw.wo), tile64(lw.w1), tile64(lw.w2)


def _get(obj, *names):
    for n in names:
        if hasattr(obj, n):
            return getattr(obj, n)
    raise AttributeError(names[0])


def init_weights(config: ModelConfig, dtype: str = "bf16", device="cuda",
                 layers: int | None = None, scoring: str = "native") -> ModelWeights:
    """GPU restatement of init_weights (model.py:225-257): stream order
    embedding, then per layer wq wk wv wo w1 w2, each row-major. GQA: wk/wv are
    [d][Hkv*D] in the same stream order (reduces to the reference at Hkv == H).
    scoring="fp32" with bf16 weights also draws float32 copies of layers 1..c
    (`probe32`, the fp32 scoring mode's probe weights)."""
    config.validate()
    if scoring not in ("native", "fp32"):
        raise ValueError(f"unknown scoring mode: {scoring}")
    dev = torch.device(device)
    qdt, tdt = DTYPES[dtype]
    d, f, V = config.d_model, config.d_ff, config.vocab_size
    s = cuda_stream()
    seed = config.seed & ((1 << 64) - 1)
    emb = torch.empty(V, d, dtype=torch.float32, device=dev)
    call("qcf_init_uniform", seed, 0, V, d, 0, QCF_F32, emb.data_ptr(), d, s)
    off = V * d
    n_build = config.n_layers if layers is None else layers
    tiled = use_tiled_weights(config, dtype)
    dl = []
    kvd = config.kv_dim
    for _ in range(n_build):
        wqkv = torch.empty(d + 2 * kvd, d, dtype=tdt, device=dev)
        wo = torch.empty(d, d, dtype=tdt, device=dev)
        w1 = torch.empty(f, d, dtype=tdt, device=dev)
        w2 = torch.empty(d, f, dtype=tdt, device=dev)
        esz = wqkv.element_size()
        row = 0
        for cols in (d, kvd, kvd):  # wq, wk, wv -> consecutive row blocks of wqkv (K-major)
            call("qcf_init_uniform", seed, off, d, cols, 1, qdt, wqkv.data_ptr() + row * d * esz, d, s)
            off += d * cols
            row += cols
        call("qcf_init_uniform", seed, off, d, d, 1, qdt, wo.data_ptr(), d, s)
        off += d * d
        call("qcf_init_uniform", seed, off, d, f, 1, qdt, w1.data_ptr(), d, s)
        off += d * f
        call("qcf_init_uniform", seed, off, f, d, 1, qdt, w2.data_ptr(), f, s)
        off += f * d
        ones = torch.ones(d, dtype=torch.float32, device=dev)
        zeros = torch.zeros(d, dtype=torch.float32, device=dev)
        layer = DeviceLayer(wqkv, wo, w1, w2, ones, zeros, ones.clone(), zeros.clone())
        _tile_layers([layer], tiled)
        dl.append(layer)
    ones = torch.ones(d, dtype=torch.float32, device=dev)
    probe32 = None
    if scoring == "fp32" and dtype == "bf16":
        probe32 = init_weights(config, "f32", device, layers=min(n_build, config.critical_layer))
    return ModelWeights(config, dtype, emb, dl, ones, torch.zeros_like(ones), dev,
                        _lib.B_TILE64 if tiled else _lib.B_ROWMAJOR, probe32)


class RopeTable:
    """float64 cos/sin [n_pos][D/2] on the device, built with numpy exactly as
    the reference builds its angles (model.py:264-280): angle = pos · θ^(−2j/D)
    in float64, np.cos / np.sin. Grows on demand; positions index rows."""

    def __init__(self, d_head: int, theta: float, device, n_pos: int = 8192):
        self.d_head, self.theta, self.device = d_head, theta, torch.device(device)
        self.n_pos = 0
        self.cos = self.sin = self.cs32 = None
        # tables replaced by growth stay allocated: captured graphs and launches
        # still in flight on other streams keep valid pointers (each old table is
        # a prefix of the new one, so their positions still read correct values)
        self.retired: list[tuple] = []
        self.ensure(n_pos)

    def ensure(self, n_pos: int) -> None:
        if n_pos <= self.n_pos:
            return
        if self.cos is not None:
            self.retired.append((self.cos, self.sin, self.cs32))
        n = max(n_pos, 2 * self.n_pos)
        j = np.arange(self.d_head // 2, dtype=np.float64)
        inv = self.theta ** (-2.0 * j / self.d_head)
        ang = np.arange(n, dtype=np.float64)[:, None] * inv[None, :]
        self.cos = torch.as_tensor(np.cos(ang)).to(self.device)
        self.sin = torch.as_tensor(np.sin(ang)).to(self.device)
        # (cos, sin) pairs in float32 for the bf16 tcgen05 QKV epilogue (which
        # rotates in fp32: same values as casting the float64 tables there)
        self.cs32 = torch.stack([self.cos, self.sin], -1).float().contiguous()
        self.n_pos = n
