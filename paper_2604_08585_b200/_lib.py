"""ctypes binding of `libqcfuse_b200.so` (the C ABI declared in
`include/qcfuse_b200.h`).

This is the reference-side FFI a maintainer would add: the reference package is
pure Python (`/root/reference/pkg/src/qcfuse`), so its kernels are bound with
ctypes. Status codes map onto the exceptions the reference raises
(`fusion.py:151,206,238,...` ValueError; NotImplementedError for shapes not
built; RuntimeError for CUDA failures). There is no fallback: if the library is
missing, importing the engine fails loudly.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

_HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("QCFUSE_B200_LIB", _HERE / "libqcfuse_b200.so"))

QCF_F32, QCF_BF16 = 0, 1
B_ROWMAJOR, B_TILE64 = 0, 1
EPI_STORE, EPI_RELU, EPI_ADD_F32 = 0, 1, 2

QCF_OK, QCF_EINVAL, QCF_ESHAPE, QCF_ECUDA, QCF_EUNSUPPORTED, QCF_EWORKSPACE = 0, -1, -2, -3, -4, -5

_P = ctypes.c_void_p
_I = ctypes.c_int
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_U64 = ctypes.c_uint64
_F = ctypes.c_float
_D = ctypes.c_double
_SZ = ctypes.c_size_t


class ChunkDesc(ctypes.Structure):
    """Mirror of `qcf_chunk_desc` (include/qcfuse_b200.h)."""
    _fields_ = [("k", _P), ("v", _P), ("layer_stride", _I64), ("n_tok", _I32), ("offset", _I32)]


# name -> (restype, argtypes); every symbol include/qcfuse_b200.h declares
SIGNATURES: dict[str, tuple] = {
    "qcf_version": (ctypes.c_char_p, []),
    "qcf_last_error": (ctypes.c_char_p, []),
    "qcf_tc_available": (_I, []),
    "qcf_simt_fallbacks": (ctypes.c_longlong, []),
    "qcf_set_strict_tc": (_I, [_I]),
    "qcf_init_uniform": (_I, [_U64, _U64, _I64, _I64, _I, _I, _P, _I64, _P]),
    "qcf_assemble": (_I, [_P, _I, _I, _P, _P, _P, _P, _I64, _I, _I, _I, _P, _P, _I64, _I, _P]),
    "qcf_assemble_rot": (_I, [_P, _I, _I, _P, _P, _P, _P, _I64, _I, _I, _I, _P, _P, _I64, _P, _I, _I, _P]),
    "qcf_assemble_range": (_I, [_P, _I, _I, _P, _P, _P, _P, _I64, _I, _I, _I, _I, _P, _P, _I64, _I, _P]),
    "qcf_assemble_range_skip": (_I, [_P, _I, _I, _P, _P, _P, _P, _I64, _I, _I, _I, _I, _P, _P, _I64, _I, _P, _P]),
    "qcf_rows_bitmap": (_I, [_P, _I64, _I, _I64, _P, _I64, _P]),
    "qcf_gather_rows": (_I, [_P, _P, _I64, _P, _I64, _P, _P, _I64, _I, _I64, _I, _P]),
    "qcf_embed": (_I, [_P, _P, _I32, _I64, _P, _I, _P, _P]),
    "qcf_layernorm": (_I, [_P, _I64, _I, _P, _P, _F, _P, _I, _P]),
    "qcf_add_layernorm": (_I, [_P, _P, _I64, _I, _P, _P, _F, _P, _I, _P]),
    "qcf_add_rows": (_I, [_P, _P, _I64, _P]),
    "qcf_lm_head": (_I, [_P, _P, _I64, _I, _P, _P, _F, _P, _I, _P, _P]),
    "qcf_decode_advance": (_I, [_P, _I, _P, _P, _P, _P, _I, _P]),
    "qcf_key_norms": (_I, [_P, _I64, _I, _I, _P, _I, _P]),
    "qcf_gemm": (_I, [_I, _P, _I64, _P, _I64, _P, _I64, _I64, _I64, _I64, _I, _I, _P]),
    "qcf_gemm_simt": (_I, [_I, _P, _I64, _P, _I64, _P, _I64, _I64, _I64, _I64, _I, _I, _P]),
    "qcf_gemm_workspace": (_SZ, [_I64, _I64, _I64]),
    "qcf_gemm_ws": (_I, [_I, _P, _I64, _P, _I64, _P, _I64, _I64, _I64, _I64, _I, _I, _I, _P, _SZ, _P]),
    "qcf_rope_qkv_scatter": (_I, [_P, _I64, _I, _I, _I, _P, _P, _P, _P, _I64, _P, _P, _P, _I, _P]),
    "qcf_gemm_qkv_rope": (_I, [_P, _I64, _P, _I64, _I, _I64, _I64, _I, _I, _I, _P, _P, _P, _I64, _P, _P, _P, _P,
                               _SZ, _P]),
    "qcf_attention": (_I, [_I, _P, _P, _P, _P, _I64, _I, _I, _I, _I64, _P, _P]),
    "qcf_attention_masked": (_I, [_I, _P, _P, _P, _P, _P, _I64, _I64, _I, _I, _I, _I64, _P, _P]),
    "qcf_attention_batched": (_I, [_I, _P, _P, _P, _P, _I64, _I, _I, _I, _I, _I64, _P, _P]),
    "qcf_attention_workspace": (_SZ, [_I64, _I, _I, _I64]),
    "qcf_attention_split": (_I, [_I64, _I, _I, _I64]),
    "qcf_attention_batched_ws": (_I, [_I, _P, _P, _P, _P, _I64, _I, _I, _I, _I, _I64, _P, _P, _SZ, _P]),
    "qcf_set_attention_kernel": (_I, [_I]),
    "qcf_set_attention_split": (_I, [_I]),
    "qcf_set_gemm_plan": (_I, [_I]),
    "qcf_score_workspace": (_SZ, [_I64, _I, _I]),
    "qcf_score": (_I, [_I, _P, _P, _I64, _I, _I, _I, _I, _D, _I, _I, _P, _P, _SZ, _P]),
    "qcf_score_batched_workspace": (_SZ, [_I64, _I, _I, _I, _I]),
    "qcf_score_batched": (_I, [_I, _P, _P, _I64, _I64, _I, _I, _I, _I, _I, _D, _I, _I, _P, _P, _SZ, _P]),
    "qcf_kv_deviation": (_I, [_I, _P, _P, _P, _P, _I64, _I, _I, _P, _P]),
    "qcf_received_attention": (_I, [_I, _P, _P, _I64, _I, _I, _I, _I, _D, _P, _P, _P, _SZ, _P]),
    "qcf_topn_workspace": (_SZ, [_I64]),
    "qcf_topn": (_I, [_P, _I64, _I64, _I32, _P, _P, _SZ, _P]),
    "qcf_topn_batched": (_I, [_P, _I64, _I, _I64, _I32, _P, _I64, _P, _I32, _P]),
    "qcf_topn_f64": (_I, [_P, _I64, _I64, _I32, _P, _P]),
    "qcf_iota_add": (_I, [_P, _I64, _I32, _P, _P]),
    "qcf_iota": (_I, [_I64, _I32, _P, _P]),
}


class QCFError(RuntimeError):
    pass


def _load():
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} not found: build the CUDA extension first "
            "(python -c 'import __graft_entry__ as g; g.build()' or `make`)")
    lib = ctypes.CDLL(str(LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def check(status: int, what: str = "") -> None:
    if status == QCF_OK:
        return
    msg = (lib.qcf_last_error() or b"").decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if status in (QCF_EINVAL, QCF_ESHAPE, QCF_EWORKSPACE):
        raise ValueError(text)
    if status == QCF_EUNSUPPORTED:
        raise NotImplementedError(text)
    raise QCFError(text)


# kernels launched per successful call (for the bench's gpu_launches claim)
KERNELS_PER_CALL = {"qcf_score": 3}
_NON_KERNEL = {"qcf_version", "qcf_last_error", "qcf_tc_available", "qcf_simt_fallbacks", "qcf_set_strict_tc", "qcf_score_workspace",
               "qcf_score_batched_workspace", "qcf_attention_workspace", "qcf_attention_split", "qcf_set_attention_kernel", "qcf_set_gemm_plan", "qcf_set_attention_split",
               "qcf_topn_workspace", "qcf_gemm_workspace"}
launch_count = 0


class Profiler:
    """Records a CUDA event pair around every C-ABI launch (eager, current
    stream). Used by bench.py's instrumented pass; never active in graphs."""

    def __init__(self):
        import torch
        self._torch = torch
        self.records: list[tuple[str, tuple, object, object]] = []

    def wrap(self, name, args, fn):
        ev0 = self._torch.cuda.Event(enable_timing=True)
        ev1 = self._torch.cuda.Event(enable_timing=True)
        ev0.record()
        st = fn()
        ev1.record()
        self.records.append((name, args, ev0, ev1))
        return st

    def summary(self) -> list[tuple[str, tuple, float]]:
        self._torch.cuda.synchronize()
        return [(n, a, e0.elapsed_time(e1)) for n, a, e0, e1 in self.records]


profiler: Profiler | None = None


def call(name: str, *args) -> None:
    global launch_count
    fn = getattr(lib, name)
    if profiler is not None and name not in _NON_KERNEL:
        st = profiler.wrap(name, args, lambda: fn(*args))
    else:
        st = fn(*args)
    check(st, name)
    if name not in _NON_KERNEL:
        launch_count += _kernels_per_call(name, args)


def _kernels_per_call(name: str, args: tuple) -> int:
    if name == "qcf_received_attention":
        n_keys, n_rows, h, ws_bytes = args[3], args[4], args[5], args[12]
        per_row = 8 * (h * n_keys + 2 * h)
        chunk = max(1, min(n_rows, (ws_bytes - 8 * n_keys - 256) // per_row))
        return 3 * ((n_rows + chunk - 1) // chunk)
    if name == "qcf_attention_batched_ws" and args[12] and args[0] == QCF_BF16:
        # split-KV adds the combine kernel
        return 2 if lib.qcf_attention_split(args[5], args[6], args[7], args[10]) > 1 else 1
    if name == "qcf_score_batched":
        # tensor-core path: 3 kernels for the whole batch; SIMT path: 3 per request
        dtype, n_req, precise = args[0], args[6], args[12]
        return 4 if (dtype == QCF_BF16 and not precise and lib.qcf_tc_available()) else 3 * n_req
    return KERNELS_PER_CALL.get(name, 1)
