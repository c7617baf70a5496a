"""ctypes binding of libkvpr.so (include/kvpr.h).

This is the only place Python touches the C-ABI.  Every wrapper takes raw
device pointers (ints) plus sizes, returns nothing, and raises ValueError for
KVPR_EINVAL (the reference's error class for shape/range problems,
numerics.py:22-32) or RuntimeError for CUDA failures.  There is no fallback:
if the library is missing, loading fails loudly.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libkvpr.so"

KVPR_OK = 0
KVPR_EINVAL = 1
KVPR_ECUDA = 2
KVPR_ECYCLE = 3

EPI_RELU = 1
EPI_F32 = 2
EPI_ACCUM = 4
EPI_W_TILED = 8

# Every symbol include/kvpr.h declares (tests check the .so exports all of them).
EXPORTS = (
    "kvpr_last_error",
    "kvpr_version",
    "kvpr_kernel_launches",
    "kvpr_sm_count",
    "kvpr_recompute_kv",
    "kvpr_recompute_tile",
    "kvpr_tiled_weight_bytes",
    "kvpr_tile_weight",
    "kvpr_linear",
    "kvpr_linear_ws",
    "kvpr_layernorm_linear_ws",
    "kvpr_decode_attention",
    "kvpr_decode_attention_ragged",
    "kvpr_prefill_attention",
    "kvpr_layernorm",
    "kvpr_embed",
    "kvpr_argmax",
    "kvpr_copy_async",
    "kvpr_copy_batch_async",
    "kvpr_copy_2d_async",
    "kvpr_list_schedule",
    "kvpr_kv4_page_bytes",
    "kvpr_kv4_quantize",
    "kvpr_kv4_dequantize",
    "kvpr_decode_attention_kv4",
    "kvpr_decode_layer_tail_supported",
    "kvpr_decode_layer_tail",
    "kvpr_decoder_create",
    "kvpr_decoder_destroy",
    "kvpr_decoder_run",
    "kvpr_decoder_set_timing",
    "kvpr_decoder_kernel_stats",
    "kvpr_decoder_timeline",
    "kvpr_decoder_launches",
    "kvpr_ipc_handle_bytes",
    "kvpr_ipc_alloc",
    "kvpr_ipc_open",
    "kvpr_ipc_close",
    "kvpr_ipc_free",
    "kvpr_linear_allreduce",
    "kvpr_debug_sm_pull",
)

TP_MAX_WORLD = 8
TP_MAX_TILES = 512


class OutSeg(ctypes.Structure):
    _fields_ = [("ptr", ctypes.c_void_p), ("group_stride", ctypes.c_longlong)]


class Epilogue(ctypes.Structure):
    _fields_ = [
        ("bias", ctypes.c_void_p),
        ("seg_width", ctypes.c_int),
        ("row_group", ctypes.c_int),
        ("ld", ctypes.c_longlong),
        ("seg", OutSeg * 3),
        ("scale", ctypes.c_float),
        ("scale_cols", ctypes.c_int),
        ("flags", ctypes.c_int),
    ]


class LayerDesc(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in (
        "ln1_g", "ln1_b", "wqkv", "bqkv", "wo", "bo", "ln2_g", "ln2_b", "w1", "b1", "w2", "b2",
        "host_x", "host_kv", "dev_x")]


class DecoderDesc(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in (
        "layers", "batch", "hidden", "heads", "ffn", "vocab", "capacity", "chunks", "nbuf", "x_resident")] + [
        ("eps", ctypes.c_float)] + [(n, ctypes.c_void_p) for n in (
            "embed", "pos", "lnf_g", "lnf_b", "kv_dev", "x_dev", "hres", "q", "attn", "y", "mid", "zf", "logits",
            "tok", "ws")] + [("ws_bytes", ctypes.c_size_t)] + [(n, ctypes.c_void_p) for n in (
                "compute_stream", "h2d_stream", "d2h_stream")] + [("chunk_rows", ctypes.c_int), ("chunk_wave", ctypes.c_int),
                                                      ("recompute_stream", ctypes.c_void_p), ("fused_tail", ctypes.c_int),
                                                      ("zero_copy", ctypes.c_int), ("dma_group", ctypes.c_int)]


class LayerTailDesc(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in ("batch", "hidden", "heads", "head_dim", "ffn", "seq_len")] + [
        ("scale", ctypes.c_float), ("eps", ctypes.c_float)] + [(n, ctypes.c_void_p) for n in (
            "q", "kv_pages", "attn", "wo", "bo", "hres", "ln2_g", "ln2_b", "w1", "b1", "mid", "w2", "b2", "lnx_g",
            "lnx_b", "lnx_out")] + [("lnx_ld", ctypes.c_longlong)] + [(n, ctypes.c_void_p) for n in (
                "wqkv_next", "bqkv_next", "q_next", "page_next", "kv_host")] + [
                    ("host_lo", ctypes.c_int), ("host_hi", ctypes.c_int)] + [(n, ctypes.c_void_p) for n in (
                        "x_store_next", "page_store_next", "ws")] + [("ws_bytes", ctypes.c_size_t)]


_lib: ctypes.CDLL | None = None

class TpPeers(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int), ("world", ctypes.c_int),
                ("recv", ctypes.c_void_p * TP_MAX_WORLD), ("resid", ctypes.c_void_p * TP_MAX_WORLD),
                ("flags", ctypes.c_void_p * TP_MAX_WORLD), ("err", ctypes.c_void_p)]


_vp = ctypes.c_void_p
_i = ctypes.c_int
_ll = ctypes.c_longlong
_f = ctypes.c_float
_sz = ctypes.c_size_t

_SIGS = {
    "kvpr_last_error": ([], ctypes.c_char_p),
    "kvpr_version": ([], _i),
    "kvpr_kernel_launches": ([], _ll),
    "kvpr_sm_count": ([_i], _i),
    "kvpr_recompute_kv": ([_vp, _vp, _vp, _vp, _i, _i, _i, _i, _vp], _i),
    "kvpr_recompute_tile": ([_i, _i, _i, _i], _i),
    "kvpr_tiled_weight_bytes": ([_i, _i], _sz),
    "kvpr_tile_weight": ([_vp, _ll, _i, _i, _vp, _vp], _i),
    "kvpr_linear": ([_vp, _ll, _vp, _ll, _i, _i, _i, ctypes.POINTER(Epilogue), _i, _vp], _i),
    "kvpr_linear_ws": ([_vp, _ll, _vp, _ll, _i, _i, _i, ctypes.POINTER(Epilogue), _i, _vp, _sz, _vp], _i),
    "kvpr_layernorm_linear_ws": ([_vp, _ll, _vp, _vp, _f, _vp, _ll, _vp, _ll, _i, _i, _i, ctypes.POINTER(Epilogue), _i,
                                  _vp, _sz, _vp], _i),
    "kvpr_decode_attention": ([_vp, _vp, _vp, _vp, _sz, _i, _i, _i, _i, _f, _vp], _i),
    "kvpr_decode_attention_ragged": ([_vp, _vp, _vp, _vp, _vp, _sz, _i, _i, _i, _i, _f, _vp], _i),
    "kvpr_prefill_attention": ([_vp, _vp, _vp, _i, _i, _i, _i, _f, _vp], _i),
    "kvpr_layernorm": ([_vp, _ll, _vp, _vp, _vp, _ll, _i, _i, _f, _vp], _i),
    "kvpr_embed": ([_vp, _vp, _vp, _vp, _i, _i, _i, _i, _i, _vp], _i),
    "kvpr_argmax": ([_vp, _ll, _i, _i, _vp, _vp, _vp], _i),
    "kvpr_copy_async": ([_vp, _vp, _sz, _vp], _i),
    "kvpr_copy_batch_async": ([ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.POINTER(_sz), _sz, _vp], _i),
    "kvpr_copy_2d_async": ([_vp, _sz, _vp, _sz, _sz, _sz, _vp], _i),
    "kvpr_list_schedule": ([ctypes.c_longlong] + [_vp] * 5 + [_i, _vp, _vp], _i),
    "kvpr_kv4_page_bytes": ([_i, _i], _sz),
    "kvpr_kv4_quantize": ([_vp, _vp, _i, _i, _i, _i, _vp], _i),
    "kvpr_kv4_dequantize": ([_vp, _vp, _i, _i, _i, _i, _vp], _i),
    "kvpr_decode_attention_kv4": ([_vp, _vp, _vp, _i, _i, _vp, _vp, _sz, _i, _i, _i, _i, _f, _vp], _i),
    "kvpr_decode_layer_tail_supported": ([_i, _i, _i, _i], _i),
    "kvpr_decode_layer_tail": ([ctypes.POINTER(LayerTailDesc), _vp], _i),
    "kvpr_decoder_create": ([ctypes.POINTER(DecoderDesc), ctypes.POINTER(LayerDesc), ctypes.POINTER(_vp)], _i),
    "kvpr_decoder_destroy": ([_vp], _i),
    "kvpr_decoder_run": ([_vp, _i, ctypes.POINTER(_i), _i, _vp, _vp], _i),
    "kvpr_decoder_set_timing": ([_vp, _i], _i),
    "kvpr_decoder_kernel_stats": ([_vp, _i, ctypes.POINTER(_i), ctypes.POINTER(ctypes.c_double),
                                   ctypes.POINTER(ctypes.c_double)], _i),
    "kvpr_decoder_timeline": ([_vp, ctypes.POINTER(ctypes.c_float), _i, ctypes.POINTER(ctypes.c_float), _i], _i),
    "kvpr_decoder_launches": ([_vp], _ll),
    "kvpr_ipc_handle_bytes": ([], _sz),
    "kvpr_debug_sm_pull": ([_vp, _vp, _sz, _i, _vp], _i),
    "kvpr_ipc_alloc": ([_sz, ctypes.POINTER(_vp), _vp], _i),
    "kvpr_ipc_open": ([_vp, ctypes.POINTER(_vp)], _i),
    "kvpr_ipc_close": ([_vp], _i),
    "kvpr_ipc_free": ([_vp], _i),
    "kvpr_linear_allreduce": ([_vp, _ll, _vp, _ll, _i, _i, _i, _vp, ctypes.POINTER(TpPeers), ctypes.c_uint, _vp],
                              _i),
}


def load(path: str | os.PathLike | None = None) -> ctypes.CDLL:
    """Load (once) and type the shared library; raises if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise RuntimeError(
            f"libkvpr.so not found at {p}; build it with `python -m paper_2411_17089_b200.csrc.build` "
            "(there is no CPU fallback)"
        )
    lib = ctypes.CDLL(str(p))
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def last_error() -> str:
    return load().kvpr_last_error().decode()


def check(rc: int, what: str) -> None:
    if rc == KVPR_OK:
        return
    msg = f"{what}: {last_error()}"
    if rc == KVPR_EINVAL:
        raise ValueError(msg)
    raise RuntimeError(msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)


def make_epilogue(
    segs,
    seg_width: int,
    ld: int,
    row_group: int,
    bias: int | None = None,
    scale: float = 1.0,
    scale_cols: int = 0,
    flags: int = 0,
) -> Epilogue:
    """segs: list of (ptr, group_stride) pairs, one per output column segment."""
    e = Epilogue()
    e.bias = bias or None
    e.seg_width = seg_width
    e.row_group = row_group
    e.ld = ld
    for i, (ptr, gs) in enumerate(segs):
        e.seg[i].ptr = ptr
        e.seg[i].group_stride = gs
    e.scale = scale
    e.scale_cols = scale_cols
    e.flags = flags
    return e
