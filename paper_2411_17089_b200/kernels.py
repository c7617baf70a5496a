"""Torch-tensor front end over the C-ABI (device plumbing only).

Each function checks dtype/device/contiguity, pulls raw pointers and the
current CUDA stream, and calls exactly one libkvpr entry point.  Nothing here
computes on the CPU; a missing library or a non-CUDA tensor is an error.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch

from . import _lib


def _stream(stream: torch.cuda.Stream | None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _need(t: torch.Tensor, dtype: torch.dtype, name: str) -> None:
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")


def recompute_kv(x: torch.Tensor, w_kv: torch.Tensor, b_kv: torch.Tensor | None, kv_pages: torch.Tensor,
                 batch: int, pos_begin: int, pos_end: int, stream=None) -> None:
    """K1: K/V of positions [pos_begin, pos_end) from X, written into the page buffer."""
    _need(x, torch.float16, "x")
    _need(w_kv, torch.float16, "w_kv")
    _need(kv_pages, torch.float16, "kv_pages")
    hidden = w_kv.shape[1]
    if w_kv.shape[0] != 2 * hidden or not w_kv.is_contiguous():
        raise ValueError("w_kv must be contiguous [2*hidden, hidden]")
    if b_kv is not None:
        _need(b_kv, torch.float16, "b_kv")
    need_x = pos_end * batch * hidden
    need_kv = pos_end * 2 * batch * hidden
    if x.numel() < need_x or kv_pages.numel() < need_kv:
        raise ValueError("x / kv_pages too small for the requested positions")
    _lib.call(
        "kvpr_recompute_kv",
        x.data_ptr(), w_kv.data_ptr(), b_kv.data_ptr() if b_kv is not None else None, kv_pages.data_ptr(),
        batch, pos_begin, pos_end, hidden, _stream(stream),
    )


@dataclass(frozen=True)
class TiledWeight:
    """A weight W [N, K] in kvpr_tile_weight's box-tiled layout (decode GEMMs, M <= 64)."""

    data: torch.Tensor
    N: int
    K: int

    @property
    def shape(self):
        return (self.N, self.K)


def linear(a: torch.Tensor, w, epi: _lib.Epilogue, M: int | None = None, bn: int = 0,
           stream=None, lda: int | None = None, ws: torch.Tensor | None = None) -> None:
    """out = epilogue(A[M,K] . W[N,K]^T + bias) via the tcgen05 GEMM (ws enables stream-K for decode GEMMs).
    w: [N, K] fp16 tensor, or a TiledWeight (streams 16 KB-contiguous boxes; swap-AB decode GEMM only)."""
    _need(a, torch.float16, "a")
    if isinstance(w, TiledWeight):
        _need(w.data, torch.float16, "w")
        N, K, wptr, ldw = w.N, w.K, w.data.data_ptr(), 64
        epi.flags |= _lib.EPI_W_TILED
    else:
        _need(w, torch.float16, "w")
        (N, K), wptr, ldw = w.shape, w.data_ptr(), w.stride(0)
    if M is None:
        M = a.shape[0]
    lda = K if lda is None else lda
    if ws is None:
        _lib.call("kvpr_linear", a.data_ptr(), lda, wptr, ldw, M, N, K, epi, bn, _stream(stream))
    else:
        _lib.call("kvpr_linear_ws", a.data_ptr(), lda, wptr, ldw, M, N, K, epi, bn,
                  ws.data_ptr(), ws.numel() * ws.element_size(), _stream(stream))


def tile_weight(w: torch.Tensor, stream=None) -> TiledWeight:
    """W [N, K] fp16 -> its box-tiled copy for the decode GEMM (kvpr_tile_weight)."""
    _need(w, torch.float16, "w")
    N, K = w.shape
    out = torch.empty(_lib.load().kvpr_tiled_weight_bytes(N, K) // 2, dtype=torch.float16, device=w.device)
    _lib.call("kvpr_tile_weight", w.data_ptr(), w.stride(0), N, K, out.data_ptr(), _stream(stream))
    return TiledWeight(out, N, K)


def linear_simple(a: torch.Tensor, w: torch.Tensor, bias: torch.Tensor | None, out: torch.Tensor,
                  flags: int = 0, bn: int = 0, stream=None, ws: torch.Tensor | None = None) -> torch.Tensor:
    """Row-major out[M, N] (fp16 or fp32 per flags) = epilogue(a . w^T + bias)."""
    N = w.shape[0]
    M = a.shape[0]
    if out.dtype == torch.float32:
        flags |= _lib.EPI_F32
    # one output segment covering all N columns, rows at out.stride(0)
    epi = _lib.make_epilogue([(out.data_ptr(), 0)], seg_width=((N + 31) // 32) * 32, ld=out.stride(0), row_group=M,
                             bias=bias.data_ptr() if bias is not None else None, flags=flags)
    linear(a, w, epi, M=M, bn=bn, stream=stream, ws=ws)
    return out


def decode_attention(q: torch.Tensor, kv_pages: torch.Tensor, out: torch.Tensor, ws: torch.Tensor | None,
                     batch: int, heads: int, head_dim: int, seq_len: int, scale: float | None = None,
                     stream=None) -> torch.Tensor:
    """K2: softmax(scale * K q) V per (sequence, head) over pages [0, seq_len)."""
    _need(q, torch.float16, "q")
    _need(kv_pages, torch.float16, "kv_pages")
    _need(out, torch.float16, "out")
    if scale is None:
        scale = 1.0 / math.sqrt(head_dim)
    ws_ptr, ws_bytes = (ws.data_ptr(), ws.numel() * ws.element_size()) if ws is not None else (None, 0)
    _lib.call(
        "kvpr_decode_attention",
        q.data_ptr(), kv_pages.data_ptr(), out.data_ptr(), ws_ptr, ws_bytes,
        batch, heads, head_dim, seq_len, float(scale), _stream(stream),
    )
    return out


def layer_tail_supported(batch: int, hidden: int, heads: int, ffn: int) -> bool:
    """Shapes the fused small-batch layer tail handles (batch <= 8, hidden <= 1024, ffn <= 4096, head_dim 64/128)."""
    return bool(_lib.load().kvpr_decode_layer_tail_supported(batch, hidden, heads, ffn))


def layer_tail(q: torch.Tensor, kv_pages: torch.Tensor, seq_len: int, lw, hres: torch.Tensor, attn: torch.Tensor,
               mid: torch.Tensor, ws: torch.Tensor, heads: int, eps: float, lnx: tuple | None = None,
               qkv_next: tuple | None = None, host_kv: tuple | None = None, stores: tuple | None = None,
               stream=None) -> None:
    """K2 -> out-proj + residual -> LN2 -> fc1 + ReLU -> fc2 + residual in one cooperative kernel
    (kvpr_decode_layer_tail).  lw: the layer's weights (wo, bo, ln2_g, ln2_b, w1, b1, w2, b2);
    lnx = (gamma, beta, out fp16 [batch][>= hidden]) for the optional LayerNorm of the new residual;
    qkv_next = (wqkv [3h, h], bqkv [3h], q_out [batch, h], page [2, batch, h]) for the next layer's q/k/v
    of the new token from that LayerNorm (needs lnx); host_kv = (page-locked KV store of the layer, lo, hi): attention
    positions [lo, hi) read from it over PCIe (zero-copy); stores = (host X row or None, host KV page) the
    normalised rows / the next k, v page are also written to (page-locked, zero-copy)."""
    batch, hidden = q.shape
    for t, n in ((q, "q"), (kv_pages, "kv_pages"), (attn, "attn"), (mid, "mid")):
        _need(t, torch.float16, n)
    _need(hres, torch.float32, "hres")
    d = _lib.LayerTailDesc()
    d.batch, d.hidden, d.heads, d.head_dim, d.ffn, d.seq_len = batch, hidden, heads, hidden // heads, mid.shape[1], seq_len
    d.scale, d.eps = 1.0 / math.sqrt(hidden // heads), eps
    d.q, d.kv_pages, d.attn, d.hres, d.mid = q.data_ptr(), kv_pages.data_ptr(), attn.data_ptr(), hres.data_ptr(), \
        mid.data_ptr()
    for name in ("wo", "bo", "ln2_g", "ln2_b", "w1", "b1", "w2", "b2"):
        setattr(d, name, getattr(lw, name).data_ptr())
    if lnx is not None:
        g, b, out = lnx
        _need(out, torch.float16, "lnx out")
        d.lnx_g, d.lnx_b, d.lnx_out, d.lnx_ld = g.data_ptr(), b.data_ptr(), out.data_ptr(), out.stride(0)
    if qkv_next is not None:
        wq, bq, qo, page = qkv_next
        for t, n in ((wq, "wqkv"), (bq, "bqkv"), (qo, "q_next"), (page, "page_next")):
            _need(t, torch.float16, n)
        d.wqkv_next, d.bqkv_next, d.q_next, d.page_next = wq.data_ptr(), bq.data_ptr(), qo.data_ptr(), page.data_ptr()
    if host_kv is not None:
        kvh, lo, hi = host_kv
        if kvh.is_cuda:
            raise ValueError("host_kv must be a page-locked host tensor")
        d.kv_host, d.host_lo, d.host_hi = kvh.data_ptr(), lo, hi
    if stores is not None:
        xs, ps = stores
        d.x_store_next = xs.data_ptr() if xs is not None else None
        d.page_store_next = ps.data_ptr() if ps is not None else None
    d.ws, d.ws_bytes = ws.data_ptr(), ws.numel() * ws.element_size()
    import ctypes

    _lib.call("kvpr_decode_layer_tail", ctypes.byref(d), _stream(stream))


def decode_attention_ragged(q: torch.Tensor, kv_pages: torch.Tensor, seq_lens: torch.Tensor, out: torch.Tensor,
                            ws: torch.Tensor | None, heads: int, head_dim: int, scale: float | None = None,
                            stream=None) -> torch.Tensor:
    """K2 over a ragged batch: sequence b attends over pages [0, seq_lens[b]) (device int32 [batch],
    1 <= seq_lens[b] <= kv_pages.shape[0]); kv_pages [max_len][2][batch][hidden]."""
    _need(q, torch.float16, "q")
    _need(kv_pages, torch.float16, "kv_pages")
    _need(seq_lens, torch.int32, "seq_lens")
    _need(out, torch.float16, "out")
    batch = q.shape[0]
    if seq_lens.numel() != batch:
        raise ValueError(f"seq_lens has {seq_lens.numel()} entries for a batch of {batch}")
    if scale is None:
        scale = 1.0 / math.sqrt(head_dim)
    ws_ptr, ws_bytes = (ws.data_ptr(), ws.numel() * ws.element_size()) if ws is not None else (None, 0)
    _lib.call("kvpr_decode_attention_ragged", q.data_ptr(), kv_pages.data_ptr(), seq_lens.data_ptr(), out.data_ptr(),
              ws_ptr, ws_bytes, batch, heads, head_dim, int(kv_pages.shape[0]), float(scale), _stream(stream))
    return out


def decode_attention_kv4(q: torch.Tensor, kv_pages: torch.Tensor, qpages: torch.Tensor, q_lo: int, q_hi: int,
                         out: torch.Tensor, ws: torch.Tensor | None, batch: int, heads: int, head_dim: int,
                         seq_len: int, scale: float | None = None, stream=None) -> torch.Tensor:
    """K2 with positions [q_lo, q_hi) read from 4-bit compressed pages (dequantised in registers,
    same bits as kv4_dequantize followed by decode_attention)."""
    _need(q, torch.float16, "q")
    _need(kv_pages, torch.float16, "kv_pages")
    _need(qpages, torch.uint8, "qpages")
    _need(out, torch.float16, "out")
    if scale is None:
        scale = 1.0 / math.sqrt(head_dim)
    ws_ptr, ws_bytes = (ws.data_ptr(), ws.numel() * ws.element_size()) if ws is not None else (None, 0)
    _lib.call(
        "kvpr_decode_attention_kv4",
        q.data_ptr(), kv_pages.data_ptr(), qpages.data_ptr(), q_lo, q_hi, out.data_ptr(), ws_ptr, ws_bytes,
        batch, heads, head_dim, seq_len, float(scale), _stream(stream),
    )
    return out


def prefill_attention(q: torch.Tensor, kv_pages: torch.Tensor, out: torch.Tensor, batch: int, heads: int,
                      head_dim: int, seq_len: int, scale: float | None = None, stream=None) -> torch.Tensor:
    """Causal attention of positions [0, seq_len): q / out [pos][batch][heads * head_dim] and the pages
    [pos][2][batch][heads * head_dim], all contiguous fp16 (the kernel's TMA maps assume those strides)."""
    for t, name in ((q, "q"), (kv_pages, "kv_pages"), (out, "out")):
        _need(t, torch.float16, name)
        if not t.is_contiguous():
            raise ValueError(f"{name} must be contiguous")
    h = heads * head_dim
    if q.numel() < seq_len * batch * h or out.numel() < seq_len * batch * h or kv_pages.numel() < seq_len * 2 * batch * h:
        raise ValueError("prefill_attention: q / out need seq_len x batch x hidden and kv_pages seq_len x 2 x batch x "
                         "hidden elements")
    if scale is None:
        scale = 1.0 / math.sqrt(head_dim)
    _lib.call(
        "kvpr_prefill_attention",
        q.data_ptr(), kv_pages.data_ptr(), out.data_ptr(), batch, heads, head_dim, seq_len, float(scale),
        _stream(stream),
    )
    return out


def layernorm(x: torch.Tensor, gamma: torch.Tensor, beta: torch.Tensor, out: torch.Tensor, rows: int | None = None,
              eps: float = 1e-5, stream=None) -> torch.Tensor:
    _need(x, torch.float32, "x")
    _need(out, torch.float16, "out")
    hidden = gamma.numel()
    rows = x.shape[0] if rows is None else rows
    _lib.call(
        "kvpr_layernorm", x.data_ptr(), x.stride(0), gamma.data_ptr(), beta.data_ptr(), out.data_ptr(),
        out.stride(0), rows, hidden, float(eps), _stream(stream),
    )
    return out


def layernorm_linear(x: torch.Tensor, gamma: torch.Tensor, beta: torch.Tensor, y: torch.Tensor, w: torch.Tensor,
                     bias: torch.Tensor | None, out: torch.Tensor, rows: int, eps: float = 1e-5, flags: int = 0,
                     bn: int = 0, stream=None, ws: torch.Tensor | None = None) -> torch.Tensor:
    """y[:rows] = LayerNorm(x[:rows]) (fp16) and out[:rows] = epilogue(y . w^T + bias); one launch when the
    projection takes the CUDA-core decode path (rows <= 8 with ws), bit-identical to layernorm + linear."""
    _need(x, torch.float32, "x")
    _need(y, torch.float16, "y")
    _need(w, torch.float16, "w")
    N, K = w.shape
    if out.dtype == torch.float32:
        flags |= _lib.EPI_F32
    epi = _lib.make_epilogue([(out.data_ptr(), 0)], seg_width=((N + 31) // 32) * 32, ld=out.stride(0), row_group=rows,
                             bias=bias.data_ptr() if bias is not None else None, flags=flags)
    _lib.call("kvpr_layernorm_linear_ws", x.data_ptr(), x.stride(0), gamma.data_ptr(), beta.data_ptr(), float(eps),
              y.data_ptr(), y.stride(0), w.data_ptr(), w.stride(0), rows, N, K, epi, bn,
              ws.data_ptr() if ws is not None else None, ws.numel() * ws.element_size() if ws is not None else 0,
              _stream(stream))
    return out


def embed(tokens: torch.Tensor, tok_emb: torch.Tensor, pos_emb: torch.Tensor, out: torch.Tensor, batch: int,
          pos_begin: int, pos_offset: int = 2, stream=None) -> torch.Tensor:
    _need(tokens, torch.int32, "tokens")
    rows = tokens.numel()
    _lib.call(
        "kvpr_embed", tokens.data_ptr(), tok_emb.data_ptr(), pos_emb.data_ptr(), out.data_ptr(), rows, batch,
        pos_begin, tok_emb.shape[1], pos_offset, _stream(stream),
    )
    return out


def argmax(logits: torch.Tensor, out_idx: torch.Tensor, out_val: torch.Tensor | None = None, cols: int | None = None,
           stream=None) -> torch.Tensor:
    _need(logits, torch.float32, "logits")
    cols = logits.shape[1] if cols is None else cols
    _lib.call(
        "kvpr_argmax", logits.data_ptr(), logits.stride(0), logits.shape[0], cols, out_idx.data_ptr(),
        out_val.data_ptr() if out_val is not None else None, _stream(stream),
    )
    return out_idx


def kv4_page_bytes(batch: int, hidden: int) -> int:
    """Bytes of one compressed (4-bit groupwise) KV page: 2*batch*hidden*0.5625."""
    return int(_lib.load().kvpr_kv4_page_bytes(batch, hidden))


def kv4_quantize(pages: torch.Tensor, qpages: torch.Tensor, batch: int, pos_begin: int, pos_end: int,
                 stream=None) -> None:
    _need(pages, torch.float16, "pages")
    _need(qpages, torch.uint8, "qpages")
    hidden = pages.shape[-1]
    _lib.call("kvpr_kv4_quantize", pages.data_ptr(), qpages.data_ptr(), batch, hidden, pos_begin, pos_end,
              _stream(stream))


def kv4_dequantize(qpages: torch.Tensor, pages: torch.Tensor, batch: int, pos_begin: int, pos_end: int,
                   stream=None) -> None:
    _need(pages, torch.float16, "pages")
    _need(qpages, torch.uint8, "qpages")
    hidden = pages.shape[-1]
    _lib.call("kvpr_kv4_dequantize", qpages.data_ptr(), pages.data_ptr(), batch, hidden, pos_begin, pos_end,
              _stream(stream))
