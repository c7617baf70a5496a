"""Per-kernel numerics on the B200 against plain PyTorch fp32 references.

Tolerances (floating point, fp16 storage / fp32 accumulation):
  GEMM / recompute / LN outputs: |out - ref| <= 2e-3 * max|ref| + 2e-3  (fp16 output rounding)
  attention outputs:             |out - ref| <= 2e-3 * max|ref| + 2e-3
The bit-level split/merge property (recomputed pages == prefill pages) is
checked in test_runtime_gpu.py.
"""

from __future__ import annotations

import math

import pytest
import torch

from paper_2411_17089_b200 import _lib, kernels

pytestmark = pytest.mark.gpu


def _close(out, ref, rtol=2e-3, atol=2e-3):
    out = out.float()
    ref = ref.float()
    err = (out - ref).abs().max().item()
    bound = rtol * ref.abs().max().item() + atol
    assert err <= bound, f"max err {err:.3e} > {bound:.3e}"


def _rand(*shape, scale=1.0, dev="cuda", seed=None, dtype=torch.float16):
    g = torch.Generator(device="cpu")
    g.manual_seed(seed if seed is not None else sum(shape))
    return (torch.randn(*shape, generator=g) * scale).to(dtype).to(dev)


@pytest.mark.parametrize(
    "M,N,K,bn",
    [
        (128, 256, 64, 256),
        (300, 512, 4096, 256),
        (32, 768, 768, 64),
        (32, 2304, 768, 128),
        (4096, 4096, 512, 256),  # > 148 tiles: persistent loop + TMEM double buffer
        (1, 64, 128, 64),
        (5, 50272, 768, 0),  # vocab-sized N tail, auto BN
        (777, 1024, 1000, 128),  # K tail (TMA zero fill)
        (28224, 8192, 4096, 512),  # K1 at OPT-6.7B config 2 (l=882): CTA-pair tcgen05 (cta_group::2)
        (300, 512, 4096, 512),  # pair tile with an M tail inside the peer CTA
        (100, 768, 768, 512),  # M < 128: the peer CTA's rows are all out of range
        (4096, 2304, 768, 512),  # N tail within the pair tile (2304 = 9 x 256)
        (32, 4096, 16384, 32),  # decode fc2 shape on narrow 128x32 tiles
        (32, 4096, 4096, 0),  # decode out-proj, auto BN (swap-AB)
        (4, 2304, 768, -1),  # swap-AB decode GEMM, config-1 q/k/v
        (32, 12288, 4096, -1),  # swap-AB, config-2 q/k/v
        (50, 1024, 512, -1),  # swap-AB with 64 padded activation rows
        (1, 50272, 768, -1),  # swap-AB, LM-head N tail, persistent tiles
        (17, 640, 1000, -1),  # swap-AB, K tail and an N tail inside a tile
    ],
)
def test_linear_matches_fp32(dev, M, N, K, bn):
    a = _rand(M, K, scale=0.5, seed=1)
    w = _rand(N, K, scale=0.05, seed=2)
    bias = _rand(N, scale=0.1, seed=3)
    out = torch.empty(M, N, dtype=torch.float16, device=dev)
    kernels.linear_simple(a, w, bias, out, bn=bn)
    ref = a.float() @ w.float().T + bias.float()
    torch.cuda.synchronize()
    _close(out, ref)


def test_pair_tile_bitwise_equals_single_cta(dev):
    """The CTA-pair kernel and the 1-CTA kernel accumulate K in the same order: identical bits."""
    M, N, K = 1000, 1024, 2048
    a = _rand(M, K, scale=0.5, seed=41)
    w = _rand(N, K, scale=0.05, seed=42)
    o1 = torch.empty(M, N, dtype=torch.float16, device=dev)
    o2 = torch.empty(M, N, dtype=torch.float16, device=dev)
    kernels.linear_simple(a, w, None, o1, bn=256)
    kernels.linear_simple(a, w, None, o2, bn=512)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2)


@pytest.mark.parametrize("M", [1, 4, 16, 32, 33, 64])
def test_swapab_bitwise_equals_regular(dev, M):
    """The swapped-operand decode GEMM keeps the regular kernel's k order: identical bits unsplit
    (so the decode-time k, v of a new token equal what K1 rebuilds later)."""
    N, K = 768, 2048
    a = _rand(M, K, scale=0.5, seed=51)
    w = _rand(N, K, scale=0.05, seed=52)
    bias = _rand(N, scale=0.1, seed=53)
    o1 = torch.empty(M, N, dtype=torch.float16, device=dev)
    o2 = torch.empty(M, N, dtype=torch.float16, device=dev)
    kernels.linear_simple(a, w, bias, o1, bn=-1)
    kernels.linear_simple(a, w, bias, o2, bn=128)
    r1 = torch.randn(M, N, device=dev)
    r2 = r1.clone()
    kernels.linear_simple(a, w, bias, r1, bn=-1, flags=_lib.EPI_ACCUM)
    kernels.linear_simple(a, w, bias, r2, bn=128, flags=_lib.EPI_ACCUM)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2)
    assert torch.equal(r1, r2)


def test_swapab_qkv_equals_k1_rebuild(dev):
    """Decode q/k/v via the swap-AB GEMM vs K1 recomputing the same position: k, v bit-identical."""
    b, h = 32, 1024
    x = _rand(1, b, h, scale=1.0, seed=61)
    wqkv = _rand(3 * h, h, scale=0.03, seed=62)
    bqkv = _rand(3 * h, scale=0.1, seed=63)
    q = torch.empty(b, h, dtype=torch.float16, device=dev)
    page_dec = torch.zeros(1, 2, b, h, dtype=torch.float16, device=dev)
    bh = b * h
    kp = page_dec.data_ptr()
    epi = _lib.make_epilogue([(q.data_ptr(), 0), (kp, 2 * bh), (kp + bh * 2, 2 * bh)], seg_width=h, ld=h,
                             row_group=b, bias=bqkv.data_ptr())
    kernels.linear(x.view(b, h), wqkv, epi, M=b, bn=-1)
    page_k1 = torch.zeros(1, 2, b, h, dtype=torch.float16, device=dev)
    kernels.recompute_kv(x, wqkv[h:], bqkv[h:], page_k1, b, 0, 1)
    torch.cuda.synchronize()
    assert torch.equal(page_dec, page_k1)


@pytest.mark.parametrize("M,N,K", [(32, 4096, 16384), (32, 4096, 4096), (4, 768, 3072), (4, 50272, 768)])
def test_swapab_splitk_matches_fp32(dev, M, N, K):
    a = _rand(M, K, scale=0.5, seed=71)
    w = _rand(N, K, scale=0.05, seed=72)
    bias = _rand(N, scale=0.1, seed=73)
    ws = torch.empty(16 << 20, dtype=torch.uint8, device=dev)
    out = torch.randn(M, N, device=dev)
    ref = out.clone() + (a.float() @ w.float().T + bias.float())
    kernels.linear_simple(a, w, bias, out, flags=_lib.EPI_ACCUM, ws=ws)
    torch.cuda.synchronize()
    _close(out, ref, rtol=1e-4, atol=2e-3)


def test_linear_epilogues(dev):
    M, N, K = 96, 512, 256
    a = _rand(M, K, scale=0.5, seed=4)
    w = _rand(N, K, scale=0.05, seed=5)
    bias = _rand(N, scale=0.1, seed=6)
    ref = a.float() @ w.float().T + bias.float()
    # relu, fp16
    out = torch.empty(M, N, dtype=torch.float16, device=dev)
    kernels.linear_simple(a, w, bias, out, flags=_lib.EPI_RELU)
    _close(out, ref.clamp_min(0))
    # fp32 out
    out32 = torch.empty(M, N, dtype=torch.float32, device=dev)
    kernels.linear_simple(a, w, bias, out32)
    _close(out32, ref, rtol=1e-5, atol=1e-4)
    # residual accumulate
    resid = torch.randn(M, N, device=dev)
    acc = resid.clone()
    kernels.linear_simple(a, w, bias, acc, flags=_lib.EPI_ACCUM)
    _close(acc, resid + ref, rtol=1e-5, atol=1e-4)
    # scaled leading columns + 3 segments with row groups (q | k | v scatter)
    seg = 128
    M2 = 4 * 3  # 3 positions x batch 4
    a2 = _rand(M2, K, scale=0.5, seed=7)
    w2 = _rand(3 * seg, K, scale=0.05, seed=8)
    b2 = _rand(3 * seg, scale=0.1, seed=9)
    qbuf = torch.zeros(M2, seg, dtype=torch.float16, device=dev)
    pages = torch.zeros(3, 2, 4, seg, dtype=torch.float16, device=dev)
    epi = _lib.make_epilogue(
        [(qbuf.data_ptr(), 4 * seg), (pages[:, 0].data_ptr(), 2 * 4 * seg), (pages[:, 1].data_ptr(), 2 * 4 * seg)],
        seg_width=seg, ld=seg, row_group=4, bias=b2.data_ptr(), scale=0.125, scale_cols=seg,
    )
    kernels.linear(a2, w2, epi)
    ref2 = a2.float() @ w2.float().T + b2.float()
    torch.cuda.synchronize()
    _close(qbuf, ref2[:, :seg] * 0.125)
    _close(pages[:, 0].reshape(M2, seg), ref2[:, seg:2 * seg])
    _close(pages[:, 1].reshape(M2, seg), ref2[:, 2 * seg:])


@pytest.mark.parametrize(
    "M,N,K",
    [
        (4, 768, 768),  # config-1 out-proj (KS = 4 k-slices per column group)
        (4, 3072, 768),  # config-1 fc1
        (4, 768, 3072),  # config-1 fc2 (units beyond the prefetched ones: main loop)
        (4, 50272, 768),  # config-1 LM head (N tail inside the last CTA)
        (1, 64, 128),  # single row, N < one CTA's columns, most lanes idle
        (8, 1024, 6144),  # long main loop (software-pipelined batches), MP = 8, 96 KB of staged A
        (5, 640, 1000),  # MP = 8 with 3 dead rows; K not a multiple of 256 (partial unit slices)
        (3, 96, 8),  # K = one 16-byte unit
    ],
)
def test_gemv_matches_fp32(dev, M, N, K):
    """CUDA-core decode projection (bn = -2): fp32 accumulation, every epilogue form."""
    a = _rand(M, K, scale=0.5, seed=81)
    w = _rand(N, K, scale=0.05, seed=82)
    bias = _rand(N, scale=0.1, seed=83)
    ref = a.float() @ w.float().T + bias.float()
    out = torch.empty(M, N, dtype=torch.float16, device=dev)
    kernels.linear_simple(a, w, bias, out, bn=-2)
    relu = torch.empty(M, N, dtype=torch.float16, device=dev)
    kernels.linear_simple(a, w, bias, relu, flags=_lib.EPI_RELU, bn=-2)
    resid = torch.randn(M, N, device=dev)
    acc = resid.clone()
    kernels.linear_simple(a, w, bias, acc, flags=_lib.EPI_ACCUM, bn=-2)
    acc2 = resid.clone()
    kernels.linear_simple(a, w, bias, acc2, flags=_lib.EPI_ACCUM, bn=-2)
    torch.cuda.synchronize()
    _close(out, ref)
    _close(relu, ref.clamp_min(0))
    _close(acc, resid + ref, rtol=1e-5, atol=1e-4)
    assert torch.equal(acc, acc2)  # fixed reduction order


def test_gemv_segments_and_auto_routing(dev):
    """Segment scatter / scale through the GEMV epilogue; auto mode picks it only via the ws entry
    at M <= 8 (kvpr_linear keeps the K1-compatible swap-AB kernel)."""
    seg, K, B = 128, 512, 4
    a = _rand(B, K, scale=0.5, seed=84)
    w = _rand(3 * seg, K, scale=0.05, seed=85)
    b = _rand(3 * seg, scale=0.1, seed=86)
    ref = a.float() @ w.float().T + b.float()
    qbuf = torch.zeros(B, seg, dtype=torch.float16, device=dev)
    page = torch.zeros(2, B, seg, dtype=torch.float16, device=dev)
    epi = _lib.make_epilogue([(qbuf.data_ptr(), 0), (page[0].data_ptr(), 0), (page[1].data_ptr(), 0)],
                             seg_width=seg, ld=seg, row_group=B, bias=b.data_ptr(), scale=0.125, scale_cols=seg)
    kernels.linear(a, w, epi, M=B, bn=-2)
    torch.cuda.synchronize()
    _close(qbuf, ref[:, :seg] * 0.125)
    _close(page[0], ref[:, seg:2 * seg])
    _close(page[1], ref[:, 2 * seg:])
    ws = torch.empty(1 << 20, dtype=torch.uint8, device=dev)
    outs = {}
    for name, bn, wsb in (("gemv", -2, None), ("swap", -1, None), ("auto_ws", 0, ws), ("auto", 0, None)):
        o = torch.empty(B, 3 * seg, dtype=torch.float16, device=dev)
        kernels.linear_simple(a, w, b, o, bn=bn, ws=wsb)
        outs[name] = o
    torch.cuda.synchronize()
    assert torch.equal(outs["auto_ws"], outs["gemv"])
    assert torch.equal(outs["auto"], outs["swap"])


@pytest.mark.parametrize("M,N,K", [(4, 3072, 768), (1, 256, 64), (8, 512, 5120), (3, 640, 1000), (32, 1024, 768)])
def test_layernorm_linear_fused_bitwise(dev, M, N, K):
    """kvpr_layernorm_linear_ws: y and out bit-identical to kvpr_layernorm + kvpr_linear_ws.  The
    one-launch form (KVPR_LN_FUSE=1, CUDA-core path at M <= 8) runs in a subprocess, since the switch
    is read once per process; here the default two-launch form."""
    x = torch.randn(M + 2, K + 4, device=dev) * 3 + 0.5  # row stride > K
    g = _rand(K, scale=0.2, seed=91) + 1
    be = _rand(K, scale=0.2, seed=92)
    w = _rand(N, K, scale=0.05, seed=93)
    bias = _rand(N, scale=0.1, seed=94)
    ws = torch.empty(1 << 22, dtype=torch.uint8, device=dev)
    y1 = torch.zeros(M, K, dtype=torch.float16, device=dev)
    o1 = torch.empty(M, N, dtype=torch.float16, device=dev)
    kernels.layernorm(x, g, be, y1, rows=M)
    kernels.linear_simple(y1, w, bias, o1, flags=_lib.EPI_RELU, ws=ws)
    y2 = torch.zeros(M, K, dtype=torch.float16, device=dev)
    o2 = torch.empty(M, N, dtype=torch.float16, device=dev)
    kernels.layernorm_linear(x, g, be, y2, w, bias, o2, rows=M, flags=_lib.EPI_RELU, ws=ws)
    torch.cuda.synchronize()
    assert torch.equal(y1, y2)
    assert torch.equal(o1, o2)
    xr = x[:M, :K]
    ref_y = (xr - xr.mean(-1, keepdim=True)) / torch.sqrt(xr.var(-1, unbiased=False, keepdim=True) + 1e-5)
    _close(y2, ref_y * g.float() + be.float())


_FUSED_LN_SCRIPT = r"""
import sys, torch
sys.path.insert(0, sys.argv[1])
from paper_2411_17089_b200 import _lib, kernels
torch.manual_seed(0)
for M, N, K in ((4, 3072, 768), (8, 512, 2048), (3, 640, 1000)):
    x = torch.randn(M + 2, K + 4, device="cuda") * 3 + 0.5
    g = torch.randn(K, device="cuda").half() * 0.2 + 1
    be = torch.randn(K, device="cuda").half() * 0.2
    w = (torch.randn(N, K, device="cuda") * 0.05).half()
    bias = (torch.randn(N, device="cuda") * 0.1).half()
    ws = torch.empty(1 << 22, dtype=torch.uint8, device="cuda")
    y1 = torch.zeros(M, K, dtype=torch.float16, device="cuda"); o1 = torch.empty(M, N, dtype=torch.float16, device="cuda")
    kernels.layernorm(x, g, be, y1, rows=M)
    kernels.linear_simple(y1, w, bias, o1, flags=_lib.EPI_RELU, ws=ws)
    y2 = torch.zeros_like(y1); o2 = torch.empty_like(o1)
    n0 = _lib.load().kvpr_kernel_launches()
    kernels.layernorm_linear(x, g, be, y2, w, bias, o2, rows=M, flags=_lib.EPI_RELU, ws=ws)
    n = _lib.load().kvpr_kernel_launches() - n0
    torch.cuda.synchronize()
    assert n == 1, n
    assert torch.equal(y1, y2) and torch.equal(o1, o2), (M, N, K)
print("fused ok")
"""


def test_layernorm_linear_one_launch_form_bitwise(dev):
    """KVPR_LN_FUSE=1: LN computed inside every CTA of the CUDA-core projection (one launch), y and
    out bit-identical to the LN kernel + projection."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = str(Path(__file__).resolve().parents[1])
    r = subprocess.run([sys.executable, "-c", _FUSED_LN_SCRIPT, root], env={**os.environ, "KVPR_LN_FUSE": "1"},
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "fused ok" in r.stdout, r.stdout + r.stderr


def test_gemv_rejects_large_m_and_k(dev):
    a = _rand(9, 64, seed=87)
    w = _rand(64, 64, seed=88)
    out = torch.empty(9, 64, dtype=torch.float16, device=dev)
    with pytest.raises(ValueError, match="gemv"):
        kernels.linear_simple(a, w, None, out, bn=-2)
    a = _rand(8, 8192, seed=89)  # 128 KB of activations to stage
    w = _rand(64, 8192, seed=90)
    out = torch.empty(8, 64, dtype=torch.float16, device=dev)
    with pytest.raises(ValueError, match="gemv"):
        kernels.linear_simple(a, w, None, out, bn=-2)
    ws = torch.empty(1 << 20, dtype=torch.uint8, device=dev)
    kernels.linear_simple(a, w, None, out, ws=ws)  # auto mode falls back to the swap-AB kernel
    torch.cuda.synchronize()
    _close(out, a.float() @ w.float().T)


@pytest.mark.parametrize("batch,hidden,p0,p1", [(4, 768, 0, 257), (4, 768, 3, 250), (3, 256, 5, 6), (32, 512, 0, 40)])
def test_recompute_kv_writes_pages(dev, batch, hidden, p0, p1):
    S = p1 + 3
    x = _rand(S, batch, hidden, scale=1.0, seed=10)
    w_kv = _rand(2 * hidden, hidden, scale=0.03, seed=11)
    b_kv = _rand(2 * hidden, scale=0.1, seed=12)
    pages = torch.full((S, 2, batch, hidden), 7.0, dtype=torch.float16, device=dev)
    kernels.recompute_kv(x, w_kv, b_kv, pages, batch, p0, p1)
    torch.cuda.synchronize()
    ref = x[p0:p1].float() @ w_kv.float().T + b_kv.float()  # [P, batch, 2h]
    _close(pages[p0:p1, 0], ref[..., :hidden])
    _close(pages[p0:p1, 1], ref[..., hidden:])
    # positions outside [p0, p1) untouched
    assert torch.all(pages[:p0] == 7.0) and torch.all(pages[p1:] == 7.0)


def test_recompute_split_zero_is_noop(dev):
    pages = torch.full((4, 2, 2, 64), 3.0, dtype=torch.float16, device=dev)
    x = torch.zeros(4, 2, 64, dtype=torch.float16, device=dev)
    w = torch.zeros(128, 64, dtype=torch.float16, device=dev)
    kernels.recompute_kv(x, w, None, pages, 2, 2, 2)
    assert torch.all(pages == 3.0)


def test_recompute_rejects_bad_split(dev):
    pages = torch.zeros(4, 2, 2, 64, dtype=torch.float16, device=dev)
    x = torch.zeros(4, 2, 64, dtype=torch.float16, device=dev)
    w = torch.zeros(128, 64, dtype=torch.float16, device=dev)
    with pytest.raises(ValueError, match="split"):
        kernels.recompute_kv(x, w, None, pages, 2, 3, 1)


def _attn_ref(q, pages, batch, heads, d, seq):
    # q [batch, h]; pages [S, 2, batch, h]
    K = pages[:seq, 0].float().reshape(seq, batch, heads, d)
    V = pages[:seq, 1].float().reshape(seq, batch, heads, d)
    qh = q.float().reshape(batch, heads, d)
    logits = torch.einsum("sbhd,bhd->bhs", K, qh) / math.sqrt(d)
    w = torch.softmax(logits, dim=-1)
    return torch.einsum("bhs,sbhd->bhd", w, V).reshape(batch, heads * d)


@pytest.mark.parametrize(
    "batch,heads,d,seq",
    [(4, 12, 64, 257), (2, 32, 128, 1025), (32, 32, 128, 1025), (1, 2, 64, 1), (3, 4, 128, 70), (1, 1, 128, 8193)],
)
def test_decode_attention_matches_fp32(dev, batch, heads, d, seq):
    h = heads * d
    pages = _rand(seq + 5, 2, batch, h, scale=1.0, seed=seq)
    q = _rand(batch, h, scale=1.0, seed=seq + 1)
    out = torch.empty(batch, h, dtype=torch.float16, device=dev)
    ws = torch.empty(64 << 20, dtype=torch.uint8, device=dev)
    kernels.decode_attention(q, pages, out, ws, batch, heads, d, seq)
    torch.cuda.synchronize()
    _close(out, _attn_ref(q, pages, batch, heads, d, seq))
    # without workspace (single split) gives the same answer
    out1 = torch.empty_like(out)
    kernels.decode_attention(q, pages, out1, None, batch, heads, d, seq)
    torch.cuda.synchronize()
    _close(out1, _attn_ref(q, pages, batch, heads, d, seq))


def test_decode_attention_empty_cache_rejected(dev):
    q = torch.zeros(1, 64, dtype=torch.float16, device=dev)
    pages = torch.zeros(1, 2, 1, 64, dtype=torch.float16, device=dev)
    with pytest.raises(ValueError, match="empty"):
        kernels.decode_attention(q, pages, torch.empty_like(q), None, 1, 1, 64, 0)


@pytest.mark.parametrize("batch,heads,d,seq", [(2, 4, 64, 37), (3, 2, 128, 130), (1, 3, 64, 1), (2, 2, 128, 64),
                                               (2, 4, 128, 1000), (1, 2, 64, 513),
                                               (3, 40, 64, 1000), (2, 37, 128, 777)])
def test_prefill_attention_causal(dev, batch, heads, d, seq):
    """Last two cases: more work items (query-tile pairs x sequences x heads: 480, 296) than SMs, so
    the persistent CTAs walk several zigzag rounds, the last one partial."""
    h = heads * d
    pages = _rand(seq, 2, batch, h, seed=20)
    q = _rand(seq, batch, h, seed=21)
    out = torch.empty(seq, batch, h, dtype=torch.float16, device=dev)
    kernels.prefill_attention(q, pages, out, batch, heads, d, seq)
    torch.cuda.synchronize()
    K = pages[:, 0].float().reshape(seq, batch, heads, d)
    V = pages[:, 1].float().reshape(seq, batch, heads, d)
    qh = q.float().reshape(seq, batch, heads, d)
    logits = torch.einsum("tbhd,sbhd->bhts", qh, K) / math.sqrt(d)
    mask = torch.triu(torch.ones(seq, seq, dtype=torch.bool, device=dev), 1)
    logits = logits.masked_fill(mask, float("-inf"))
    ref = torch.einsum("bhts,sbhd->tbhd", torch.softmax(logits, -1), V).reshape(seq, batch, h)
    _close(out, ref)


def _prefill_ref(q, pages, batch, heads, d, seq):
    K = pages[:, 0].float().reshape(seq, batch, heads, d)
    V = pages[:, 1].float().reshape(seq, batch, heads, d)
    qh = q.float().reshape(seq, batch, heads, d)
    logits = torch.einsum("tbhd,sbhd->bhts", qh, K) / math.sqrt(d)
    mask = torch.triu(torch.ones(seq, seq, dtype=torch.bool, device=q.device), 1)
    logits = logits.masked_fill(mask, float("-inf"))
    return torch.einsum("bhts,sbhd->tbhd", torch.softmax(logits, -1), V).reshape(seq, batch, heads * d)


@pytest.mark.parametrize("d", [64, 128])
def test_prefill_attention_running_max_moves(dev, d):
    """Scores that grow along the keys (0.6 per position, ~10 log2 units per 128-key tile): every
    tile moves each row's running max past the lazy-rescale threshold (2^8), so the O correction in
    TMEM runs on every tile of every row -- the path random inputs almost never take."""
    batch, heads, seq = 2, 2, 700
    h = heads * d
    pos = torch.arange(seq, device=dev, dtype=torch.float32)
    k = (pos * 0.6 / d)[:, None, None].expand(seq, batch, h)
    v = _rand(seq, batch, h, seed=22).float()
    pages = torch.stack([k, v], 1).half().contiguous()
    q = torch.ones(seq, batch, h, dtype=torch.float16, device=dev)
    out = torch.empty(seq, batch, h, dtype=torch.float16, device=dev)
    kernels.prefill_attention(q, pages, out, batch, heads, d, seq)
    torch.cuda.synchronize()
    _close(out, _prefill_ref(q, pages, batch, heads, d, seq))


@pytest.mark.parametrize("rows,hidden", [(32, 4096), (7, 768), (3, 7168), (1, 5120)])
def test_layernorm(dev, rows, hidden):
    x = torch.randn(rows, hidden, device=dev) * 3 + 1
    g = _rand(hidden, scale=0.1, seed=30) + 1
    b = _rand(hidden, scale=0.1, seed=31)
    out = torch.empty(rows, hidden, dtype=torch.float16, device=dev)
    kernels.layernorm(x, g, b, out)
    ref = torch.nn.functional.layer_norm(x, (hidden,), g.float(), b.float(), 1e-5)
    torch.cuda.synchronize()
    _close(out, ref)


def test_embed_and_argmax(dev):
    V, P, h, batch = 1000, 40, 256, 3
    E = _rand(V, h, seed=40)
    Pe = _rand(P, h, seed=41)
    toks = torch.tensor([5, 999, 0, 17, 3, 3], dtype=torch.int32, device=dev)  # 2 positions x 3
    out = torch.empty(6, h, device=dev)
    kernels.embed(toks, E, Pe, out, batch=batch, pos_begin=7, pos_offset=2)
    pos = torch.tensor([7, 7, 7, 8, 8, 8], device=dev) + 2
    ref = E[toks.long()].float() + Pe[pos].float()
    torch.cuda.synchronize()
    assert torch.equal(out, ref)
    logits = torch.randn(5, 50272, device=dev)
    logits[2, 123] = 1e4
    logits[3, 7] = logits[3, 9] = 1e4  # tie -> smallest index
    idx = torch.empty(5, dtype=torch.int32, device=dev)
    val = torch.empty(5, device=dev)
    kernels.argmax(logits, idx, val)
    torch.cuda.synchronize()
    ref_idx = logits.argmax(dim=1)
    assert idx.tolist() == ref_idx.tolist()
    assert idx[3].item() == 7


@pytest.mark.parametrize("P,batch,hidden", [(3, 4, 768), (17, 32, 4096), (1, 1, 64)])
def test_kv4_codec_bitwise_vs_oracle(dev, P, batch, hidden):
    """4-bit groupwise KV pages: GPU codec == oracle/kvquant_ref.py byte for byte, both directions."""
    import numpy as np

    from oracle import kvquant_ref

    g = torch.Generator().manual_seed(P * 31 + hidden)
    x = (torch.randn(P + 2, 2, batch, hidden, generator=g) * 2).half()
    x[0, 0, 0, :64] = 1.5  # a constant group (scale 0)
    pages = x.to(dev)
    qb = kernels.kv4_page_bytes(batch, hidden)
    assert qb == kvquant_ref.page_bytes(batch, hidden) == int(2 * batch * hidden * 0.5625)
    q = torch.zeros(P + 2, qb, dtype=torch.uint8, device=dev)
    kernels.kv4_quantize(pages, q, batch, 1, P + 1)
    back = torch.zeros_like(pages)
    kernels.kv4_dequantize(q, back, batch, 1, P + 1)
    torch.cuda.synchronize()
    want_q = kvquant_ref.quantize(x[1:P + 1].numpy())
    assert np.array_equal(q[1:P + 1].cpu().numpy(), want_q)
    assert torch.all(q[0] == 0) and torch.all(q[P + 1] == 0)  # outside [pos_begin, pos_end) untouched
    want_x = kvquant_ref.dequantize(want_q, batch, hidden)
    assert np.array_equal(back[1:P + 1].cpu().numpy(), want_x)
    err = (back[1:P + 1].float() - pages[1:P + 1].float()).abs().max().item()
    assert err <= (x.float().max() - x.float().min()).item() / 15 / 2 + 1e-2


@pytest.mark.parametrize("batch,heads,d,seq,lo,hi", [
    (4, 12, 64, 257, 200, 256), (32, 32, 128, 1025, 0, 1024), (3, 8, 128, 300, 17, 299), (2, 4, 64, 70, 5, 5),
    (1, 2, 128, 9, 0, 9)])
def test_decode_attention_kv4_fused_bitwise(dev, batch, heads, d, seq, lo, hi):
    """K2 reading [lo, hi) from 4-bit pages == kv4_dequantize into the fp16 pages, then K2 — bit for bit
    (the fused read uses the dequantize kernel's arithmetic)."""
    h = heads * d
    g = torch.Generator().manual_seed(seq + lo)
    pages = (torch.randn(seq + 1, 2, batch, h, generator=g)).half().to(dev)
    q = torch.randn(batch, h, generator=g).half().to(dev)
    qp = torch.zeros(seq + 1, kernels.kv4_page_bytes(batch, h), dtype=torch.uint8, device=dev)
    kernels.kv4_quantize(pages, qp, batch, 0, seq)
    ws = torch.empty(8 << 20, dtype=torch.uint8, device=dev)
    mixed = pages.clone()
    mixed[lo:hi] = float("nan")  # the fused path must not read the fp16 tail
    fused = torch.empty(batch, h, dtype=torch.float16, device=dev)
    kernels.decode_attention_kv4(q, mixed, qp, lo, hi, fused, ws, batch, heads, d, seq)
    ref_pages = pages.clone()
    kernels.kv4_dequantize(qp, ref_pages, batch, lo, hi)
    ref = torch.empty_like(fused)
    kernels.decode_attention(q, ref_pages, ref, ws, batch, heads, d, seq)
    torch.cuda.synchronize()
    assert torch.equal(fused, ref)
    with pytest.raises(ValueError):
        kernels.decode_attention_kv4(q, mixed, qp, 0, seq + 1, fused, ws, batch, heads, d, seq)


@pytest.mark.parametrize("M,N,K", [(32, 4096, 16384), (32, 4096, 4096), (7, 768, 3072), (128, 1024, 8192)])
def test_split_k_decode_gemm(dev, M, N, K):
    """Single-row-block GEMMs with a workspace split K across CTAs; partials reduced in slice order:
    fp32-reference accurate, run-to-run deterministic, all epilogues (bias, ReLU, fp32 residual add)."""
    a = _rand(M, K, scale=0.5, seed=51)
    w = _rand(N, K, scale=0.02, seed=52)
    bias = _rand(N, scale=0.1, seed=53)
    ws = torch.empty(16 << 20, dtype=torch.uint8, device=dev)
    ref = a.float() @ w.float().T + bias.float()
    out = torch.empty(M, N, dtype=torch.float16, device=dev)
    kernels.linear_simple(a, w, bias, out, flags=_lib.EPI_RELU, ws=ws)
    out2 = torch.empty_like(out)
    kernels.linear_simple(a, w, bias, out2, flags=_lib.EPI_RELU, ws=ws)
    resid = torch.randn(M, N, device=dev)
    acc = resid.clone()
    kernels.linear_simple(a, w, bias, acc, flags=_lib.EPI_ACCUM, ws=ws)
    torch.cuda.synchronize()
    _close(out, ref.clamp_min(0))
    assert torch.equal(out, out2)
    _close(acc, resid + ref, rtol=1e-5, atol=1e-4)


@pytest.mark.parametrize("batch,heads,d,seq", [(32, 32, 128, 1025), (4, 12, 64, 257), (2, 4, 128, 300)])
def test_decode_attention_cluster_merge_equals_combine_kernel(dev, batch, heads, d, seq, monkeypatch):
    """Split-KV merge in the cluster leader's shared memory (one launch) == the combine kernel, bit for bit."""
    h = heads * d
    q = _rand(batch, h, scale=1.0, seed=81)
    pages = _rand(seq + 3, 2, batch, h, scale=1.0, seed=82)
    ws = torch.empty(16 << 20, dtype=torch.uint8, device=dev)
    outs = []
    for flag in ("1", "0"):
        monkeypatch.setenv("KVPR_K2_CLUSTER", flag)
        o = torch.empty(batch, h, dtype=torch.float16, device=dev)
        kernels.decode_attention(q, pages, o, ws, batch, heads, d, seq)
        torch.cuda.synchronize()
        outs.append(o)
    assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("M,N,K", [(32, 4096, 4096), (32, 16384, 4096), (32, 4096, 16384), (64, 4096, 4096),
                                   (17, 50272, 768), (1, 1024, 4096), (12, 384, 256)])
def test_stream_k_decode_gemm(dev, M, N, K):
    """Swap-AB decode GEMM with a workspace runs stream-K (every SM an equal share of the n-tile x
    k-block units; shared tiles finished in-kernel by the last CTA, partials summed in k order):
    fp32-reference accurate, equal to the unsplit kernel within fp32 reassociation, bit-identical across
    calls even when the workspace (its counter tail included) is overwritten with garbage in between."""
    a = _rand(M, K, scale=0.5, seed=61)
    w = _rand(N, K, scale=0.02, seed=62)
    bias = _rand(N, scale=0.1, seed=63)
    ws = torch.empty(16 << 20, dtype=torch.uint8, device=dev)
    ref = a.float() @ w.float().T + bias.float()
    outs = []
    for trial in range(3):
        ws.random_(0, 256)  # arbitrary scratch contents, counters included
        o = torch.empty(M, N, dtype=torch.float32, device=dev)
        kernels.linear_simple(a, w, bias, o, bn=-1, ws=ws)
        outs.append(o)
    plain = torch.empty(M, N, dtype=torch.float32, device=dev)
    kernels.linear_simple(a, w, bias, plain, bn=-1)  # no workspace: whole tiles, one CTA each
    resid = torch.randn(M, N, device=dev)
    acc = resid.clone()
    kernels.linear_simple(a, w, bias, acc, flags=_lib.EPI_ACCUM, bn=-1, ws=ws)
    torch.cuda.synchronize()
    _close(outs[0], ref, rtol=1e-3, atol=1e-3)
    assert all(torch.equal(outs[0], x) for x in outs[1:])
    _close(outs[0], plain, rtol=1e-4, atol=1e-4)
    _close(acc, resid + outs[0], rtol=1e-6, atol=1e-5)


@pytest.mark.parametrize("M,N,K", [(32, 4096, 4096), (17, 50272, 768), (32, 12288, 4096), (5, 384, 200)])
def test_tiled_weights_bit_identical(dev, M, N, K):
    """Box-tiled weights (kvpr_tile_weight, each 128 x 64 box contiguous; zero-padded to whole boxes) feed
    the same smem bytes to the same MMA sequence: bit-identical to the row-major operand, unsplit and
    stream-K alike (the q/k/v projection relies on it to keep K1's bits)."""
    a = _rand(M, K, scale=0.5, seed=71)
    w = _rand(N, K, scale=0.02, seed=72)
    bias = _rand(N, scale=0.1, seed=73)
    wt = kernels.tile_weight(w)
    ws = torch.empty(16 << 20, dtype=torch.uint8, device=dev)
    for use_ws in (None, ws):
        o1 = torch.empty(M, N, dtype=torch.float32, device=dev)
        o2 = torch.empty_like(o1)
        kernels.linear_simple(a, w, bias, o1, bn=-1, ws=use_ws)
        kernels.linear_simple(a, wt, bias, o2, ws=use_ws)
        torch.cuda.synchronize()
        assert torch.equal(o1, o2)
    with pytest.raises(ValueError, match="tiled"):
        kernels.linear_simple(_rand(80, K, seed=74), wt, bias, torch.empty(80, N, device=dev))


def test_copy_entry_points(dev):
    """kvpr_copy_async / kvpr_copy_batch_async / kvpr_copy_2d_async (the schedule's DMAs): bytes land
    where the pitches say, zero-byte entries are skipped, a pitch below the width is rejected."""
    import ctypes

    from paper_2411_17089_b200 import _lib, hostmem

    lib = _lib.load()
    s = torch.cuda.current_stream()
    host = hostmem.pinned_empty((4, 1000), torch.uint8)
    host.copy_(torch.randint(0, 255, (4, 1000), dtype=torch.uint8))
    dst = torch.zeros(4, 600, dtype=torch.uint8, device=dev)
    # 2-D: 4 rows of 300 bytes from host pitch 1000 (offset 100) into device pitch 600 (offset 50)
    _lib.call("kvpr_copy_2d_async", dst.data_ptr() + 50, 600, host.data_ptr() + 100, 1000, 300, 4, s.cuda_stream)
    torch.cuda.synchronize()
    assert torch.equal(dst[:, 50:350].cpu(), host[:, 100:400])
    assert int(dst[:, :50].sum()) == 0 and int(dst[:, 350:].sum()) == 0
    with pytest.raises(ValueError):
        _lib.call("kvpr_copy_2d_async", dst.data_ptr(), 100, host.data_ptr(), 1000, 300, 2, s.cuda_stream)
    # batch: two copies and a zero-byte entry, one call
    out = torch.zeros(3, 256, dtype=torch.uint8, device=dev)
    dsts = (ctypes.c_void_p * 3)(out[0].data_ptr(), out[1].data_ptr(), out[2].data_ptr())
    srcs = (ctypes.c_void_p * 3)(host[0].data_ptr(), host[1].data_ptr(), host[2].data_ptr())
    sizes = (ctypes.c_size_t * 3)(256, 0, 128)
    _lib.call("kvpr_copy_batch_async", dsts, srcs, sizes, 3, s.cuda_stream)
    _lib.call("kvpr_copy_async", out[1].data_ptr() + 10, host[3].data_ptr(), 20, s.cuda_stream)
    torch.cuda.synchronize()
    o = out.cpu()
    assert torch.equal(o[0], host[0, :256]) and torch.equal(o[2, :128], host[2, :128]) and int(o[2, 128:].sum()) == 0
    assert torch.equal(o[1, 10:30], host[3, :20]) and int(o[1, :10].sum()) == 0
