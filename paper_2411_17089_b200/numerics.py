"""GPU drop-in for ``kvoverlap.numerics``' split/merge attention
(/root/reference/pkg/src/kvoverlap/numerics.py), same names and arguments.

``split_merge_kv`` rebuilds positions [0, split) with the K1 tcgen05 GEMM and
``decode_attention`` runs K2 + the W_O projection, so the reference's own
test style (pkg/tests/test_numerics.py) can be pointed at the B200 path.
Differences, by design of the target: arithmetic is fp16 storage / fp32
accumulation (the reference is fp64), so agreement is within the north-star
tolerance (2e-2 relative), not 1e-12; arrays come back as float64 NumPy to
keep the reference's types.  Validation (ValueError conditions and messages)
follows numerics.py:22-32, 121-126, 172-182.  The reference matrices are
[in, out] (``x @ w_k``); the kernels take the torch [out, in] layout, so
weights are transposed on upload.  Any head_dim up to 128 works (K2 reads
64- or 128-wide heads; narrower ones are zero-padded per head, which leaves
K q and the kept output lanes unchanged), so the reference's randomized
validate harness (cli.py:343-377, head_dim 1..4) runs through this module.
``decode_attention_batch`` attends several per-sequence caches of different
lengths in one ragged K2 launch (kvpr_decode_attention_ragged).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, kernels


def _mat(label, arr, rows=None, cols=None) -> np.ndarray:
    """numerics.py:22-32: a finite 2-D float64 matrix, optionally (rows, cols)."""
    out = np.asarray(arr, dtype=np.float64)
    if out.ndim != 2:
        raise ValueError(f"{label} must be 2-D, got shape {out.shape}")
    for axis, (want, what) in enumerate(((rows, "rows"), (cols, "cols"))):
        if want is not None and out.shape[axis] != want:
            raise ValueError(f"{label} must have {want} {what}, got {out.shape[axis]}")
    if not np.all(np.isfinite(out)):
        raise ValueError(f"{label} contains non-finite entries")
    return out


@dataclass(frozen=True)
class KVState:
    """Per-sequence cache (numerics.py:43-72): keys / values as (num_heads, seq_len, d_head) float64."""

    keys: np.ndarray
    values: np.ndarray

    def __post_init__(self):
        pair = tuple(np.asarray(t, dtype=np.float64) for t in (self.keys, self.values))
        if any(t.ndim != 3 for t in pair):
            raise ValueError("keys/values must be (num_heads, seq_len, d_head)")
        if pair[0].shape != pair[1].shape:
            raise ValueError(f"key shape {pair[0].shape} != value shape {pair[1].shape}")
        if not all(np.all(np.isfinite(t)) for t in pair):
            raise ValueError("KV entries must be finite")
        object.__setattr__(self, "keys", pair[0])
        object.__setattr__(self, "values", pair[1])

    num_heads = property(lambda self: self.keys.shape[0])
    seq_len = property(lambda self: self.keys.shape[1])
    head_dim = property(lambda self: self.keys.shape[2])


def _dev():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2411_17089_b200.numerics runs on the GPU only (no CPU fallback)")
    _lib.load()
    return torch.device("cuda")


def _pad_to(n: int, m: int) -> int:
    return (n + m - 1) // m * m


def _heads(rows: np.ndarray, heads: int) -> np.ndarray:
    """(n, h) -> (heads, n, d) (numerics.py:35-40)."""
    n, h = rows.shape
    if h % heads:
        raise ValueError("hidden size not divisible by head count")
    return np.ascontiguousarray(rows.reshape(n, heads, h // heads).transpose(1, 0, 2))


def _k1_rows(x: np.ndarray, w_k: np.ndarray, w_v: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """K = x W_k, V = x W_v for the rows of x, by K1 (the tcgen05 recompute GEMM) into a page buffer."""
    n, h = x.shape
    dev = _dev()
    hp = _pad_to(h, 64)  # GEMM needs K % 8 and N % 32; pad the hidden dim with zeros
    xd = torch.zeros(n, 1, hp, dtype=torch.float16, device=dev)
    xd[:, 0, :h] = torch.from_numpy(x).to(dev, torch.float16)
    w = torch.zeros(2 * hp, hp, dtype=torch.float16, device=dev)
    w[:h, :h] = torch.from_numpy(w_k.T.copy()).to(dev, torch.float16)
    w[hp:hp + h, :h] = torch.from_numpy(w_v.T.copy()).to(dev, torch.float16)
    pages = torch.empty(n, 2, 1, hp, dtype=torch.float16, device=dev)
    kernels.recompute_kv(xd, w, None, pages, 1, 0, n)
    kv = pages[:, :, 0, :h].double().cpu().numpy()  # [n, 2, h]
    return kv[:, 0], kv[:, 1]


def project_qkv(x, w_q, w_k, w_v, num_heads: int):
    """Q/K/V of the rows of x, per head (numerics.py:75-92): one tcgen05 GEMM against [W_q|W_k|W_v]."""
    x = _mat("x", x)
    n, h = x.shape
    mats = [_mat(name, m, h, h) for name, m in (("w_q", w_q), ("w_k", w_k), ("w_v", w_v))]
    dev = _dev()
    hp = _pad_to(h, 64)
    xd = torch.zeros(n, hp, dtype=torch.float16, device=dev)
    xd[:, :h] = torch.from_numpy(x).to(dev, torch.float16)
    w = torch.zeros(3 * hp, hp, dtype=torch.float16, device=dev)
    for i, m in enumerate(mats):
        w[i * hp:i * hp + h, :h] = torch.from_numpy(m.T.copy()).to(dev, torch.float16)
    out = torch.empty(n, 3 * hp, dtype=torch.float32, device=dev)
    kernels.linear_simple(xd, w, None, out)
    o = out.double().cpu().numpy()
    return tuple(_heads(o[:, i * hp:i * hp + h], num_heads) for i in range(3))


def build_kv(x, w_k, w_v, num_heads: int) -> KVState:
    """Full cache from all layer inputs (numerics.py:95-104), by K1."""
    x = _mat("x", x)
    h = x.shape[1]
    k, v = _k1_rows(x, _mat("w_k", w_k, h, h), _mat("w_v", w_v, h, h))
    return KVState(_heads(k, num_heads), _heads(v, num_heads))


def split_merge_kv(x_full, split: int, w_k, w_v, kv_suffix: KVState) -> KVState:
    """K1 rebuild of [0, split) concatenated with the transferred suffix (numerics.py:107-137)."""
    x_full = _mat("x_full", x_full)
    seq, h = x_full.shape
    if not 0 <= split <= seq:
        raise ValueError(f"split must be in [0, {seq}], got {split}")
    if kv_suffix.seq_len != seq - split:
        raise ValueError(f"suffix covers {kv_suffix.seq_len} positions, expected {seq - split}")
    if split == 0:
        return kv_suffix
    k, v = _k1_rows(x_full[:split], _mat("w_k", w_k, h, h), _mat("w_v", w_v, h, h))
    heads = kv_suffix.num_heads
    return KVState(np.concatenate([_heads(k, heads), kv_suffix.keys], axis=1),
                   np.concatenate([_heads(v, heads), kv_suffix.values], axis=1))


def append_token_kv(kv: KVState, x_new, w_k, w_v) -> KVState:
    """The cache with the new token's k, v appended (numerics.py:140-156); K1 on one row, so the
    appended entry carries the bits a later split_merge_kv rebuild of that position produces."""
    row = np.asarray(x_new, dtype=np.float64)
    if row.ndim == 1:
        row = row[None, :]
    row = _mat("x_new", row, rows=1)
    h = row.shape[1]
    if kv.num_heads * kv.head_dim != h:
        raise ValueError("token width does not match cache geometry")
    k, v = _k1_rows(row, _mat("w_k", w_k, h, h), _mat("w_v", w_v, h, h))
    return KVState(np.concatenate([kv.keys, _heads(k, kv.num_heads)], axis=1),
                   np.concatenate([kv.values, _heads(v, kv.num_heads)], axis=1))


def stable_softmax(logits) -> np.ndarray:
    """Max-subtracted softmax of a 1-D vector (numerics.py:159-163).  A host-side utility of the
    reference API (K2 fuses its own exp2-domain online softmax); computed on the device in fp64."""
    z = torch.from_numpy(np.asarray(logits, dtype=np.float64)).to(_dev())
    e = torch.exp(z - z.max())
    return (e / e.sum()).cpu().numpy()


def _check_query(q, h) -> np.ndarray:
    q = np.asarray(q, dtype=np.float64)
    if q.ndim != 1:
        raise ValueError("q_token must be a 1-D row of length h")
    if q.size != h:
        raise ValueError(f"q_token has length {q.size}, expected {h}")
    if not np.all(np.isfinite(q)):
        raise ValueError("q_token contains non-finite entries")
    return q


def _attend(qs: list[np.ndarray], kvs: list[KVState], w_o: np.ndarray) -> np.ndarray:
    """K2 over one or more per-sequence caches (ragged lengths), then W_O, on the device.

    K2 reads whole 16-byte rows of a 64- or 128-wide head; any other head_dim <= 128 is zero-padded
    per head (zero query and key lanes add nothing to K q, zero value lanes produce output lanes that
    are dropped), with the softmax scale of the real head_dim, 1/sqrt(d) (numerics.py:184)."""
    heads, d = kvs[0].num_heads, kvs[0].head_dim
    if d > 128:
        raise ValueError(f"head_dim {d} unsupported by the decode-attention kernel (at most 128)")
    n, h, dp = len(kvs), heads * d, (64 if d <= 64 else 128)
    dev = _dev()
    smax = max(kv.seq_len for kv in kvs)
    pages = torch.zeros(smax, 2, n, heads, dp, dtype=torch.float16, device=dev)
    qd = torch.zeros(n, heads, dp, dtype=torch.float16, device=dev)
    for i, (q, kv) in enumerate(zip(qs, kvs)):
        s = kv.seq_len
        pages[:s, 0, i, :, :d] = torch.from_numpy(kv.keys.transpose(1, 0, 2)).to(dev, torch.float16)
        pages[:s, 1, i, :, :d] = torch.from_numpy(kv.values.transpose(1, 0, 2)).to(dev, torch.float16)
        qd[i, :, :d] = torch.from_numpy(q.reshape(heads, d)).to(dev, torch.float16)
    att = torch.empty(n, heads * dp, dtype=torch.float16, device=dev)
    ws = torch.zeros(1 << 20, dtype=torch.uint8, device=dev)
    scale = 1.0 / math.sqrt(d)
    if n == 1:
        kernels.decode_attention(qd.view(1, -1), pages.view(smax, 2, 1, -1), att, ws, 1, heads, dp, smax, scale=scale)
    else:
        lens = torch.tensor([kv.seq_len for kv in kvs], dtype=torch.int32, device=dev)
        kernels.decode_attention_ragged(qd.view(n, -1), pages.view(smax, 2, n, -1), lens, att, ws, heads, dp,
                                        scale=scale)
    hp = _pad_to(h, 64)  # W_O GEMM: K % 8, N % 32 -> zero-padded hidden
    a = torch.zeros(n, hp, dtype=torch.float16, device=dev)
    a[:, :h] = att.view(n, heads, dp)[:, :, :d].reshape(n, h)
    wo = torch.zeros(hp, hp, dtype=torch.float16, device=dev)
    wo[:h, :h] = torch.from_numpy(w_o.T.copy()).to(dev, torch.float16)  # [out, in]
    out = torch.empty(n, hp, dtype=torch.float32, device=dev)
    kernels.linear_simple(a, wo, None, out)
    return out[:, :h].double().cpu().numpy()


def decode_attention(q_token, kv: KVState, w_o) -> np.ndarray:
    """K2 split-KV attention over the cache, then W_O (numerics.py:166-191)."""
    if not kv.seq_len:
        raise ValueError("cannot attend over an empty cache")
    h = kv.num_heads * kv.head_dim
    q = _check_query(q_token, h)
    return _attend([q], [kv], _mat("w_o", w_o, h, h))[0]


def decode_attention_batch(q_tokens, kvs: list[KVState], w_o) -> np.ndarray:
    """decode_attention for several sequences with their own caches (ragged lengths, the reference's
    per-sequence KVState) in ONE K2 launch: row i = decode_attention(q_tokens[i], kvs[i], w_o)."""
    if not kvs:
        raise ValueError("need at least one sequence")
    heads, d = kvs[0].num_heads, kvs[0].head_dim
    if any((kv.num_heads, kv.head_dim) != (heads, d) for kv in kvs):
        raise ValueError("all caches must share num_heads and head_dim")
    if any(not kv.seq_len for kv in kvs):
        raise ValueError("cannot attend over an empty cache")
    qs = np.asarray(q_tokens, dtype=np.float64)
    if qs.ndim != 2 or qs.shape[0] != len(kvs):
        raise ValueError(f"q_tokens must be ({len(kvs)}, h)")
    h = heads * d
    return _attend([_check_query(q, h) for q in qs], kvs, _mat("w_o", w_o, h, h))
