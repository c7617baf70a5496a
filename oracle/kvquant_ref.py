"""NumPy restatement of the 4-bit groupwise KV page format — oracle only
(see oracle/__init__.py).  Costing follows costmodel.groupwise_quant_bytes_per_element
(costmodel.py:109-118: 4 bits + 4 scale bytes per 64-element group = 0.5625 B/elem);
the reference prices the format but has no codec, so the codec here restates the
asymmetric min/max scheme the product kernel implements (csrc/kvquant.cu), in
float32 with the same rounding points, so outputs are bit-comparable.
"""

from __future__ import annotations

import numpy as np


def page_bytes(batch: int, hidden: int) -> int:
    e = 2 * batch * hidden
    return e // 2 + (e // 64) * 4


def quantize(pages: np.ndarray) -> np.ndarray:
    """fp16 pages [P][2][b][h] -> uint8 compressed pages [P][page_bytes] (codes then (min, scale) fp16)."""
    P, two, b, h = pages.shape
    x = pages.astype(np.float32).reshape(P, -1, 64)  # groups along h
    mn16 = x.min(axis=-1).astype(np.float16)
    mnf = mn16.astype(np.float32)
    sc16 = ((x.max(axis=-1) - mnf) / np.float32(15)).astype(np.float16)
    scf = sc16.astype(np.float32)
    safe = np.where(scf > 0, scf, np.float32(1))
    q = np.rint((x - mnf[..., None]) / safe[..., None])
    q = np.where(scf[..., None] > 0, np.clip(q, 0, 15), 0).astype(np.uint8)
    codes = (q[..., 0::2] | (q[..., 1::2] << 4)).reshape(P, -1)
    prm = np.stack([mn16, sc16], axis=-1).reshape(P, -1).view(np.uint8)
    return np.concatenate([codes, prm], axis=1)


def dequantize(qpages: np.ndarray, batch: int, hidden: int) -> np.ndarray:
    P = qpages.shape[0]
    e = 2 * batch * hidden
    codes = qpages[:, : e // 2].reshape(P, -1, 32)
    prm = np.ascontiguousarray(qpages[:, e // 2:]).view(np.float16).reshape(P, -1, 2).astype(np.float32)
    q = np.empty(codes.shape[:-1] + (64,), dtype=np.float32)
    q[..., 0::2] = codes & 15
    q[..., 1::2] = codes >> 4
    x = prm[..., 0:1] + q * prm[..., 1:2]
    return x.astype(np.float16).reshape(P, 2, batch, hidden)


def roundtrip(pages: np.ndarray) -> np.ndarray:
    P, _, b, h = pages.shape
    return dequantize(quantize(pages), b, h)
