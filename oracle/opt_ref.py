"""NumPy OPT decoder with host-offloaded layer inputs / KV and the KVPR
split-merge rebuild — the CPU oracle for logits and greedy tokens.
Oracle only — see oracle/__init__.py.

Algorithm per decode step (s' = prompt_len + step, split l from the plan):
  for each layer j:
    x      = LN1(h)                                   -> X store[j][s'-1]
    q,k,v  = x W_{q,k,v}^T + b                        -> KV store[j][s'-1] (k, v)
    K,V[0:l')   = X store[j][0:l'] W_{k,v}^T + b       (l' = min(l, s'-1); numerics.py:129-133)
    K,V[l':s'-1) = KV store[j][l':s'-1)                (the "transferred" tail; numerics.py:134-137)
    K,V[s'-1]   = k, v                                 (append; numerics.py:140-156)
    a      = per-head softmax(K q / sqrt(d)) V         (numerics.py:166-190, max-subtracted softmax :159-163)
    h     += a W_o^T + b_o;  h += relu(LN2(h) W_1^T + b_1) W_2^T + b_2
  logits = LN_f(h) E^T, token = argmax (ties -> smallest index)

OPT layer semantics (pre-LN, learned positions with offset 2, tied LM head,
biases on every projection) follow transformers' modeling_opt.py; the
reference package has no decoder (SURVEY.md §8a note 2, §8c).

`storage` emulates the dtype of every tensor the B200 path materialises in
memory (X / KV stores and pages, q/k/v, attention output, LN outputs, fc1
output): np.float16 mirrors the GPU run, np.float64 with compute=np.float64
gives the reference's exact-arithmetic semantics.  The residual stream stays
in `compute` precision (fp32 on the GPU).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


# ---------------------------------------------------------------------------
# float16 <-> float32 casts.  NumPy's are scalar; oracle/csrc/fp16conv.c does the same IEEE
# conversions (exact widening, round-to-nearest-even narrowing) with F16C over OpenMP threads.
# Bit-identical either way (tests/test_oracle_cpu.py); the C helper only makes full-depth parity
# checks at OPT-6.7B width affordable.

_FP16 = None


def _fp16lib():
    global _FP16
    if _FP16 is None:
        import ctypes
        from pathlib import Path

        p = Path(__file__).resolve().parent / "libfp16conv.so"
        _FP16 = False
        if p.exists():
            lib = ctypes.CDLL(str(p))
            for name in ("oracle_f16_to_f32", "oracle_f32_to_f16"):
                getattr(lib, name).argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t]
            lib.oracle_f32_round_f16.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
            vp, lg, i = ctypes.c_void_p, ctypes.c_long, ctypes.c_int
            lib.oracle_decode_attention.argtypes = [vp, lg, lg, lg, lg, vp, lg, vp, vp, vp, vp, i, i, i,
                                                    ctypes.c_double, vp]
            _FP16 = lib
    return _FP16


def widen(a: np.ndarray, out: np.ndarray | None = None) -> np.ndarray:
    """float16 array -> float32 (exact), into `out` (C-contiguous, same shape) when given."""
    lib = _fp16lib()
    if out is not None and (not lib or a.dtype != np.float16 or out.dtype != np.float32 or
                            not out.flags.c_contiguous):
        out[...] = a
        return out
    if not lib or a.dtype != np.float16:
        return np.asarray(a, dtype=np.float32).copy() if a.dtype == np.float32 else a.astype(np.float32)
    a = np.ascontiguousarray(a)
    if out is None:
        out = np.empty(a.shape, dtype=np.float32)
    elif out.shape != a.shape or out.dtype != np.float32:
        raise ValueError("widen: out must be float32 of the input's shape")
    lib.oracle_f16_to_f32(a.ctypes.data, out.ctypes.data, a.size)
    return out


def narrow(a: np.ndarray) -> np.ndarray:
    """float32 array -> new float16 array (round to nearest even)."""
    lib = _fp16lib()
    if not lib or a.dtype != np.float32:
        return a.astype(np.float16)
    a = np.ascontiguousarray(a)
    out = np.empty(a.shape, dtype=np.float16)
    lib.oracle_f32_to_f16(a.ctypes.data, out.ctypes.data, a.size)
    return out


def round16(a: np.ndarray) -> np.ndarray:
    """float32 array -> new float32 array holding float(half(a))."""
    lib = _fp16lib()
    if not lib or a.dtype != np.float32:
        return a.astype(np.float16).astype(a.dtype)
    out = np.array(a, dtype=np.float32, order="C")
    lib.oracle_f32_round_f16(out.ctypes.data, out.size)
    return out


def _cast(a: np.ndarray, dtype) -> np.ndarray:
    """a.astype(dtype) through the fast helpers where they apply."""
    if a.dtype == np.float16 and dtype == np.float32:
        return widen(a)
    if a.dtype == np.float32 and dtype == np.float16:
        return narrow(a)
    return a.astype(dtype)


@dataclass(frozen=True)
class OPTShape:
    hidden: int
    layers: int
    heads: int
    ffn: int
    vocab: int
    max_pos: int
    eps: float = 1e-5

    @property
    def head_dim(self) -> int:
        return self.hidden // self.heads


def _mm(x, w):
    """x[..., k] @ w[n, k]^T as ONE GEMM over the flattened leading dims (a 3-D `x @ w.T` is a stack
    of small GEMMs in NumPy, ~3x slower at the rebuild's [l, b, h] shape); same per-row arithmetic."""
    return (x.reshape(-1, x.shape[-1]) @ w.T).reshape(x.shape[:-1] + (w.shape[0],))


def _ln(x, g, b, eps):
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    return (x - mu) / np.sqrt(var + eps) * g + b


def _softmax(z, axis=-1):
    z = z - z.max(axis=axis, keepdims=True)
    e = np.exp(z)
    return e / e.sum(axis=axis, keepdims=True)


class OPTOracle:
    """Weights dict uses the runtime's names (paper_2411_17089_b200.weights), torch layout [out, in]."""

    def __init__(self, shape: OPTShape, weights: dict[str, np.ndarray], batch: int, storage=np.float16,
                 compute=np.float32, kv_bits: int | None = None):
        if kv_bits not in (None, 4):
            raise ValueError("kv_bits must be None or 4")
        if kv_bits and storage is not np.float16:
            raise ValueError("4-bit KV emulation needs fp16 storage")
        self.kv_bits = kv_bits
        self.s = shape
        self.b = batch
        self.storage = storage
        self.compute = compute
        self.w = {k: _cast(np.asarray(v), compute) for k, v in weights.items()}
        self.X: list[np.ndarray] = []   # per layer [S, b, h] storage dtype
        self.KV: list[np.ndarray] = []  # per layer [S, 2, b, h] storage dtype
        self.len = 0

    # -- helpers ------------------------------------------------------------
    def _fast_attention(self, d) -> bool:
        """fp16 storage / fp32 compute: attention straight from the fp16 store rows in C (same math as
        the NumPy branch, double accumulation), which keeps full-depth OPT-6.7B checks affordable."""
        return bool(_fp16lib()) and self.storage is np.float16 and self.compute is np.float32 and \
            d % 8 == 0 and d <= 256

    def _attention_c(self, j, q, k, v, lp, seq):
        b, hd, H, d = self.b, self.s.hidden, self.s.heads, self.s.head_dim
        lib = _fp16lib()
        # rebuilt prefix in the GEMM's own layout [pos][b][K|V] (no re-layout copy)
        kv32 = self._rebuild_rows(j, lp) if lp > 0 else np.zeros((1, b, 2 * hd), dtype=np.float32)
        tail = self.KV[j][lp:seq - 1]
        assert tail.flags.c_contiguous and tail.dtype == np.float16
        q, k, v = (np.ascontiguousarray(t, dtype=np.float32) for t in (q, k, v))
        out = np.empty((b, hd), dtype=np.float32)
        scratch = getattr(self, "_scratch", None)
        if scratch is None or scratch.size < b * H * seq:
            scratch = self._scratch = np.empty(b * H * (len(self.KV[j]) + 1), dtype=np.float64)
        lib.oracle_decode_attention(kv32.ctypes.data, lp, b * 2 * hd, 2 * hd, hd, tail.ctypes.data, seq - 1 - lp,
                                    k.ctypes.data,
                                    v.ctypes.data, q.ctypes.data, out.ctypes.data, b, H, d, 1.0 / np.sqrt(d),
                                    scratch.ctypes.data)
        return out

    def _merge_buffer(self, seq):
        cap = max(seq, len(self.KV[0]) if self.KV else seq)
        buf = getattr(self, "_mbuf", None)
        if buf is None or buf.shape[0] < cap:
            buf = self._mbuf = np.empty((cap, 2, self.b, self.s.hidden), dtype=self.compute)
        return buf

    def _st(self, a):
        if self.storage is np.float16 and self.compute is np.float32:
            return round16(np.asarray(a, dtype=np.float32))
        return a.astype(self.storage).astype(self.compute)

    def _kv_store(self, kv):
        """What the host KV store holds: the fp16 page, or its 4-bit groupwise round trip."""
        if self.kv_bits == 4:
            from . import kvquant_ref

            return kvquant_ref.roundtrip(np.asarray(kv, dtype=np.float16))
        return kv

    def _lw(self, j, name):
        return self.w[f"layers.{j}.{name}"]

    def _proj_qkv(self, j, x):
        h = self.s.hidden
        y = _mm(x, self._lw(j, "wqkv")) + self._lw(j, "bqkv")
        return self._st(y[..., :h]), self._st(y[..., h:2 * h]), self._st(y[..., 2 * h:])

    def _rebuild(self, j, upto):
        """K, V for positions [0, upto) from the X store (numerics.py:129-133)."""
        h = self.s.hidden
        x = _cast(self.X[j][:upto], self.compute)
        wkv = self._lw(j, "wqkv")[h:]
        bkv = self._lw(j, "bqkv")[h:]
        y = _mm(x, wkv) + bkv
        return self._st(y[..., :h]), self._st(y[..., h:])

    def _rebuild_rows(self, j, upto):
        """_rebuild as one [upto, b, 2h] array (K then V per row), fp16-rounded in place."""
        h = self.s.hidden
        y = _mm(_cast(self.X[j][:upto], self.compute), self._lw(j, "wqkv")[h:])
        y += self._lw(j, "bqkv")[h:]
        _fp16lib().oracle_f32_round_f16(y.ctypes.data, y.size)
        return y

    def _mlp_tail(self, j, h, attn):
        h = h + _mm(attn, self._lw(j, "wo")) + self._lw(j, "bo")
        y = self._st(_ln(h, self._lw(j, "ln2.g"), self._lw(j, "ln2.b"), self.s.eps))
        f = self._st(np.maximum(_mm(y, self._lw(j, "w1")) + self._lw(j, "b1"), 0))
        return h + _mm(f, self._lw(j, "w2")) + self._lw(j, "b2")

    def _logits(self, h):
        z = self._st(_ln(h, self.w["lnf.g"], self.w["lnf.b"], self.s.eps))
        return (z @ self.w["embed"].T).astype(np.float32)

    # -- prefill --------------------------------------------------------------
    def prefill(self, tokens: np.ndarray, capacity: int) -> np.ndarray:
        """tokens [b, S0] -> logits of the last prompt position [b, V]; fills the stores."""
        S0 = tokens.shape[1]
        b, hd, H, d = self.b, self.s.hidden, self.s.heads, self.s.head_dim
        pos = np.arange(S0)
        h = (self.w["embed"][tokens.T] + self.w["pos"][pos + 2][:, None, :]).astype(self.compute)  # [S0, b, h]
        self.X, self.KV = [], []
        mask = np.triu(np.ones((S0, S0), dtype=bool), 1)
        for j in range(self.s.layers):
            x = self._st(_ln(h, self._lw(j, "ln1.g"), self._lw(j, "ln1.b"), self.s.eps))
            q, k, v = self._proj_qkv(j, x)
            Xs = np.zeros((capacity, b, hd), dtype=self.storage)
            KVs = np.zeros((capacity, 2, b, hd), dtype=self.storage)
            Xs[:S0] = _cast(x, self.storage)
            KVs[:S0] = self._kv_store(_cast(np.stack([k, v], axis=1), self.storage))
            self.X.append(Xs)
            self.KV.append(KVs)
            qh = q.reshape(S0, b, H, d)
            kh = k.reshape(S0, b, H, d)
            vh = v.reshape(S0, b, H, d)
            lg = np.einsum("tbhd,sbhd->bhts", qh, kh) / np.sqrt(d)
            lg = np.where(mask, -np.inf, lg)
            a = self._st(np.einsum("bhts,sbhd->tbhd", _softmax(lg), vh).reshape(S0, b, hd))
            h = self._mlp_tail(j, h, a)
        self.len = S0
        return self._logits(h[-1])

    # -- one decode step ---------------------------------------------------------
    def decode_step(self, tokens: np.ndarray, split: int, write_stores: bool = True) -> np.ndarray:
        """Input tokens [b] at position self.len; s' = self.len + 1; returns logits [b, V].

        write_stores=False keeps externally supplied store rows for the new position
        (teacher-forced comparison against another run's stores)."""
        seq = self.len + 1
        if not 0 <= split <= seq:
            raise ValueError(f"split must be in [0, {seq}], got {split}")
        b, hd, H, d = self.b, self.s.hidden, self.s.heads, self.s.head_dim
        h = (self.w["embed"][tokens] + self.w["pos"][seq - 1 + 2]).astype(self.compute)  # [b, h]
        lp = min(split, seq - 1)
        for j in range(self.s.layers):
            x = self._st(_ln(h, self._lw(j, "ln1.g"), self._lw(j, "ln1.b"), self.s.eps))
            q, k, v = self._proj_qkv(j, x)
            if write_stores:  # store the new position (store_activation / store_cache, graph.py:340-347)
                self.X[j][seq - 1] = x
                self.KV[j][seq - 1] = self._kv_store(np.stack([k, v])[None].astype(self.storage))[0]
            if self._fast_attention(d):
                a = self._st(self._attention_c(j, q, k, v, lp, seq))
                h = self._mlp_tail(j, h, a)
                continue
            # the merged cache [pos][K|V][b][h] in one buffer reused across layers and steps (first-touch
            # page faults of fresh multi-GB temporaries dominated the oracle's time at full width)
            buf = self._merge_buffer(seq)
            if lp > 0:
                buf[:lp, 0], buf[:lp, 1] = self._rebuild(j, lp)
            if seq - 1 > lp:
                widen(self.KV[j][lp:seq - 1], out=buf[lp:seq - 1])
            buf[seq - 1, 0], buf[seq - 1, 1] = k, v
            K, V = buf[:seq, 0], buf[:seq, 1]
            lg = np.einsum("sbhd,bhd->bhs", K.reshape(seq, b, H, d), q.reshape(b, H, d)) / np.sqrt(d)
            a = self._st(np.einsum("bhs,sbhd->bhd", _softmax(lg), V.reshape(seq, b, H, d)).reshape(b, hd))
            h = self._mlp_tail(j, h, a)
        self.len = seq
        return self._logits(h)


def greedy(logits: np.ndarray) -> np.ndarray:
    return np.argmax(logits, axis=-1).astype(np.int64)


def margins(logits: np.ndarray) -> np.ndarray:
    """top-1 minus top-2 logit per row (how robust the greedy choice is)."""
    part = np.partition(logits, -2, axis=-1)
    return part[:, -1] - part[:, -2]


def generate(shape: OPTShape, weights, prompt: np.ndarray, splits: list[int], storage=np.float16,
             compute=np.float32, forced: np.ndarray | None = None, stores=None, kv_bits: int | None = None):
    """Prefill + len(splits) decode steps. Returns (tokens [steps+1, b], logits list, margins list).

    forced  [steps+1, b]: teacher forcing — step i consumes forced[i] instead of the
            previous greedy token (compares logits on identical inputs).
    stores  (X [L][S][b][h], KV [L][S][2][b][h], first_tokens [b]): decode from
            externally produced host stores (e.g. the GPU run's final stores, which
            also hold the rows it wrote during decode) instead of the oracle's own
            prefill; those rows are read, never overwritten; logits[0] is then None.
    """
    b, S0 = prompt.shape
    o = OPTOracle(shape, weights, b, storage=storage, compute=compute, kv_bits=kv_bits)
    if stores is None:
        lg = o.prefill(prompt, capacity=S0 + len(splits) + 1)
        toks = [greedy(lg)]
        logits = [lg]
    else:
        X, KV, first = stores
        cap = S0 + len(splits) + 1
        # read-only views when the dtype matches (the teacher-forced decode never writes them); the caller
        # keeps the arrays alive (e.g. a runtime's pinned host stores) until generate returns
        o.X = [np.asarray(X[j][:cap], dtype=storage) for j in range(shape.layers)]
        o.KV = [np.asarray(KV[j][:cap], dtype=storage) for j in range(shape.layers)]
        o.len = S0
        toks = [np.asarray(first, dtype=np.int64)]
        logits = [None]
    for i, l in enumerate(splits):
        inp = toks[-1] if forced is None else np.asarray(forced[i], dtype=np.int64)
        lg = o.decode_step(inp, l, write_stores=stores is None)
        logits.append(lg)
        toks.append(greedy(lg))
    return np.stack(toks), logits, [margins(x) if x is not None else None for x in logits]
