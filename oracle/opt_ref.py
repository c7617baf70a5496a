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
        self.w = {k: np.asarray(v).astype(compute) for k, v in weights.items()}
        self.X: list[np.ndarray] = []   # per layer [S, b, h] storage dtype
        self.KV: list[np.ndarray] = []  # per layer [S, 2, b, h] storage dtype
        self.len = 0

    # -- helpers ------------------------------------------------------------
    def _st(self, a):
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
        y = x @ self._lw(j, "wqkv").T + self._lw(j, "bqkv")
        return self._st(y[..., :h]), self._st(y[..., h:2 * h]), self._st(y[..., 2 * h:])

    def _rebuild(self, j, upto):
        """K, V for positions [0, upto) from the X store (numerics.py:129-133)."""
        h = self.s.hidden
        x = self.X[j][:upto]
        wkv = self._lw(j, "wqkv")[h:]
        bkv = self._lw(j, "bqkv")[h:]
        y = x @ wkv.T + bkv
        return self._st(y[..., :h]), self._st(y[..., h:])

    def _mlp_tail(self, j, h, attn):
        h = h + attn @ self._lw(j, "wo").T + self._lw(j, "bo")
        y = self._st(_ln(h, self._lw(j, "ln2.g"), self._lw(j, "ln2.b"), self.s.eps))
        f = self._st(np.maximum(y @ self._lw(j, "w1").T + self._lw(j, "b1"), 0))
        return h + f @ self._lw(j, "w2").T + self._lw(j, "b2")

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
            Xs[:S0] = x
            KVs[:S0] = self._kv_store(np.stack([k, v], axis=1).astype(self.storage))
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
            K = np.empty((seq, b, hd), dtype=self.compute)
            V = np.empty((seq, b, hd), dtype=self.compute)
            if lp > 0:
                K[:lp], V[:lp] = self._rebuild(j, lp)
            K[lp:seq - 1] = self.KV[j][lp:seq - 1, 0]
            V[lp:seq - 1] = self.KV[j][lp:seq - 1, 1]
            K[seq - 1], V[seq - 1] = k, v
            # store the new position (store_activation / store_cache, graph.py:340-347)
            if write_stores:
                self.X[j][seq - 1] = x
                self.KV[j][seq - 1] = self._kv_store(np.stack([k, v])[None].astype(self.storage))[0]
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
        o.X = [np.array(X[j][:cap], dtype=storage) for j in range(shape.layers)]
        o.KV = [np.array(KV[j][:cap], dtype=storage) for j in range(shape.layers)]
        o.len = S0
        toks = [np.asarray(first, dtype=np.int64)]
        logits = [None]
    for i, l in enumerate(splits):
        inp = toks[-1] if forced is None else np.asarray(forced[i], dtype=np.int64)
        lg = o.decode_step(inp, l, write_stores=stores is None)
        logits.append(lg)
        toks.append(greedy(lg))
    return np.stack(toks), logits, [margins(x) if x is not None else None for x in logits]
