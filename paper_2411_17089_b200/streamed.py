"""Throughput-oriented KVPR decode (paper §3.3, Table 3):
weights offloaded to page-locked host memory and streamed per layer over
PCIe, `num_batches` GPU batches walked layer-major (the column schedule,
graph.py:128-134) so one weight load is amortised over all batches, and
fine-grained weight loads — W_K|W_V first, so K1 (which needs only them) can
start as soon as the first X chunk lands, then W_Q|W_O and the FFN — the
priority order of graph.py:56-67, 237-264 (load_weight kv / qo halves).

Per global layer g = step*L + j the copy stream carries, in order,
    [W_kv(g)] [X chunks of (g, k=0)] [W_q, W_o, FFN (g)] [KV tail (g, 0)]
    [X (g, 1)] [KV (g, 1)] ... [X (g, K-1)] [KV (g, K-1)]
and the compute stream runs, per batch k, K1 on each landed chunk, then
LN1 -> q,k,v -> [KV landed] K2 -> out-proj -> FFN.  Weights are double
buffered by layer, KV/X pages by unit; events only, no host syncs.
Everything else (layouts, kernels, plan) is the resident runtime's.
"""

from __future__ import annotations

import torch

from . import _lib, kernels
from .hostmem import pinned_empty, unpin
from .runtime import F16, F32, HostStores, _copy, chunk_bounds
from .weights import LayerWeights, OPTWeights

_FIELDS = ("wqkv", "bqkv", "wo", "bo", "ln1_g", "ln1_b", "ln2_g", "ln2_b", "w1", "b1", "w2", "b2")


def _shapes(h: int, f: int) -> dict:
    return {"wqkv": (3 * h, h), "bqkv": (3 * h,), "wo": (h, h), "bo": (h,), "ln1_g": (h,), "ln1_b": (h,),
            "ln2_g": (h,), "ln2_b": (h,), "w1": (f, h), "b1": (f,), "w2": (h, f), "b2": (h,)}


def _numel(shape) -> int:
    n = 1
    for s in shape:
        n *= s
    return n


def _views(flat: torch.Tensor, h: int, f: int) -> LayerWeights:
    """LayerWeights whose tensors are views into one flat fp16 buffer (layout = _FIELDS order)."""
    out, off = {}, 0
    for name, shape in _shapes(h, f).items():
        n = _numel(shape)
        out[name] = flat[off:off + n].view(*shape)
        off += n
    return LayerWeights(**out)


def weight_regions(h: int, f: int, part: str) -> list[tuple[int, int]]:
    """(byte offset, bytes) DMA ranges of one layer's flat weight buffer.

    'kv' = W_k|W_v rows and b_k|b_v (what K1 needs, loaded first under fine granularity);
    'rest' = W_q rows, b_q, and W_o .. b2; 'all' = the whole layer.  kv + rest tile the buffer.
    """
    total = sum(_numel(s) for s in _shapes(h, f).values()) * 2
    if part == "all":
        return [(0, total)]
    wq = h * h * 2  # bytes of W_q rows (wqkv rows [0:h])
    bqkv0 = 3 * h * h * 2  # byte offset of bqkv
    if part == "kv":
        return [(wq, 2 * h * h * 2), (bqkv0 + 2 * h, 4 * h)]
    if part == "rest":
        rest0 = bqkv0 + 6 * h
        return [(0, wq), (bqkv0, 2 * h), (rest0, total - rest0)]
    raise ValueError(f"unknown weight part {part!r}")


class StreamedRuntime:
    """num_batches x batch sequences; layer weights streamed from host each layer."""

    def __init__(self, weights: OPTWeights, batch: int, num_batches: int, capacity: int,
                 device: torch.device | str | None = None, granularity: str = "fine", chunks: int = 4):
        if granularity not in ("fine", "coarse"):
            raise ValueError("granularity must be 'fine' or 'coarse'")
        cfg = weights.cfg
        if capacity > cfg.max_pos:
            raise ValueError(f"capacity {capacity} exceeds the position table ({cfg.max_pos})")
        self.cfg, self.batch, self.K, self.capacity = cfg, batch, num_batches, capacity
        self.fine, self.chunks = granularity == "fine", chunks
        self.dev = torch.device(device) if device is not None else weights.embed.device
        _lib.load()
        h, f, b, L = cfg.hidden, cfg.ffn, batch, cfg.layers
        self.layer_numel = sum(_numel(s) for s in _shapes(h, f).values())
        # host: all layers' weights in one page-locked flat buffer (views per layer)
        self.host_w = pinned_empty((L, self.layer_numel), F16)  # page-locked like the host stores (hostmem)
        for j, lw in enumerate(weights.layers):
            hv = _views(self.host_w[j], h, f)
            for name in _FIELDS:
                getattr(hv, name).copy_(getattr(lw, name))
        # resident: embeddings / final LN (tied LM head); device weight slots for 2 layers
        self.embed, self.pos, self.lnf_g, self.lnf_b = (t.to(self.dev) for t in
                                                         (weights.embed, weights.pos, weights.lnf_g, weights.lnf_b))
        self.dev_w = torch.empty(2, self.layer_numel, dtype=F16, device=self.dev)
        self.slots = [_views(self.dev_w[i], h, f) for i in range(2)]
        self.stores = [HostStores(L, capacity, b, h) for _ in range(num_batches)]
        z = lambda *s, dt=F16: torch.empty(*s, dtype=dt, device=self.dev)  # noqa: E731
        self.kv_dev = z(2, capacity, 2, b, h)
        self.x_dev = z(2, capacity, b, h)
        self.hres = z(num_batches, b, h, dt=F32)
        self.tok = z(num_batches, b, dt=torch.int32)
        self.q, self.attn, self.y, self.zf = z(b, h), z(b, h), z(b, h), z(b, h)
        self.mid = z(b, f)
        self.logits = z(b, cfg.vocab, dt=F32)
        self.ws = z(16 << 20, dt=torch.uint8)
        self.cs = torch.cuda.Stream(self.dev, priority=-1)
        self.hs = torch.cuda.Stream(self.dev)
        self.ds = torch.cuda.Stream(self.dev)
        self.len = 0
        self.launches = 0
        self.h2d_bytes = 0

    # ------------------------------------------------------------ weight DMA
    def _load_w(self, g: int, part: str, stream) -> None:
        j, slot = g % self.cfg.layers, g % 2
        src = self.host_w[j].data_ptr()
        dst = self.dev_w[slot].data_ptr()
        for off, n in weight_regions(self.cfg.hidden, self.cfg.ffn, part):
            _copy(dst + off, src + off, n, stream)
            self.h2d_bytes += n

    # ----------------------------------------------------------------- prefill
    def prefill(self, prompts: list[torch.Tensor]) -> torch.Tensor:
        """prompts: num_batches tensors [batch, S0].  Returns first tokens [num_batches, batch]."""
        cfg, b, h, K = self.cfg, self.batch, self.cfg.hidden, self.K
        if len(prompts) != K:
            raise ValueError(f"need {K} prompts, got {len(prompts)}")
        S0 = int(prompts[0].shape[1])
        rows = S0 * b
        cs = self.cs
        with torch.cuda.stream(cs):
            hb = [torch.empty(rows, h, dtype=F32, device=self.dev) for _ in range(K)]
            x = torch.empty(rows, h, dtype=F16, device=self.dev)
            q = torch.empty(rows, h, dtype=F16, device=self.dev)
            a = torch.empty(rows, h, dtype=F16, device=self.dev)
            mid = torch.empty(rows, cfg.ffn, dtype=F16, device=self.dev)
            pages = self.kv_dev[0]
            for k, p in enumerate(prompts):
                toks = p.to(self.dev).to(torch.int32).t().contiguous()
                kernels.embed(toks.view(-1), self.embed, self.pos, hb[k], batch=b, pos_begin=0, stream=cs)
            for j in range(cfg.layers):
                self._load_w(j, "all", cs)
                lw = self.slots[j % 2]
                for k in range(K):
                    st = self.stores[k]
                    kernels.layernorm(hb[k], lw.ln1_g, lw.ln1_b, x, eps=cfg.eps, stream=cs)
                    self._qkv(x, rows, lw, q, pages[:S0], q_group=b * h, stream=cs)
                    _copy(st.x[j].data_ptr(), x.data_ptr(), rows * h * 2, cs)
                    _copy(st.kv[j].data_ptr(), pages.data_ptr(), S0 * 2 * b * h * 2, cs)
                    kernels.prefill_attention(q, pages, a, b, cfg.heads, cfg.head_dim, S0, stream=cs)
                    acc = _lib.EPI_F32 | _lib.EPI_ACCUM
                    kernels.linear_simple(a, lw.wo, lw.bo, hb[k], flags=acc, stream=cs, ws=self.ws)
                    kernels.layernorm(hb[k], lw.ln2_g, lw.ln2_b, x, eps=cfg.eps, stream=cs)
                    kernels.linear_simple(x, lw.w1, lw.b1, mid, flags=_lib.EPI_RELU, stream=cs, ws=self.ws)
                    kernels.linear_simple(mid, lw.w2, lw.b2, hb[k], flags=acc, stream=cs, ws=self.ws)
            for k in range(K):
                self._head(hb[k][(S0 - 1) * b:], k)
        with torch.cuda.stream(cs):
            first = self.tok.clone()
        cs.synchronize()
        self.len = S0
        return first

    # ---------------------------------------------------------- layer pieces
    def _qkv(self, x, M, lw, q_out, pages, q_group, stream):
        b, h = self.batch, self.cfg.hidden
        bh = b * h
        kp = pages.data_ptr()
        epi = _lib.make_epilogue([(q_out.data_ptr(), q_group), (kp, 2 * bh), (kp + bh * 2, 2 * bh)],
                                 seg_width=h, ld=h, row_group=b, bias=lw.bqkv.data_ptr())
        kernels.linear(x, lw.wqkv, epi, M=M, stream=stream)

    def _head(self, hrows, k):
        cs = self.cs
        kernels.layernorm(hrows, self.lnf_g, self.lnf_b, self.zf, eps=self.cfg.eps, stream=cs)
        kernels.linear_simple(self.zf, self.embed, None, self.logits, stream=cs, ws=self.ws)
        kernels.argmax(self.logits, self.tok[k], stream=cs)

    # ------------------------------------------------------------------ decode
    def decode(self, splits: list[int], tokens: torch.Tensor | None = None, keep_logits: bool = False) -> torch.Tensor:
        """len(splits) steps for all num_batches batches; returns device int32 [steps, num_batches, batch]."""
        cfg, b, h, K, L = self.cfg, self.batch, self.cfg.hidden, self.K, self.cfg.layers
        steps, base = len(splits), self.len
        if base + steps > self.capacity:
            raise ValueError(f"cache capacity {self.capacity} exceeded ({base} + {steps} steps)")
        for i, l in enumerate(splits):
            if not 0 <= l <= base + i + 1:
                raise ValueError(f"step {i + 1}: split {l} out of range [0, {base + i + 1}]")
        cs, hs, ds = self.cs, self.hs, self.ds
        cur = torch.cuda.current_stream(self.dev)
        cs.wait_stream(cur)  # the caller's work (e.g. the H2D of `tokens`) precedes this run
        hs.wait_stream(cur)
        if tokens is not None:
            with torch.cuda.stream(cs):
                self.tok.copy_(tokens.to(torch.int32), non_blocking=True)
        out = torch.empty(steps, K, b, dtype=torch.int32, device=self.dev)
        logits = torch.empty(steps, K, b, cfg.vocab, dtype=F32, device=self.dev) if keep_logits else None
        ev = {k: {} for k in ("x", "kv", "wkv", "wrest", "done", "d2h", "layer_done")}
        E = lambda: torch.cuda.Event()  # noqa: E731
        n = steps * L * K

        def unit(u):
            g, k = divmod(u, K)
            i, j = divmod(g, L)
            s = base + i + 1
            return g, k, i, j, s, min(splits[i], s - 1)

        def issue(u):
            g, k, _, j, s, lp = unit(u)
            buf = u % 2
            if u >= 2:
                hs.wait_event(ev["done"][u - 2])
                hs.wait_event(ev["d2h"][u - 2])
            if u >= L * K:
                hs.wait_event(ev["d2h"][u - L * K])
            if k == 0:
                if g >= 2:  # weight slot g % 2 free once layer g-2's last batch finished
                    hs.wait_event(ev["layer_done"][g - 2])
                self._load_w(g, "kv" if self.fine else "all", hs)
                ev["wkv"][g] = E()
                ev["wkv"][g].record(hs)
            st = self.stores[k]
            xd, kvd = self.x_dev[buf], self.kv_dev[buf]
            row = b * h * 2
            ev["x"][u] = []
            for p0, p1 in chunk_bounds(lp, self.chunks):
                _copy(xd[p0].data_ptr(), st.x[j][p0].data_ptr(), (p1 - p0) * row, hs)
                self.h2d_bytes += (p1 - p0) * row
                e = E()
                e.record(hs)
                ev["x"][u].append(e)
            if k == 0:
                if self.fine:
                    self._load_w(g, "rest", hs)
                ev["wrest"][g] = E()
                ev["wrest"][g].record(hs)
            _copy(kvd[lp].data_ptr(), st.kv[j][lp].data_ptr(), (s - 1 - lp) * 2 * row, hs)
            self.h2d_bytes += (s - 1 - lp) * 2 * row
            ev["kv"][u] = E()
            ev["kv"][u].record(hs)

        def compute(u):
            g, k, i, j, s, lp = unit(u)
            buf = u % 2
            lw = self.slots[g % 2]
            st = self.stores[k]
            xd, kvd = self.x_dev[buf], self.kv_dev[buf]
            x_slot, page = xd[s - 1], kvd[s - 1]
            hres = self.hres[k]
            if u >= 2:
                cs.wait_event(ev["d2h"][u - 2])
            if j == 0:
                kernels.embed(self.tok[k], self.embed, self.pos, hres, batch=b, pos_begin=s - 1, stream=cs)
            cs.wait_event(ev["wkv"][g])
            for e, (p0, p1) in zip(ev["x"][u], chunk_bounds(lp, self.chunks)):
                cs.wait_event(e)
                kernels.recompute_kv(xd, lw.w_kv, lw.b_kv, kvd, b, p0, p1, stream=cs)
            cs.wait_event(ev["wrest"][g])
            kernels.layernorm(hres, lw.ln1_g, lw.ln1_b, x_slot, eps=cfg.eps, stream=cs)
            self._qkv(x_slot, b, lw, self.q, page, 0, cs)
            eq = E()
            eq.record(cs)
            ds.wait_event(eq)
            _copy(st.x[j][s - 1].data_ptr(), x_slot.data_ptr(), b * h * 2, ds)
            _copy(st.kv[j][s - 1].data_ptr(), page.data_ptr(), 2 * b * h * 2, ds)
            ev["d2h"][u] = E()
            ev["d2h"][u].record(ds)
            cs.wait_event(ev["kv"][u])
            kernels.decode_attention(self.q, kvd, self.attn, self.ws, b, cfg.heads, cfg.head_dim, s, stream=cs)
            acc = _lib.EPI_F32 | _lib.EPI_ACCUM
            kernels.linear_simple(self.attn, lw.wo, lw.bo, hres, flags=acc, stream=cs, ws=self.ws)
            kernels.layernorm(hres, lw.ln2_g, lw.ln2_b, self.y, eps=cfg.eps, stream=cs)
            kernels.linear_simple(self.y, lw.w1, lw.b1, self.mid, flags=_lib.EPI_RELU, stream=cs, ws=self.ws)
            kernels.linear_simple(self.mid, lw.w2, lw.b2, hres, flags=acc, stream=cs, ws=self.ws)
            ev["done"][u] = E()
            ev["done"][u].record(cs)
            if k == K - 1:
                ev["layer_done"][g] = ev["done"][u]
            if j == L - 1:
                self._head(hres, k)
                with torch.cuda.stream(cs):
                    out[i, k].copy_(self.tok[k], non_blocking=True)
                    if logits is not None:
                        logits[i, k].copy_(self.logits, non_blocking=True)

        n0 = _lib.load().kvpr_kernel_launches()
        issue(0)
        ahead = L * K > 1  # a single unit per step: unit u+1's loads wait on unit u's D2H (its compute)
        for u in range(n):
            if ahead and u + 1 < n:
                issue(u + 1)
            compute(u)
            if not ahead and u + 1 < n:
                issue(u + 1)
            g_now = u // K
            for name, d in ev.items():  # drop events no longer referenced (unit- or layer-keyed)
                lim = g_now - 4 if name in ("wkv", "wrest", "layer_done") else u - L * K - 4
                for key in [key for key in d if key < lim]:
                    del d[key]
        self.len = base + steps
        self.launches += _lib.load().kvpr_kernel_launches() - n0
        cur.wait_stream(cs)
        cur.wait_stream(ds)
        self.last_logits = logits
        return out

    def close(self) -> None:
        for st in self.stores:
            st.close()
        unpin(self.host_w)
