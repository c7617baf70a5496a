"""KVPR decode runtime on one B200: weights resident in HBM, each layer's
inputs X and KV cache offloaded to page-locked host memory, and per layer

    copy stream     H2D X[:, :l] (chunked)  ->  H2D KV[l:s'-1]          (one DMA each)
    compute stream  LN1 -> q,k,v (k,v appended at page s'-1) -> K1 on each
                    landed X chunk -> [wait KV] -> K2 attention -> out-proj
                    -> LN2 -> fc1 -> fc2
    d2h stream      new X row and new K,V page -> host stores

ordered only by CUDA events, with layer u+1's transfers issued while layer u
computes (double-buffered device pages).  This realises the task DAG of the
reference simulator (pipesim/graph.py:1-28, 232-347; Algorithm 1 of the
paper): MHA waits on recompute AND the KV load, the
recompute waits on its staged activations, the KV load of step i waits on the
store of step i-1, H2D issue order is activations-for-recompute before KV
(graph.py:56-67), double-buffer depth 2 (graph.py:215-221).  The split l per
step comes from the bit-exact solver (scheduler.plan_generation); the
runtime executes whatever plan it is given (plan JSON, constant plans for
sweeps).  Nothing here computes on the CPU and there is no fallback path:
every kernel is a libkvpr.so launch.

Device layouts (include/kvpr.h): pages [pos][2][batch][hidden] fp16 (K then V);
X [pos][batch][hidden] fp16; residual stream fp32 [batch][hidden].
Host stores use the same position-major layout per layer, so X[:, :l] and
KV[l:s'-1] are single contiguous byte ranges.
"""

from __future__ import annotations

import os

from dataclasses import dataclass, field

import torch

from . import _lib, kernels
from .hostmem import pinned_empty, unpin
from .weights import OPTWeights

F16 = torch.float16
F32 = torch.float32


def _copy(dst_ptr: int, src_ptr: int, nbytes: int, stream: torch.cuda.Stream) -> None:
    if nbytes:
        _lib.call("kvpr_copy_async", dst_ptr, src_ptr, nbytes, stream.cuda_stream)


def _copy_batch(copies, stream: torch.cuda.Stream) -> None:
    """[(dst_ptr, src_ptr, nbytes), ...] enqueued by one C call (kvpr_copy_batch_async; one cudaMemcpyAsync each)."""
    import ctypes

    n = len(copies)
    dsts = (ctypes.c_void_p * n)(*[c[0] for c in copies])
    srcs = (ctypes.c_void_p * n)(*[c[1] for c in copies])
    sizes = (ctypes.c_size_t * n)(*[c[2] for c in copies])
    _lib.call("kvpr_copy_batch_async", dsts, srcs, sizes, n, stream.cuda_stream)


class HostStores:
    """Per-layer X and KV stores in page-locked host memory, exact size (hostmem.pinned_empty)."""

    def __init__(self, layers: int, capacity: int, batch: int, hidden: int, kv_page_bytes: int | None = None,
                 with_x: bool = True):
        self.layers, self.capacity, self.batch, self.hidden = layers, capacity, batch, hidden
        self.x = pinned_empty((layers, capacity if with_x else 0, batch, hidden), F16)
        if kv_page_bytes is None:  # fp16 pages [pos][2][b][h]
            self.kv = pinned_empty((layers, capacity, 2, batch, hidden), F16)
        else:  # compressed pages (4-bit groupwise), kv_page_bytes each
            self.kv = pinned_empty((layers, capacity, kv_page_bytes), torch.uint8)

    @property
    def nbytes(self) -> int:
        return self.x.numel() * 2 + self.kv.numel() * self.kv.element_size()

    def close(self) -> None:
        unpin(self.x)
        unpin(self.kv)

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass


@dataclass
class DecodeTiming:
    """CUDA-event timings of a decode run (compute stream)."""

    step_ms: list[float] = field(default_factory=list)
    layer_ms: list[list[float]] = field(default_factory=list)  # per step, per layer (consecutive layer ends)


def chunk_bounds(n: int, chunks: int, min_rows: int = 64, wave: int = 0) -> list[tuple[int, int]]:
    """Split [0, n) into <= chunks contiguous position ranges (>= min_rows each when possible).

    wave > 0 (and n >= wave): every range but the last is a multiple of `wave` positions, so the
    K1 launch of each full chunk is a whole number of tile waves (wave_positions())."""
    if n <= 0:
        return []
    if wave > 0 and n >= wave:
        per = wave * -(-(-(-n // wave)) // chunks)  # wave x ceil(ceil(n / wave) / chunks)
        per = max(per, wave * -(-min_rows // wave))
        out = [(p, min(n, p + per)) for p in range(0, n, per)]
        if len(out) > 1 and out[-1][1] - out[-1][0] < per // 2:  # a short tail rides on the last chunk
            out[-2:] = [(out[-2][0], n)]
        return out
    c = max(1, min(chunks, n // min_rows if n >= min_rows else 1))
    base, rem = divmod(n, c)
    out, p = [], 0
    for i in range(c):
        q = p + base + (1 if i < rem else 0)
        out.append((p, q))
        p = q
    return out


def wave_positions(batch: int, hidden: int, sms: int, max_positions: int = 1024) -> int:
    """Smallest position count whose K1 launch is whole waves of the CTA-pair kernel, else 0.

    K1 over P positions is ceil(P*batch/256) x ceil(2h/256) tiles of 256 x 256 on sms/2 CTA pairs
    (csrc/gemm_tcgen05.cu).  At OPT-6.7B b32 that is P = 296 (37 m-blocks x 32 n-blocks = 16 waves
    of 74 pairs) instead of the 12.1 waves of an even 4-way split of l = 888, whose last wave runs
    ~10% full."""
    pairs, n_blk = sms // 2, -(-2 * hidden // 256)
    for p in range(1, max_positions + 1):
        if (p * batch) % 256 == 0 and ((p * batch // 256) * n_blk) % pairs == 0:
            return p
    return 0


class KVPRRuntime:
    """One decoder replica on one GPU (the unit the batch-partitioned multi-GPU mode replicates)."""

    def __init__(self, weights: OPTWeights, batch: int, capacity: int, device: torch.device | str | None = None,
                 chunks: int = 4, nbuf: int | None = None, stores: HostStores | None = None, kv_bits: int | None = None,
                 x_resident: bool = False, chunk_rows: int | None = None, chunk_wave: int | None = None,
                 k1_stream: bool | None = None, fused_tail: bool | None = None, dma_group: int | None = None):
        """kv_bits=4 stores/streams the KV cache as 4-bit groupwise pages (kv_bytes_per_element 0.5625).

        x_resident=True is the reference's *row* schedule (graph.py:16-17, scheduler.py:88-92): layer
        inputs X stay in HBM (no activation traffic, t_act = 0), only KV[l:s'-1] crosses PCIe, and K1
        reads X[0:l] from the resident store; plan it with mode "row"."""
        cfg = weights.cfg
        if kv_bits not in (None, 4):
            raise ValueError("kv_bits must be None (fp16) or 4")
        self.kv_bits = kv_bits
        if capacity > cfg.max_pos:
            raise ValueError(f"capacity {capacity} exceeds the position table ({cfg.max_pos})")
        self.cfg, self.w, self.batch, self.capacity = cfg, weights, batch, capacity
        self.dev = torch.device(device) if device is not None else weights.embed.device
        # env: A/B knob; at most 16 chunks, the native executor's per-unit chunk table (executor.cu)
        # device buffers per category (graph.py:215-221 uses 2): small-batch layers whose step is bound by
        # the DMA pipeline rather than the GPU keep 4 in flight; KVPR_NBUF overrides
        if fused_tail is None:
            fused_tail = os.environ.get("KVPR_FUSED_TAIL", "1") != "0"
        fused_ok = (bool(fused_tail) and kv_bits is None
                    and kernels.layer_tail_supported(batch, cfg.hidden, cfg.heads, cfg.ffn))
        if nbuf is None:
            nbuf = int(os.environ.get("KVPR_NBUF", 4 if fused_ok else 2))
        # small layers (a whole X store under 8 MB): the KV tails of G consecutive layers go as one strided
        # DMA (native executor); a ~0.1 MB tail is ~1.8 us of PCIe but ~3.7 us of copy-engine overhead on
        # its own (profiles/r02_dma_2d_probe.json).  X stays one DMA per layer.  G divides the layers
        # (layers >= 2G), G buffers per group in flight twice over (nbuf >= 2G); the smallest G wins (config
        # 1, medians of 5: G 1 / 2 / 3 / 4 = 0.511 / 0.473 / 0.477 / 0.483 ms per step,
        # profiles/r02_c1_dma_group.jsonl: larger groups hold the first layer's K2 for the group's copy).
        # KVPR_DMA_GROUP overrides.
        if dma_group is None:
            dma_group = int(os.environ.get("KVPR_DMA_GROUP", -1))
        if dma_group < 0:
            small = capacity * batch * cfg.hidden * 2 < (8 << 20)
            dma_group = next((g for g in (2, 3, 4) if small and cfg.layers % g == 0 and cfg.layers >= 2 * g), 1)
        self.dma_group = max(1, dma_group)
        if self.dma_group > 1:
            nbuf = self.dma_group * max(2, -(-nbuf // self.dma_group))
        self.chunks, self.nbuf = max(1, min(16, int(os.environ.get("KVPR_CHUNKS", chunks)))), nbuf
        # a K1 chunk carries >= KVPR_CHUNK_MB (default 32) MiB of X (>= 64 positions): every extra X
        # DMA costs copy-engine time (OPT-6.7B b4: 1/2/4/8 chunks of ~30 MB of X in total -> 98.8 /
        # 97.4 / 96.0 / 94.1% of the overlap roofline, profiles/r01_chunk_ab.jsonl), so small batches
        # and small models issue one X copy + one K1 per layer (tests lower it to cover chunking)
        chunk_mb = float(os.environ.get("KVPR_CHUNK_MB", 32))
        self.chunk_rows = chunk_rows or max(64, -(-int(chunk_mb * (1 << 20)) // (batch * cfg.hidden * 2)))
        # X chunks in whole K1 waves when the wave is short enough to still pipeline (<= l / 2)
        if chunk_wave is None:
            chunk_wave = 0 if chunk_rows else wave_positions(
                batch, cfg.hidden, torch.cuda.get_device_properties(self.dev).multi_processor_count)
        self.chunk_wave = chunk_wave
        _lib.load()
        h, b = cfg.hidden, batch
        with torch.cuda.device(self.dev):
            self.cs = torch.cuda.Stream(self.dev, priority=-1)  # compute
            self.hs = torch.cuda.Stream(self.dev)              # H2D copy engine
            self.ds = torch.cuda.Stream(self.dev)              # D2H copy engine
            self.rs = torch.cuda.Stream(self.dev)              # K1 issued a unit ahead (native executor)
        # native executor: K1 on its own stream, issued a unit ahead, for small models whose K1 never
        # fills a wave (the layer chain is latency-bound and K1 overlaps it).  At full width K1 stays on
        # the compute stream: a PCIe-bound column schedule hides it anyway, and in the row schedule a K1
        # holding SMs under the next layer's stream-K projections costs more than the overlap gains
        # (config 2 row, same box: 536 vs 514 tok/s, profiles/r02_row_k1_stream.jsonl).
        # KVPR_K1_STREAM=0/1 forces it.
        env = os.environ.get("KVPR_K1_STREAM")
        if k1_stream is None:
            k1_stream = (env == "1") if env in ("0", "1") else None
        self.k1_stream = (self.chunk_wave == 0) if k1_stream is None else bool(k1_stream)
        # batch <= 8 on a small model: the layer after q/k/v runs as one cooperative kernel (K2 -> out-proj
        # -> LN2 -> fc1 -> fc2, plus the next LN1), csrc/layer_tail.cu; fused_tail=False (or
        # KVPR_FUSED_TAIL=0) keeps the multi-kernel chain, whose bits the streamed and TP runtimes share.
        # Not with 4-bit KV (K2-kv4) or a trace (per-kind spans need the separate kernels)
        self.fused_tail = fused_ok
        # with the fused tail, PCIe traffic the SMs move themselves instead of a copy-engine DMA
        # (KVPR_TAIL_ZC: "r" = the tail reads KV[l:s'-1] from the host store, "w" = it writes the next
        # unit's X row and k,v page to the host stores)
        zc = os.environ.get("KVPR_TAIL_ZC", "")
        self.zc_read = self.fused_tail and "r" in zc
        self.zc_write = self.fused_tail and "w" in zc
        self.qbytes = kernels.kv4_page_bytes(b, h) if kv_bits == 4 else None
        self.page_bytes = self.qbytes if kv_bits == 4 else 2 * b * h * 2
        self.x_resident = x_resident
        self.stores = stores or HostStores(cfg.layers, capacity, batch, h, self.qbytes, with_x=not x_resident)
        z = lambda *s, dt=F16: torch.empty(*s, dtype=dt, device=self.dev)  # noqa: E731
        self.kv_dev = z(nbuf, capacity, 2, b, h)
        self.x_store = z(cfg.layers, capacity, b, h) if x_resident else None
        if kv_bits == 4:  # compressed staging: the transferred tail, and the new page on its way out
            self.kvq_dev = z(nbuf, capacity, self.qbytes, dt=torch.uint8)
            self.qnew = z(nbuf, self.qbytes, dt=torch.uint8)
        self.x_dev = z(nbuf, capacity, b, h)
        self.hres = z(b, h, dt=F32)
        self.q = z(b, h)
        self.attn = z(b, h)
        self.y = z(b, h)
        self.mid = z(b, cfg.ffn)
        self.zf = z(b, h)
        self.logits = z(b, cfg.vocab, dt=F32)
        self.tok = z(b, dt=torch.int32)
        self.ws = z(16 << 20, dt=torch.uint8)
        self.len = 0
        R = cfg.layers + nbuf + 2
        self._R = R
        ev = lambda: torch.cuda.Event(enable_timing=False)  # noqa: E731
        self.ev_x = [[ev() for _ in range(self.chunks)] for _ in range(R)]
        self.ev_kv = [ev() for _ in range(R)]
        self.ev_qkv = [ev() for _ in range(R)]
        self.ev_d2h = [ev() for _ in range(R)]
        self.ev_done = [torch.cuda.Event(enable_timing=True) for _ in range(R)]
        self.launches = 0  # kernels libkvpr launched for this runtime's decode calls (library counter)
        self._trace = None
        self.kernel_timing: list | None = None  # set to [] to time K1 / K2 launches with CUDA events

    # ------------------------------------------------------------------ utils
    def _ktimer(self, name: str, units: float, stream):
        """With kernel_timing enabled, bracket one hot-kernel launch with CUDA events on its stream."""
        if self.kernel_timing is None:
            return None
        a = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        return name, units, a

    def _ktimer_end(self, kt, stream) -> None:
        if kt is not None:
            e = torch.cuda.Event(enable_timing=True)
            e.record(stream)
            self.kernel_timing.append((kt[0], kt[1], kt[2], e))

    def kernel_stats(self) -> dict:
        """{name: (launches, mean seconds per launch, mean algorithmic units per launch)} of the timed launches
        (native executor: also "h2d", every host-to-device DMA with its bytes)."""
        if getattr(self, "_native", None) is not None and not self.kernel_timing:
            import ctypes

            res = {}
            for kind, name in ((0, "k1"), (1, "k2"), (2, "h2d")):
                n, t, u = ctypes.c_int(), ctypes.c_double(), ctypes.c_double()
                _lib.check(_lib.load().kvpr_decoder_kernel_stats(self._native, kind, ctypes.byref(n), ctypes.byref(t),
                                                                 ctypes.byref(u)), "kvpr_decoder_kernel_stats")
                if n.value:
                    res[name] = (n.value, t.value, u.value)
            if res:
                return res
        out = {}
        for name, units, a, e in self.kernel_timing or []:
            e.synchronize()
            n, t, u = out.get(name, (0, 0.0, 0.0))
            out[name] = (n + 1, t + a.elapsed_time(e) / 1e3, u + units)
        return {k: (n, t / n, u / n) for k, (n, t, u) in out.items()}

    def reset(self, length: int) -> None:
        """Rewind the logical cache length (positions >= length are overwritten by later steps)."""
        torch.cuda.synchronize(self.dev)
        self.len = length

    # ---------------------------------------------------------------- prefill
    def prefill(self, prompt: torch.Tensor) -> torch.Tensor:
        """Run the prompt [batch, S0] through all layers on the GPU, filling the host stores.

        Returns the first greedy token per sequence (device int32 [batch]).
        Not on the timed decode path; uses the same kernels as decode.
        """
        cfg, b, h = self.cfg, self.batch, self.cfg.hidden
        S0 = int(prompt.shape[1])
        if prompt.shape[0] != b or S0 <= 0 or S0 >= self.capacity:
            raise ValueError(f"prompt must be [batch={b}, 1 <= S0 < capacity={self.capacity}]")
        rows = S0 * b
        cs = self.cs
        with torch.cuda.stream(cs):
            toks = prompt.to(self.dev, non_blocking=True).to(torch.int32).t().contiguous()  # [S0, b] pos-major
            hbuf = torch.empty(rows, h, dtype=F32, device=self.dev)
            x = torch.empty(rows, h, dtype=F16, device=self.dev)
            q = torch.empty(rows, h, dtype=F16, device=self.dev)
            a = torch.empty(rows, h, dtype=F16, device=self.dev)
            mid = torch.empty(rows, cfg.ffn, dtype=F16, device=self.dev)
            pages = self.kv_dev[0]
            kernels.embed(toks.view(-1), self.w.embed, self.w.pos, hbuf, batch=b, pos_begin=0, stream=cs)
            for j, lw in enumerate(self.w.layers):
                kernels.layernorm(hbuf, lw.ln1_g, lw.ln1_b, x, eps=cfg.eps, stream=cs)
                self._qkv(x, rows, lw, q, pages[:S0], q_group=b * h, stream=cs)
                xs = self.x_store[j] if self.x_resident else self.stores.x[j]
                _copy(xs.data_ptr(), x.data_ptr(), rows * h * 2, cs)
                if self.kv_bits == 4:
                    kernels.kv4_quantize(pages, self.kvq_dev[0], b, 0, S0, stream=cs)
                    _copy(self.stores.kv[j].data_ptr(), self.kvq_dev[0].data_ptr(), S0 * self.qbytes, cs)
                else:
                    _copy(self.stores.kv[j].data_ptr(), pages.data_ptr(), S0 * 2 * b * h * 2, cs)
                kernels.prefill_attention(q, pages, a, b, cfg.heads, cfg.head_dim, S0, stream=cs)
                self._mlp(a, rows, lw, hbuf, x, mid, stream=cs)
            last = hbuf[(S0 - 1) * b:]
            self._head(last, stream=cs)
            first = self.tok.clone()
        cs.synchronize()
        self.len = S0
        return first

    # ------------------------------------------------------------ layer pieces
    def _qkv(self, x: torch.Tensor, M: int, lw, q_out: torch.Tensor, pages: torch.Tensor, q_group: int, stream):
        """q -> q_out ([M, h] row-major), k/v -> pages (position-major, row m = (pos m // b, seq m % b))."""
        b, h = self.batch, self.cfg.hidden
        bh = b * h
        kp = pages.data_ptr()
        epi = _lib.make_epilogue(
            [(q_out.data_ptr(), q_group), (kp, 2 * bh), (kp + bh * 2, 2 * bh)],
            seg_width=h, ld=h, row_group=b, bias=lw.bqkv.data_ptr(),
        )
        kernels.linear(x, lw.wqkv, epi, M=M, stream=stream)

    def _mlp(self, attn: torch.Tensor, M: int, lw, hres: torch.Tensor, ybuf: torch.Tensor, mid: torch.Tensor, stream):
        """h += attn W_o^T + b_o;  h += relu(LN2(h) W_1^T + b_1) W_2^T + b_2  (OPT pre-LN block)."""
        acc = _lib.EPI_F32 | _lib.EPI_ACCUM
        kernels.linear_simple(attn[:M], lw.wo, lw.bo, hres[:M], flags=acc, stream=stream, ws=self.ws)
        self._ffn(M, lw, hres, ybuf, mid, stream)

    def _ffn(self, M: int, lw, hres: torch.Tensor, ybuf: torch.Tensor, mid: torch.Tensor, stream):
        cfg = self.cfg
        acc = _lib.EPI_F32 | _lib.EPI_ACCUM
        kernels.layernorm_linear(hres, lw.ln2_g, lw.ln2_b, ybuf, lw.w1, lw.b1, mid, rows=M, eps=cfg.eps,
                                 flags=_lib.EPI_RELU, stream=stream, ws=self.ws)
        kernels.linear_simple(mid[:M], lw.w2, lw.b2, hres[:M], flags=acc, stream=stream, ws=self.ws)

    def _head(self, hrows: torch.Tensor, stream, ln: bool = True) -> None:
        """Final LN (unless the fused layer tail already wrote it into zf), tied LM head (fp32 logits) and
        greedy argmax into self.tok."""
        cfg = self.cfg
        if ln:
            kernels.layernorm(hrows, self.w.lnf_g, self.w.lnf_b, self.zf, eps=cfg.eps, stream=stream)
        kernels.linear_simple(self.zf, self.w.embed, None, self.logits, stream=stream, ws=self.ws)
        kernels.argmax(self.logits, self.tok, stream=stream)

    # ------------------------------------------------------------------ decode
    def _unit(self, u: int, base_len: int, splits: list[int]):
        L = self.cfg.layers
        i, j = divmod(u, L)
        s = base_len + i + 1
        lp = min(splits[i], s - 1)
        return i, j, s, lp, u % self.nbuf, u % self._R

    def _issue_h2d(self, u: int, base_len: int, splits: list[int]) -> None:
        """load_activation_recompute then load_cache for unit u (graph.py:266-293), on the copy stream."""
        L, b, h = self.cfg.layers, self.batch, self.cfg.hidden
        i, j, s, lp, buf, r = self._unit(u, base_len, splits)
        hs = self.hs
        if u >= self.nbuf:  # device buffer free: its previous user finished computing and storing
            rp = (u - self.nbuf) % self._R
            hs.wait_event(self.ev_done[rp])
            hs.wait_event(self.ev_d2h[rp])
        if u >= L:  # host store of the previous step's new position has landed (graph.py:286-287)
            hs.wait_event(self.ev_d2h[(u - L) % self._R])
        xh, kvh = self.stores.x[j], self.stores.kv[j]
        xd, kvd = self.x_dev[buf], self.kv_dev[buf]
        row = b * h * 2
        tr = self._trace
        kv_dma = s - 1 > lp and not (self.zc_read and tr is None)  # zero-copy: the tail reads it from the host
        kv_copy = ((self.kvq_dev[buf][lp] if self.kv_bits == 4 else kvd[lp]).data_ptr(), kvh[lp].data_ptr(),
                   (s - 1 - lp) * self.page_bytes) if kv_dma else None
        chunks = chunk_bounds(0 if self.x_resident else lp, self.chunks, self.chunk_rows, self.chunk_wave)
        if len(chunks) == 1 and tr is None:  # one X chunk: X and the KV tail in one C call (executor.cu)
            (p0, p1), = chunks
            _copy_batch([(xd[p0].data_ptr(), xh[p0].data_ptr(), (p1 - p0) * row)] + ([kv_copy] if kv_copy else []), hs)
            self.ev_x[r][0].record(hs)
            self.ev_kv[r].record(hs)
            return
        for c, (p0, p1) in enumerate(chunks):
            sp = tr.begin(hs, "load_activation_recompute", i + 1, j + 1, f"c{c}") if tr else None
            _copy(xd[p0].data_ptr(), xh[p0].data_ptr(), (p1 - p0) * row, hs)
            if sp:
                tr.end(hs, sp)
            self.ev_x[r][c].record(hs)
        if kv_copy:
            sp = tr.begin(hs, "load_cache", i + 1, j + 1) if tr else None
            _copy(*kv_copy, hs)
            if sp:
                tr.end(hs, sp)
        self.ev_kv[r].record(hs)

    def _compute_layer(self, u: int, base_len: int, splits: list[int]) -> None:
        cfg, b, h = self.cfg, self.batch, self.cfg.hidden
        i, j, s, lp, buf, r = self._unit(u, base_len, splits)
        lw = self.w.layers[j]
        cs, ds = self.cs, self.ds
        xd = self.x_store[j] if self.x_resident else self.x_dev[buf]
        kvd = self.kv_dev[buf]
        x_slot, page = xd[s - 1], kvd[s - 1]
        tr = self._trace
        I, J = i + 1, j + 1
        if u >= self.nbuf:  # the previous user's D2H has read this buffer's slot s'-1 / staging page
            cs.wait_event(self.ev_d2h[(u - self.nbuf) % self._R])
        # new token: X = LN1(h) straight into the X slot of position s'-1, q/k/v with k,v into page s'-1
        fused = self.fused_tail and tr is None
        sp = tr.begin(cs, "compute_mha", I, J, "proj") if tr else None
        if not fused or j == 0:  # fused: the previous layer's tail made LN1 into this slot and q, k, v
            kernels.layernorm(self.hres, lw.ln1_g, lw.ln1_b, x_slot, eps=cfg.eps, stream=cs)
            self._qkv(x_slot, b, lw, self.q, page, q_group=0, stream=cs)
        if self.kv_bits == 4:  # the stored copy of the new page is compressed; K2 reads the exact fp16 page
            kernels.kv4_quantize(kvd[s - 1:s], self.qnew[buf:buf + 1], b, 0, 1, stream=cs)
        if sp:
            tr.end(cs, sp)
        self.ev_qkv[r].record(cs)
        if fused and j > 0 and self.zc_write:  # the previous tail wrote this unit's X row and k, v page to the host
            self.ev_d2h[r].record(cs)
        else:
            # store_activation / store_cache (graph.py:340-347) on the D2H engine
            ds.wait_event(self.ev_qkv[r])
            src = self.qnew[buf] if self.kv_bits == 4 else page
            if tr is None:  # two DMAs in one C call (executor.cu); the row schedule's X row already sits in the store
                _copy_batch([(self.stores.kv[j][s - 1].data_ptr(), src.data_ptr(), self.page_bytes)] +
                            ([] if self.x_resident else [(self.stores.x[j][s - 1].data_ptr(), x_slot.data_ptr(),
                                                          b * h * 2)]), ds)
            else:
                if not self.x_resident:
                    sp = tr.begin(ds, "store_activation", I, J)
                    _copy(self.stores.x[j][s - 1].data_ptr(), x_slot.data_ptr(), b * h * 2, ds)
                    tr.end(ds, sp)
                sp = tr.begin(ds, "store_cache", I, J)
                _copy(self.stores.kv[j][s - 1].data_ptr(), src.data_ptr(), self.page_bytes, ds)
                tr.end(ds, sp)
            self.ev_d2h[r].record(ds)
        # K1: rebuild K,V[0:l) chunk by chunk as X lands (one launch when X is resident)
        for c, (p0, p1) in enumerate(chunk_bounds(lp, 1 if self.x_resident else self.chunks, self.chunk_rows,
                                                  0 if self.x_resident else self.chunk_wave)):
            if not self.x_resident:
                cs.wait_event(self.ev_x[r][c])
            sp = tr.begin(cs, "compute_recompute", I, J, f"c{c}") if tr else None
            kt = self._ktimer("k1", 4 * b * (p1 - p0) * h * h, cs)
            kernels.recompute_kv(xd, lw.w_kv, lw.b_kv, kvd, b, p0, p1, stream=cs)
            self._ktimer_end(kt, cs)
            if sp:
                tr.end(cs, sp)
        cs.wait_event(self.ev_kv[r])
        if fused:  # same launch and waits as executor.cu fused_tail()
            qkv = None
            if j + 1 < cfg.layers:
                nxt = self.w.layers[j + 1]
                nb = (u + 1) % self.nbuf
                xn = self.x_store[j + 1] if self.x_resident else self.x_dev[nb]
                if u + 1 >= self.nbuf:  # the next unit's X slot / page: its previous reader's D2H is done
                    cs.wait_event(self.ev_d2h[(u + 1 - self.nbuf) % self._R])
                lnx = (nxt.ln1_g, nxt.ln1_b, xn[s - 1])
                qkv = (nxt.wqkv, nxt.bqkv, self.q, self.kv_dev[nb][s - 1])
                stores = (None if self.x_resident else self.stores.x[j + 1][s - 1],
                          self.stores.kv[j + 1][s - 1]) if self.zc_write else None
            else:
                lnx, stores = (self.w.lnf_g, self.w.lnf_b, self.zf), None
            host_kv = None
            if s - 1 > lp and self.zc_read:  # KV[l:s'-1] from the host store; its last position stored by unit u - L
                if u >= cfg.layers:
                    cs.wait_event(self.ev_d2h[(u - cfg.layers) % self._R])
                host_kv = (self.stores.kv[j], lp, s - 1)
            kt = self._ktimer("k2", 2 * b * s * h * 2, cs)
            kernels.layer_tail(self.q, kvd, s, lw, self.hres, self.attn, self.mid, self.ws, cfg.heads, cfg.eps,
                               lnx=lnx, qkv_next=qkv, host_kv=host_kv, stores=stores, stream=cs)
            self._ktimer_end(kt, cs)
            self.ev_done[r].record(cs)
            return
        # K2 over the merged pages [0, s') in place (4-bit tail [lp, s'-1) dequantised inside K2), then W_O
        sp = tr.begin(cs, "compute_mha", I, J, "attn") if tr else None
        if self.kv_bits == 4 and s - 1 > lp:
            kt = self._ktimer("k2", 2 * b * (lp + 1) * h * 2 + (s - 1 - lp) * self.qbytes, cs)
            kernels.decode_attention_kv4(self.q, kvd, self.kvq_dev[buf], lp, s - 1, self.attn, self.ws, b,
                                         cfg.heads, cfg.head_dim, s, stream=cs)
        else:
            kt = self._ktimer("k2", 2 * b * s * h * 2, cs)
            kernels.decode_attention(self.q, kvd, self.attn, self.ws, b, cfg.heads, cfg.head_dim, s, stream=cs)
        self._ktimer_end(kt, cs)
        acc = _lib.EPI_F32 | _lib.EPI_ACCUM
        kernels.linear_simple(self.attn, lw.wo, lw.bo, self.hres, flags=acc, stream=cs, ws=self.ws)
        if sp:
            tr.end(cs, sp)
        sp = tr.begin(cs, "compute_ffn", I, J) if tr else None
        self._ffn(b, lw, self.hres, self.y, self.mid, stream=cs)
        if sp:
            tr.end(cs, sp)
        self.ev_done[r].record(cs)

    # ------------------------------------------------------- native executor
    def _native_handle(self):
        """Descriptor of this runtime's buffers for the C executor (csrc/executor.cu), built once."""
        if getattr(self, "_native", None) is not None:
            return self._native
        import ctypes

        cfg, ptr = self.cfg, (lambda t: t.data_ptr() if t is not None else None)  # noqa: E731
        layers = (_lib.LayerDesc * cfg.layers)()
        for j, lw in enumerate(self.w.layers):
            L = layers[j]
            for name in ("ln1_g", "ln1_b", "wqkv", "bqkv", "wo", "bo", "ln2_g", "ln2_b", "w1", "b1", "w2", "b2"):
                setattr(L, name, getattr(lw, name).data_ptr())
            L.host_x = self.stores.x[j].data_ptr() if not self.x_resident else None
            L.host_kv = self.stores.kv[j].data_ptr()
            L.dev_x = self.x_store[j].data_ptr() if self.x_resident else None
        d = _lib.DecoderDesc()
        d.layers, d.batch, d.hidden, d.heads, d.ffn = cfg.layers, self.batch, cfg.hidden, cfg.heads, cfg.ffn
        d.vocab, d.capacity, d.chunks, d.nbuf, d.x_resident = cfg.vocab, self.capacity, self.chunks, self.nbuf, int(
            self.x_resident)
        d.eps = cfg.eps
        d.embed, d.pos, d.lnf_g, d.lnf_b = ptr(self.w.embed), ptr(self.w.pos), ptr(self.w.lnf_g), ptr(self.w.lnf_b)
        d.kv_dev, d.x_dev, d.hres = ptr(self.kv_dev), ptr(self.x_dev), ptr(self.hres)
        d.q, d.attn, d.y, d.mid, d.zf = ptr(self.q), ptr(self.attn), ptr(self.y), ptr(self.mid), ptr(self.zf)
        d.logits, d.tok, d.ws, d.ws_bytes = ptr(self.logits), ptr(self.tok), ptr(self.ws), self.ws.numel()
        d.compute_stream, d.h2d_stream, d.d2h_stream = self.cs.cuda_stream, self.hs.cuda_stream, self.ds.cuda_stream
        d.chunk_rows = self.chunk_rows
        d.chunk_wave = self.chunk_wave
        d.recompute_stream = self.rs.cuda_stream if self.k1_stream else None
        d.fused_tail = int(self.fused_tail)
        d.zero_copy = int(self.zc_read) | (int(self.zc_write) << 1)
        d.dma_group = self.dma_group
        h = ctypes.c_void_p()
        _lib.check(_lib.load().kvpr_decoder_create(ctypes.byref(d), layers, ctypes.byref(h)), "kvpr_decoder_create")
        self._native_keep = (d, layers)
        self._native = h
        return h

    def _decode_native(self, splits: list[int], out_tokens: torch.Tensor, logits: torch.Tensor | None,
                       timing: DecodeTiming | None = None) -> None:
        import ctypes

        arr = (ctypes.c_int * len(splits))(*splits)
        lib, h = _lib.load(), self._native_handle()
        timed = self.kernel_timing is not None or timing is not None
        _lib.check(lib.kvpr_decoder_set_timing(h, int(timed)), "kvpr_decoder_set_timing")
        _lib.check(lib.kvpr_decoder_run(h, self.len, arr, len(splits), out_tokens.data_ptr(),
                                        logits.data_ptr() if logits is not None else None), "kvpr_decoder_run")
        if timing is not None:
            L, n = self.cfg.layers, len(splits)
            lay, stp = (ctypes.c_float * (n * L))(), (ctypes.c_float * n)()
            got = lib.kvpr_decoder_timeline(h, lay, n * L, stp, n)
            if got < 0:
                _lib.check(-got, "kvpr_decoder_timeline")
            timing.step_ms.extend(stp[:got])
            timing.layer_ms.extend([list(lay[i * L:(i + 1) * L]) for i in range(got)])

    def decode(self, splits: list[int], tokens: torch.Tensor | None = None, keep_logits: bool = False,
               timing: DecodeTiming | None = None, out_tokens: torch.Tensor | None = None,
               trace=None, native: bool | None = None) -> torch.Tensor:
        """Enqueue len(splits) decode steps (no host sync); returns device int32 [steps, batch] tokens.

        Step i attends over s' = len + i + 1 positions, rebuilding [0, min(l_i, s'-1)) with K1.
        """
        cfg, b, L = self.cfg, self.batch, self.cfg.layers
        steps = len(splits)
        base = self.len
        if base + steps > self.capacity:
            raise ValueError(f"cache capacity {self.capacity} exceeded ({base} + {steps} steps)")
        for i, l in enumerate(splits):
            if not 0 <= l <= base + i + 1:
                raise ValueError(f"step {i + 1}: split {l} out of range [0, {base + i + 1}]")
        cs = self.cs
        self._trace = trace
        if out_tokens is None:
            out_tokens = torch.empty(steps, b, dtype=torch.int32, device=self.dev)
        logits = torch.empty(steps, b, cfg.vocab, dtype=F32, device=self.dev) if keep_logits else None
        # everything the caller enqueued (e.g. the H2D of `tokens`) precedes this run on both engines
        cs.wait_stream(torch.cuda.current_stream(self.dev))
        self.hs.wait_stream(torch.cuda.current_stream(self.dev))
        if tokens is not None:
            with torch.cuda.stream(cs):
                self.tok.copy_(tokens.to(torch.int32), non_blocking=True)
        if native is None:  # the C executor covers the plain path (timed or not); tracing / 4-bit KV stay in Python
            native = trace is None and self.kv_bits is None
        n0 = _lib.load().kvpr_kernel_launches()
        if native:
            self._decode_native(splits, out_tokens, logits, timing)
            self.launches += _lib.load().kvpr_kernel_launches() - n0
            self.len = base + steps
            cur = torch.cuda.current_stream(self.dev)
            cur.wait_stream(cs)
            cur.wait_stream(self.ds)
            self._last_logits = logits
            return out_tokens
        n_units = steps * L
        t_start = torch.cuda.Event(enable_timing=True) if timing is not None else None
        step_marks, layer_marks = [], []
        if t_start is not None:
            t_start.record(cs)
        self._issue_h2d(0, base, splits)
        # unit u+1's loads are issued ahead of unit u's compute, except with a single layer, where they
        # wait on unit u's own D2H of the new position (graph.py:286-287), recorded by that compute
        ahead = L > 1
        for u in range(n_units):
            if ahead and u + 1 < n_units:
                self._issue_h2d(u + 1, base, splits)
            i, j = divmod(u, L)
            if j == 0:
                kernels.embed(self.tok, self.w.embed, self.w.pos, self.hres, batch=b, pos_begin=base + i, stream=cs)
            self._compute_layer(u, base, splits)
            if timing is not None:
                e = torch.cuda.Event(enable_timing=True)
                e.record(cs)
                layer_marks.append(e)
            if j == L - 1:
                self._head(self.hres, stream=cs, ln=not (self.fused_tail and trace is None))
                with torch.cuda.stream(cs):
                    out_tokens[i].copy_(self.tok, non_blocking=True)
                    if logits is not None:
                        logits[i].copy_(self.logits, non_blocking=True)
                if timing is not None:
                    e = torch.cuda.Event(enable_timing=True)
                    e.record(cs)
                    step_marks.append(e)
            if not ahead and u + 1 < n_units:
                self._issue_h2d(u + 1, base, splits)
        self.len = base + steps
        self._trace = None
        cur = torch.cuda.current_stream(self.dev)
        cur.wait_stream(cs)
        cur.wait_stream(self.ds)
        if timing is not None:
            cs.synchronize()
            prev = t_start
            for e in step_marks:
                timing.step_ms.append(prev.elapsed_time(e))
                prev = e
            prev = t_start
            for i in range(steps):
                row = []
                for e in layer_marks[i * L:(i + 1) * L]:
                    row.append(prev.elapsed_time(e))
                    prev = e
                timing.layer_ms.append(row)
                prev = step_marks[i]
        self.launches += _lib.load().kvpr_kernel_launches() - n0
        self._last_logits = logits
        return out_tokens

    @property
    def last_logits(self) -> torch.Tensor | None:
        return getattr(self, "_last_logits", None)

    def close(self) -> None:
        if getattr(self, "_native", None) is not None:
            _lib.load().kvpr_decoder_destroy(self._native)
            self._native = None
        self.stores.close()


def generate(weights: OPTWeights, prompt: torch.Tensor, splits: list[int], runtime: KVPRRuntime | None = None,
             keep_logits: bool = False):
    """End-to-end public call: host prompt ids in, host generated ids out.

    Returns (tokens int64 [steps + 1, batch] on the host — the prefill token then
    one per decode step — and the runtime).
    """
    b, S0 = prompt.shape
    rt = runtime or KVPRRuntime(weights, b, S0 + len(splits) + 1)
    first = rt.prefill(prompt)
    toks = rt.decode(splits, tokens=first, keep_logits=keep_logits)
    host = torch.empty(len(splits) + 1, b, dtype=torch.int32, pin_memory=True)
    with torch.cuda.stream(rt.cs):
        host[0].copy_(first, non_blocking=True)
        host[1:].copy_(toks, non_blocking=True)
    rt.cs.synchronize()
    return host.to(torch.int64), rt
