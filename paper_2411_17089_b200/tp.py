"""Head-sharded tensor parallelism for KVPR decode (BASELINE config 4:
OPT-30B b64 prompt 2048 on 8 B200s).

One process per GPU.  Rank r of G owns heads [r*H/G, (r+1)*H/G):
  * q/k/v and fc1 are column-parallel, out-proj and fc2 row-parallel; the two
    partial sums per layer are combined with an NCCL all-reduce (sum) over
    NVLink.  Rank 0 accumulates its partial onto the residual and adds the
    bias, the other ranks write their bare partial into the residual buffer,
    so one in-place all-reduce yields residual + sum of partials with no
    extra kernel.
  * the KV host store and device pages hold only the local heads
    ([pos][2][b][h/G]) -> per-GPU PCIe KV bytes scale 1/G;
  * layer inputs X are full width (every rank's K1 needs all of X[:, :l]),
    so the X store is split block-cyclically over positions (blocks of
    `block` positions, block k owned by rank k % G).  Each rank ships only
    its blocks over its own PCIe link; an all-gather over NVLink per round
    of G blocks assembles X in natural position order, and K1 runs on each
    round as soon as it is gathered.  Per-GPU H2D bytes = (X + KV)/G, so at
    zero latency the split l of the unsharded problem is also optimal per
    GPU (the ratio in scheduler.py:111-112 is invariant) and every rank runs
    the same plan (rank 0's, broadcast).
The X all-gathers and the residual all-reduces use separate communicators so
the prefetch of layer u+1 never queues the all-reduce of layer u behind it.

`TPLayout` and `shard_layer` are pure host logic (covered by gloo tests on
CPU); `TPRuntime` drives the same libkvpr kernels as the 1-GPU runtime.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import _lib, kernels
from .hostmem import pinned_empty, unpin
from .runtime import F16, F32, _copy
from .weights import LayerWeights, OPTWeights


@dataclass(frozen=True)
class TPLayout:
    world: int
    rank: int
    hidden: int
    heads: int
    ffn: int
    block: int = 64

    def __post_init__(self):
        if self.world <= 0 or not 0 <= self.rank < self.world:
            raise ValueError(f"bad rank {self.rank} of {self.world}")
        if self.heads % self.world or self.ffn % self.world:
            raise ValueError(f"heads ({self.heads}) and ffn ({self.ffn}) must divide by world ({self.world})")
        if self.block <= 0:
            raise ValueError("block must be positive")

    @property
    def head_dim(self) -> int:
        return self.hidden // self.heads

    @property
    def heads_local(self) -> int:
        return self.heads // self.world

    @property
    def hs(self) -> int:
        """Local slice of the hidden (head) dimension."""
        return self.heads_local * self.head_dim

    @property
    def fs(self) -> int:
        return self.ffn // self.world

    @property
    def round_len(self) -> int:
        return self.world * self.block

    def owner(self, pos: int) -> int:
        return (pos // self.block) % self.world

    def rounds(self, n: int) -> list[tuple[int, int, int]]:
        """(t, p0, p1): round t covers positions [t*G*B, (t+1)*G*B) clipped to [0, n)."""
        R = self.round_len
        return [(t, t * R, min((t + 1) * R, n)) for t in range((n + R - 1) // R)]

    def my_block(self, t: int, n: int) -> tuple[int, int]:
        """This rank's positions in round t, clipped to [0, n) (may be empty)."""
        p0 = (t * self.world + self.rank) * self.block
        return min(p0, n), min(p0 + self.block, n)

    def compact_index(self, pos: int) -> int:
        """Row of `pos` in this rank's compact X store (pos must be owned by this rank)."""
        if self.owner(pos) != self.rank:
            raise ValueError(f"position {pos} is owned by rank {self.owner(pos)}, not {self.rank}")
        return (pos // self.round_len) * self.block + pos % self.block

    def compact_capacity(self, capacity: int) -> int:
        return ((capacity + self.round_len - 1) // self.round_len) * self.block

    def owned_runs(self, n: int) -> list[tuple[int, int]]:
        """Maximal runs [p0, p1) of positions < n owned by this rank (one per block)."""
        out = []
        for t, _, _ in self.rounds(n):
            q0, q1 = self.my_block(t, n)
            if q1 > q0:
                out.append((q0, q1))
        return out


def shard_layer(lw: LayerWeights, lay: TPLayout) -> LayerWeights:
    """Rank-local weights: column-parallel q/k/v, fc1; row-parallel out-proj, fc2 (bias on rank 0 only)."""
    h, hs, fs, r = lay.hidden, lay.hs, lay.fs, lay.rank
    cols = slice(r * hs, (r + 1) * hs)
    fcols = slice(r * fs, (r + 1) * fs)
    q, k, v = lw.wqkv[:h], lw.wqkv[h:2 * h], lw.wqkv[2 * h:]
    bq, bk, bv = lw.bqkv[:h], lw.bqkv[h:2 * h], lw.bqkv[2 * h:]
    zero_or = (lambda t: t.clone()) if r == 0 else (lambda t: torch.zeros_like(t))  # noqa: E731
    return LayerWeights(
        ln1_g=lw.ln1_g.clone(), ln1_b=lw.ln1_b.clone(),
        wqkv=torch.cat([q[cols], k[cols], v[cols]]).contiguous(),
        bqkv=torch.cat([bq[cols], bk[cols], bv[cols]]).contiguous(),
        wo=lw.wo[:, cols].contiguous(), bo=zero_or(lw.bo),
        ln2_g=lw.ln2_g.clone(), ln2_b=lw.ln2_b.clone(),
        w1=lw.w1[fcols].contiguous(), b1=lw.b1[fcols].contiguous(),
        w2=lw.w2[:, fcols].contiguous(), b2=zero_or(lw.b2),
    )


class _CudaArray:
    """__cuda_array_interface__ view of raw device memory (torch.as_tensor wraps it without a copy)."""

    def __init__(self, ptr: int, shape: tuple, typestr: str):
        self.__cuda_array_interface__ = {"shape": shape, "typestr": typestr, "data": (ptr, False), "version": 3,
                                         "strides": None}


class PeerBuffers:
    """Symmetric peer memory for the fused TP all-reduce (csrc/tpcomm.cu, kvpr_linear_allreduce).

    Every rank allocates one CUDA IPC region [receive slots world x M x N fp32 | residual M x N fp32 |
    flags | error word], the handles are all-gathered over the process group, and every rank opens
    its peers' regions (NVLink P2P between GPUs; also valid for ranks sharing one GPU).  `resid` is
    this rank's residual as a torch tensor: the decode keeps its residual stream there, so the owners'
    broadcasts land in place.
    """

    def __init__(self, M: int, N: int, group=None, device: torch.device | None = None):
        import ctypes

        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if not 2 <= self.world <= _lib.TP_MAX_WORLD:
            raise ValueError(f"fused all-reduce needs 2..{_lib.TP_MAX_WORLD} ranks, got {self.world}")
        if M > 64 or -(-N // 128) > _lib.TP_MAX_TILES:
            raise ValueError(f"fused all-reduce: M={M} > 64 or N={N} beyond {_lib.TP_MAX_TILES} tiles")
        self.M, self.N = M, N
        lib = _lib.load()
        al = lambda x: -(-x // 256) * 256  # noqa: E731
        self.off_recv = 0
        self.off_resid = al(self.world * M * N * 4)
        self.off_flags = self.off_resid + al(M * N * 4)
        self.off_err = self.off_flags + al((_lib.TP_MAX_WORLD + 1) * _lib.TP_MAX_TILES * 4)
        total = self.off_err + 256
        hb = lib.kvpr_ipc_handle_bytes()
        handle = (ctypes.c_char * hb)()
        base = ctypes.c_void_p()
        _lib.check(lib.kvpr_ipc_alloc(total, ctypes.byref(base), handle), "kvpr_ipc_alloc")
        self._own = base.value
        handles = [None] * self.world
        dist.all_gather_object(handles, bytes(handle), group=group)
        self._opened = []
        bases = []
        for r, hnd in enumerate(handles):
            if r == self.rank:
                bases.append(self._own)
                continue
            p = ctypes.c_void_p()
            buf = (ctypes.c_char * hb).from_buffer_copy(hnd)
            _lib.check(lib.kvpr_ipc_open(buf, ctypes.byref(p)), "kvpr_ipc_open")
            self._opened.append(p.value)
            bases.append(p.value)
        pe = _lib.TpPeers()
        pe.rank, pe.world = self.rank, self.world
        for r, bp in enumerate(bases):
            pe.recv[r] = bp + self.off_recv
            pe.resid[r] = bp + self.off_resid
            pe.flags[r] = bp + self.off_flags
        pe.err = self._own + self.off_err
        self.peers = pe
        self.resid = torch.as_tensor(_CudaArray(self._own + self.off_resid, (M, N), "<f4"), device=device)
        self._err = torch.as_tensor(_CudaArray(self._own + self.off_err, (1,), "<u4"), device=device)
        self.epoch = 0
        dist.barrier(group=group)

    def linear_allreduce(self, a: torch.Tensor, w: torch.Tensor, bias: torch.Tensor | None, M: int, stream) -> None:
        """resid += sum over ranks of a_r[:M] . w_r^T + bias, on every rank (all ranks call it in lockstep)."""
        import ctypes

        self.epoch += 1
        N, K = w.shape
        _lib.check(_lib.load().kvpr_linear_allreduce(
            a.data_ptr(), a.stride(0), w.data_ptr(), w.stride(0), M, N, K,
            bias.data_ptr() if bias is not None else None, ctypes.byref(self.peers), self.epoch & 0xFFFFFFFF,
            stream.cuda_stream), "kvpr_linear_allreduce")

    def error(self) -> int:
        """Nonzero once a peer wait timed out (the fused all-reduce then produced garbage)."""
        return int(self._err.to(torch.int64).item())

    def close(self, group=None) -> None:
        """Unmap the peers' regions, wait for every rank to do the same, then free this rank's."""
        lib = _lib.load()
        torch.cuda.synchronize()
        for p in self._opened:
            lib.kvpr_ipc_close(p)
        self._opened = []
        if dist.is_initialized():
            dist.barrier(group=group)
        if self._own:
            lib.kvpr_ipc_free(self._own)
            self._own = None


class TPRuntime:
    """One rank of the head-sharded decoder.  `weights` are the full (unsharded) weights on this GPU."""

    def __init__(self, weights: OPTWeights, batch: int, capacity: int, group=None, block: int = 64,
                 device: torch.device | None = None, fused: bool | None = None):
        """fused (default: world > 1 and batch <= 64): the decode's row-parallel projections end in the
        fused peer-memory all-reduce (PeerBuffers / csrc/tpcomm.cu) instead of a collective call."""
        cfg = weights.cfg
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.lay = TPLayout(self.world, self.rank, cfg.hidden, cfg.heads, cfg.ffn, block)
        self.cfg, self.batch = cfg, batch
        self.dev = device or weights.embed.device
        lay = self.lay
        R = lay.round_len
        self.capacity = capacity
        cap_x = ((capacity + R - 1) // R) * R  # gathered rounds may run past the capacity
        self.layers = [shard_layer(lw, lay) for lw in weights.layers]
        # the fused all-reduce adds the bias once, at the owner, so every rank keeps the full biases
        self.bias_full = [(lw.bo, lw.b2) for lw in weights.layers]
        self.embed, self.pos, self.lnf_g, self.lnf_b = weights.embed, weights.pos, weights.lnf_g, weights.lnf_b
        self.group = group
        if self.world > 1:
            ranks = list(range(self.world))
            self.g_x = dist.new_group(ranks)   # X all-gathers
            self.g_h = dist.new_group(ranks)   # residual all-reduces
        else:
            self.g_x = self.g_h = None
        _lib.load()
        h, b, hs, fs = cfg.hidden, batch, lay.hs, lay.fs
        self.cs = torch.cuda.Stream(self.dev, priority=-1)
        self.hs_ = torch.cuda.Stream(self.dev)
        self.ds = torch.cuda.Stream(self.dev)
        self.comm = torch.cuda.Stream(self.dev)
        # host stores: compact X (owned blocks only) and local-head KV
        self.store_x = pinned_empty((cfg.layers, lay.compact_capacity(capacity), b, h), F16)
        self.store_kv = pinned_empty((cfg.layers, capacity, 2, b, hs), F16)
        z = lambda *s, dt=F16: torch.empty(*s, dtype=dt, device=self.dev)  # noqa: E731
        self.nbuf = 2
        self.kv_dev = z(2, capacity, 2, b, hs)
        self.x_dev = z(2, cap_x, b, h)
        self.x_new = z(2, b, h)
        self.fused = (self.world > 1 and b <= 64) if fused is None else bool(fused and self.world > 1)
        self.peer = PeerBuffers(b, h, group=group, device=self.dev) if self.fused else None
        self.hres = self.peer.resid if self.fused else z(b, h, dt=F32)
        self.q, self.attn = z(b, hs), z(b, hs)
        self.y, self.mid, self.zf = z(b, h), z(b, fs), z(b, h)
        self.logits = z(b, cfg.vocab, dt=F32)
        self.tok = z(b, dt=torch.int32)
        self.ws = z(16 << 20, dt=torch.uint8)
        self.len = 0
        self._works = {}
        self.launches = 0

    # ---------------------------------------------------------------- helpers
    def _allreduce_h(self, rows: torch.Tensor) -> None:
        if self.world > 1:
            with torch.cuda.stream(self.cs):
                dist.all_reduce(rows, op=dist.ReduceOp.SUM, group=self.g_h)

    def _rowpar(self, a, w, bias, out, M):
        """Row-parallel projection into the residual: rank 0 accumulates (+bias), others overwrite; then all-reduce."""
        flags = _lib.EPI_F32 | (_lib.EPI_ACCUM if self.rank == 0 else 0)
        kernels.linear_simple(a[:M], w, bias if self.rank == 0 else None, out[:M], flags=flags, stream=self.cs,
                              ws=self.ws)
        self._allreduce_h(out[:M])

    def _qkv(self, x, M, lw, q_out, pages, stream):
        b, hs = self.batch, self.lay.hs
        kp = pages.data_ptr()
        epi = _lib.make_epilogue([(q_out.data_ptr(), b * hs), (kp, 2 * b * hs), (kp + b * hs * 2, 2 * b * hs)],
                                 seg_width=hs, ld=hs, row_group=b, bias=lw.bqkv.data_ptr())
        kernels.linear(x, lw.wqkv, epi, M=M, stream=stream)

    def _k1(self, xd, lw, kvd, p0, p1, stream):
        """K1 for the local heads: pages[p] = X[p] . W_kv_local^T + b (positions [p0, p1))."""
        b, hs = self.batch, self.lay.hs
        if p1 <= p0:
            return
        page0 = kvd[p0].data_ptr()
        epi = _lib.make_epilogue([(page0, 2 * b * hs), (page0 + b * hs * 2, 2 * b * hs)], seg_width=hs, ld=hs,
                                 row_group=b, bias=lw.bqkv[hs:].data_ptr())
        kernels.linear(xd[p0], lw.wqkv[hs:], epi, M=(p1 - p0) * b, stream=stream)

    # ---------------------------------------------------------------- prefill
    def prefill(self, prompt: torch.Tensor) -> torch.Tensor:
        cfg, b, h, lay = self.cfg, self.batch, self.cfg.hidden, self.lay
        S0 = int(prompt.shape[1])
        rows = S0 * b
        cs = self.cs
        with torch.cuda.stream(cs):
            toks = prompt.to(self.dev).to(torch.int32).t().contiguous()
            hbuf = torch.empty(rows, h, dtype=F32, device=self.dev)
            x = torch.empty(rows, h, dtype=F16, device=self.dev)
            q = torch.empty(rows, lay.hs, dtype=F16, device=self.dev)
            a = torch.empty(rows, lay.hs, dtype=F16, device=self.dev)
            mid = torch.empty(rows, lay.fs, dtype=F16, device=self.dev)
            pages = self.kv_dev[0]
            kernels.embed(toks.view(-1), self.embed, self.pos, hbuf, batch=b, pos_begin=0, stream=cs)
            for j, lw in enumerate(self.layers):
                kernels.layernorm(hbuf, lw.ln1_g, lw.ln1_b, x, eps=cfg.eps, stream=cs)
                for p0, p1 in lay.owned_runs(S0):
                    dst = self.store_x[j][lay.compact_index(p0)]
                    _copy(dst.data_ptr(), x[p0 * b].data_ptr(), (p1 - p0) * b * h * 2, cs)
                self._qkv(x, rows, lw, q, pages, cs)
                _copy(self.store_kv[j].data_ptr(), pages.data_ptr(), S0 * 2 * b * lay.hs * 2, cs)
                kernels.prefill_attention(q, pages, a, b, lay.heads_local, lay.head_dim, S0, stream=cs)
                self._rowpar(a, lw.wo, lw.bo, hbuf, rows)
                kernels.layernorm(hbuf, lw.ln2_g, lw.ln2_b, x, eps=cfg.eps, stream=cs)
                kernels.linear_simple(x, lw.w1, lw.b1, mid, flags=_lib.EPI_RELU, stream=cs, ws=self.ws)
                self._rowpar(mid, lw.w2, lw.b2, hbuf, rows)
            self._head(hbuf[(S0 - 1) * b:])
        with torch.cuda.stream(cs):
            first = self.tok.clone()
        cs.synchronize()
        self.len = S0
        return first

    def _head(self, hrows):
        cs = self.cs
        kernels.layernorm(hrows, self.lnf_g, self.lnf_b, self.zf, eps=self.cfg.eps, stream=cs)
        kernels.linear_simple(self.zf, self.embed, None, self.logits, stream=cs, ws=self.ws)
        kernels.argmax(self.logits, self.tok, stream=cs)

    # ----------------------------------------------------------------- decode
    def _issue_loads(self, u, base, splits, ev):
        """H2D of this rank's X blocks + local KV tail on the copy stream; per-round X all-gather on comm."""
        cfg, b, h, lay = self.cfg, self.batch, self.cfg.hidden, self.lay
        L = cfg.layers
        i, j = divmod(u, L)
        s = base + i + 1
        lp = min(splits[i], s - 1)
        buf = u % 2
        hs_ = self.hs_
        if u >= 2:
            hs_.wait_event(ev["done"][u - 2])
            hs_.wait_event(ev["d2h"][u - 2])
        if u >= L:
            hs_.wait_event(ev["d2h"][u - L])
        xd, kvd = self.x_dev[buf], self.kv_dev[buf]
        rounds = lay.rounds(lp)
        xr, gw = [], []
        for t, r0, r1 in rounds:
            q0, q1 = lay.my_block(t, lp)
            if q1 > q0:
                src = self.store_x[j][lay.compact_index(q0)]
                _copy(xd[q0].data_ptr(), src.data_ptr(), (q1 - q0) * b * h * 2, hs_)
            e = torch.cuda.Event()
            e.record(hs_)
            xr.append(e)
        rowb = 2 * b * lay.hs * 2
        _copy(kvd[lp].data_ptr(), self.store_kv[j][lp].data_ptr(), (s - 1 - lp) * rowb, hs_)
        ekv = torch.cuda.Event()
        ekv.record(hs_)
        # NVLink all-gather of each round (natural position order) on the comm stream
        for (t, r0, r1), e in zip(rounds, xr):
            if self.world == 1:
                gw.append(e)
                continue
            self.comm.wait_event(e)
            blk = lay.block * b * h
            out = xd[t * lay.round_len: (t + 1) * lay.round_len].reshape(-1)
            inp = out[self.rank * blk:(self.rank + 1) * blk]
            with torch.cuda.stream(self.comm):
                gw.append(dist.all_gather_into_tensor(out, inp, group=self.g_x, async_op=True))
        self._works[u] = (rounds, gw, ekv)

    def _compute(self, u, base, splits, ev):
        cfg, b, h, lay = self.cfg, self.batch, self.cfg.hidden, self.lay
        i, j = divmod(u, cfg.layers)
        s = base + i + 1  # the rebuilt prefix length was fixed when the loads were issued (_works[u])
        buf = u % 2
        lw = self.layers[j]
        cs, ds = self.cs, self.ds
        xd, kvd, xn = self.x_dev[buf], self.kv_dev[buf], self.x_new[buf]
        page = kvd[s - 1]
        if u >= 2:  # the D2H of this buffer's previous user has read x_new / page
            cs.wait_event(ev["d2h"][u - 2])
        kernels.layernorm(self.hres, lw.ln1_g, lw.ln1_b, xn, eps=cfg.eps, stream=cs)
        self._qkv(xn, b, lw, self.q, page, cs)
        eq = torch.cuda.Event()
        eq.record(cs)
        ds.wait_event(eq)
        if lay.owner(s - 1) == self.rank:
            _copy(self.store_x[j][lay.compact_index(s - 1)].data_ptr(), xn.data_ptr(), b * h * 2, ds)
        _copy(self.store_kv[j][s - 1].data_ptr(), page.data_ptr(), 2 * b * lay.hs * 2, ds)
        ev["d2h"][u] = torch.cuda.Event()
        ev["d2h"][u].record(ds)
        rounds, gw, ekv = self._works.pop(u)
        for (t, r0, r1), w in zip(rounds, gw):
            if isinstance(w, torch.cuda.Event):
                cs.wait_event(w)
            else:
                with torch.cuda.stream(cs):
                    w.wait()
            self._k1(xd, lw, kvd, r0, r1, cs)
        cs.wait_event(ekv)
        kernels.decode_attention(self.q, kvd, self.attn, self.ws, b, lay.heads_local, lay.head_dim, s, stream=cs)
        bo, b2 = self.bias_full[j]
        if self.fused:
            self.peer.linear_allreduce(self.attn, lw.wo, bo, b, cs)
        else:
            self._rowpar(self.attn, lw.wo, lw.bo, self.hres, b)
        kernels.layernorm(self.hres, lw.ln2_g, lw.ln2_b, self.y, eps=cfg.eps, stream=cs)
        kernels.linear_simple(self.y, lw.w1, lw.b1, self.mid, flags=_lib.EPI_RELU, stream=cs, ws=self.ws)
        if self.fused:
            self.peer.linear_allreduce(self.mid, lw.w2, b2, b, cs)
        else:
            self._rowpar(self.mid, lw.w2, lw.b2, self.hres, b)
        ev["done"][u] = torch.cuda.Event()
        ev["done"][u].record(cs)

    def reset(self, length: int) -> None:
        torch.cuda.synchronize(self.dev)
        self.len = length

    def decode(self, splits: list[int], tokens: torch.Tensor | None = None, keep_logits: bool = False,
               timing=None):
        cfg, b, L = self.cfg, self.batch, self.cfg.layers
        steps, base = len(splits), self.len
        if base + steps > self.capacity:
            raise ValueError(f"cache capacity {self.capacity} exceeded ({base} + {steps} steps)")
        for i, l in enumerate(splits):
            if not 0 <= l <= base + i + 1:
                raise ValueError(f"step {i + 1}: split {l} out of range [0, {base + i + 1}]")
        cs = self.cs
        cs.wait_stream(torch.cuda.current_stream(self.dev))  # the caller's work (e.g. H2D of `tokens`) first
        self.hs_.wait_stream(torch.cuda.current_stream(self.dev))
        if tokens is not None:
            with torch.cuda.stream(cs):
                self.tok.copy_(tokens.to(torch.int32), non_blocking=True)
        out = torch.empty(steps, b, dtype=torch.int32, device=self.dev)
        logits = torch.empty(steps, b, cfg.vocab, dtype=F32, device=self.dev) if keep_logits else None
        ev = {"done": {}, "d2h": {}}
        n = steps * L
        marks = []
        t0 = torch.cuda.Event(enable_timing=True) if timing is not None else None
        if t0 is not None:
            t0.record(cs)
        n0 = _lib.load().kvpr_kernel_launches()
        self._issue_loads(0, base, splits, ev)
        ahead = L > 1  # one layer: unit u+1's loads wait on unit u's D2H, recorded by its compute
        for u in range(n):
            if ahead and u + 1 < n:
                self._issue_loads(u + 1, base, splits, ev)
            i, j = divmod(u, L)
            if j == 0:
                kernels.embed(self.tok, self.embed, self.pos, self.hres, batch=b, pos_begin=base + i, stream=cs)
            self._compute(u, base, splits, ev)
            if timing is not None:
                e = torch.cuda.Event(enable_timing=True)
                e.record(cs)
                marks.append(e)
            if j == L - 1:
                self._head(self.hres)
                with torch.cuda.stream(cs):
                    out[i].copy_(self.tok, non_blocking=True)
                    if logits is not None:
                        logits[i].copy_(self.logits, non_blocking=True)
            if not ahead and u + 1 < n:
                self._issue_loads(u + 1, base, splits, ev)
            for d in (ev["done"], ev["d2h"]):
                for key in [k for k in d if k < u - L - 2]:
                    del d[key]
        self.len = base + steps
        self.launches += _lib.load().kvpr_kernel_launches() - n0
        cur = torch.cuda.current_stream(self.dev)
        cur.wait_stream(cs)
        cur.wait_stream(self.ds)
        self.last_logits = logits
        if timing is not None:
            cs.synchronize()
            prev = t0
            for i in range(steps):
                row = []
                for e in marks[i * L:(i + 1) * L]:
                    row.append(prev.elapsed_time(e))
                    prev = e
                timing.layer_ms.append(row)
                timing.step_ms.append(sum(row))
        return out

    def close(self):
        if self.peer is not None:
            err = self.peer.error()
            self.peer.close(self.group)
            self.peer = None
            if err:
                raise RuntimeError("fused TP all-reduce: a peer flag wait timed out (results are invalid)")
        for t in (self.store_x, self.store_kv):
            unpin(t)
