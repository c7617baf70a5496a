"""Fused small-batch layer tail (csrc/layer_tail.cu) vs the multi-kernel sequence it replaces, at the
config-1 geometry (OPT-125M shape, b4, s' = 260), weights rotated over 12 layers like a decode step.

    python tools/tail_bench.py > gpurun_out/tail_bench.json
    KVPR_GEMM_TRACE=1 python -m paper_2411_17089_b200.csrc.build --force && python tools/tail_bench.py --trace
      (per-CTA globaltimer stamps of one launch: stage boundaries, see layer_tail.cu tstamp())"""
from __future__ import annotations

import ctypes
import json
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2411_17089_b200 import _lib, kernels  # noqa: E402
from paper_2411_17089_b200.weights import OPTConfig, OPTWeights  # noqa: E402


def main():
    b, S = 4, 260
    cfg = OPTConfig(hidden=768, layers=12, heads=12, ffn=3072, vocab=1024, max_pos=512)
    h, F = cfg.hidden, cfg.ffn
    dev = torch.device("cuda")
    w = OPTWeights.random(cfg, seed=0, device=dev)
    g = torch.Generator(device="cpu").manual_seed(1)
    pages = [torch.randn(S + 2, 2, b, h, generator=g).half().to(dev) for _ in range(2)]
    q = torch.randn(b, h, generator=g).half().to(dev)
    hres = torch.randn(b, h, generator=g).float().to(dev)
    attn = torch.empty(b, h, dtype=torch.float16, device=dev)
    mid = torch.empty(b, F, dtype=torch.float16, device=dev)
    y = torch.empty(b, h, dtype=torch.float16, device=dev)
    xo = torch.empty(b, h, dtype=torch.float16, device=dev)
    ws = torch.empty(16 << 20, dtype=torch.uint8, device=dev)
    s = torch.cuda.Stream(dev)
    acc = _lib.EPI_F32 | _lib.EPI_ACCUM

    def fused(j):
        nxt = w.layers[(j + 1) % cfg.layers]
        kernels.layer_tail(q, pages[j % 2], S, w.layers[j], hres, attn, mid, ws, cfg.heads, cfg.eps,
                           lnx=(nxt.ln1_g, nxt.ln1_b, xo), qkv_next=(nxt.wqkv, nxt.bqkv, q, pages[(j + 1) % 2][S]),
                           stream=s)

    from paper_2411_17089_b200 import hostmem

    host = [hostmem.pinned_empty(tuple(pages[0].shape), torch.float16) for _ in range(2)]
    for hp, dp in zip(host, pages):
        hp.copy_(dp.cpu())
    xs = hostmem.pinned_empty((b, h), torch.float16)
    ps = hostmem.pinned_empty((2, b, h), torch.float16)

    def fused_zc(j, reads=True, writes=True):
        nxt = w.layers[(j + 1) % cfg.layers]
        kernels.layer_tail(q, pages[j % 2], S, w.layers[j], hres, attn, mid, ws, cfg.heads, cfg.eps,
                           lnx=(nxt.ln1_g, nxt.ln1_b, xo), qkv_next=(nxt.wqkv, nxt.bqkv, q, pages[(j + 1) % 2][S]),
                           host_kv=(host[j % 2], S - 9, S - 1) if reads else None,
                           stores=(xs, ps) if writes else None, stream=s)

    def unfused(j):
        lw, nxt = w.layers[j], w.layers[(j + 1) % cfg.layers]
        kernels.decode_attention(q, pages[j % 2], attn, ws, b, cfg.heads, cfg.head_dim, S, stream=s)
        kernels.linear_simple(attn, lw.wo, lw.bo, hres, flags=acc, stream=s, ws=ws)
        kernels.layernorm_linear(hres, lw.ln2_g, lw.ln2_b, y, lw.w1, lw.b1, mid, rows=b, eps=cfg.eps,
                                 flags=_lib.EPI_RELU, stream=s, ws=ws)
        kernels.linear_simple(mid, lw.w2, lw.b2, hres, flags=acc, stream=s, ws=ws)
        kernels.layernorm(hres, nxt.ln1_g, nxt.ln1_b, xo, eps=cfg.eps, stream=s)
        ep = _lib.make_epilogue([(q.data_ptr(), 0), (pages[(j + 1) % 2][S].data_ptr(), 0),
                                 (pages[(j + 1) % 2][S].data_ptr() + b * h * 2, 0)], seg_width=h, ld=h, row_group=b,
                                bias=nxt.bqkv.data_ptr())
        kernels.linear(xo, nxt.wqkv, ep, M=b, stream=s)

    out = {"batch": b, "seq_len": S, "hidden": h, "ffn": F}
    variants = (("fused", fused), ("fused_zc_reads", lambda j: fused_zc(j, True, False)),
                ("fused_zc_writes", lambda j: fused_zc(j, False, True)), ("fused_zc_both", fused_zc),
                ("unfused", unfused))
    for name, fn in variants:
        for it in range(3):
            for j in range(cfg.layers):
                fn(j)
        s.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20
        e0.record(s)
        for it in range(reps):
            for j in range(cfg.layers):
                fn(j)
        e1.record(s)
        e1.synchronize()
        out[f"{name}_us_per_layer"] = e0.elapsed_time(e1) * 1e3 / (reps * cfg.layers)
    if "--trace" in sys.argv:
        lib = _lib.load()
        lib.kvpr_debug_tail_trace.argtypes = [ctypes.c_void_p]
        G = torch.cuda.get_device_properties(dev).multi_processor_count
        buf = torch.zeros(G * 24, dtype=torch.int64, device=dev)
        rows_all = []
        for rep in range(5):
            buf.zero_()
            lib.kvpr_debug_tail_trace(ctypes.c_void_p(buf.data_ptr()))
            fused(rep % cfg.layers)
            s.synchronize()
            lib.kvpr_debug_tail_trace(None)
            t = buf.view(G, 24).cpu().tolist()
            t0 = min(r[0] for r in t if r[0])
            rows_all.append([[(x - t0) if x else None for x in r[:17]] for r in t])
        names = ["entry", "pdl_wait", "A_done", "bar1", "B_done", "bar2", "C_done", "bar3", "D_done", "E_done",
                 "B_merged", "B_w_ready", "C_ln_done", "C_w_ready", "D_staged", "D_w_ready", "B_loaded"]
        summ = []
        for rows in rows_all:
            d = {}
            for k, n in enumerate(names):
                v = sorted(r[k] for r in rows if r[k] is not None)
                if v:
                    d[n] = [v[0], v[len(v) // 2], v[-1]]
            summ.append(d)
        out["trace_ns_min_med_max"] = summ
    print(json.dumps(out))


if __name__ == "__main__":
    main()
