"""Short, ncu-friendly driver: the hot kernels once each at the OPT-6.7B config-2 shapes.

    ncu --set full -k regex:gemm_tcgen05 -c 1 python tools/ncu_target.py k1
    ncu --set full -k regex:decode_attn -c 1 python tools/ncu_target.py k2
    ncu --set full -k regex:gemm_tcgen05_kernel -c 1 python tools/ncu_target.py c1   # config-1 shapes
    ncu --set full -k regex:prefill_tc -c 1 python tools/ncu_target.py prefill
    ncu --set full -k regex:prefill_tc -c 1 python tools/ncu_target.py prefill40   # config 3 (40 heads)
"""
import sys

sys.path.insert(0, ".")
import torch

from paper_2411_17089_b200 import kernels

which = sys.argv[1] if len(sys.argv) > 1 else "all"
dev = torch.device("cuda:0")
if which in ("prefill", "prefill40"):  # causal prefill attention at the config-2 (-3) prompt: b32, 32 (40) heads
    b, heads, d, S = 32, 40 if which == "prefill40" else 32, 128, 1024
    pages = torch.randn(S, 2, b, heads * d, device=dev).half()
    q = torch.randn(S, b, heads * d, device=dev).half()
    o = torch.empty_like(q)
    for _ in range(2):
        kernels.prefill_attention(q, pages, o, b, heads, d, S)
    torch.cuda.synchronize()
    print("ok")
    sys.exit(0)
if which == "c1":  # config 1 (OPT-125M shape, b4, s' = 260, l = 252): K1, q/k/v, the CUDA-core projections, K2
    b, h, l, s = 4, 768, 252, 260
    pages = torch.randn(272, 2, b, h, device=dev).half()
    x = torch.randn(l, b, h, device=dev).half()
    w = (torch.randn(3 * h, h, device=dev) * 0.02).half()
    bias = torch.zeros(3 * h, device=dev).half()
    wsb = torch.empty(16 << 20, dtype=torch.uint8, device=dev)
    for _ in range(2):
        kernels.recompute_kv(x, w[h:], bias[h:], pages, b, 0, l)
        a = x[0]
        o = torch.empty(b, 3 * h, device=dev).half()
        kernels.linear_simple(a, w, bias, o)  # q/k/v: swap-AB (kvpr_linear)
        for n, k in ((h, h), (4 * h, h), (h, 4 * h)):
            ak = torch.randn(b, k, device=dev).half()
            wt = (torch.randn(n, k, device=dev) * 0.02).half()
            ok = torch.empty(b, n, device=dev)
            kernels.linear_simple(ak, wt, None, ok, flags=4, ws=wsb)  # fp32 accumulate: gemv
        q = torch.randn(b, h, device=dev).half()
        out = torch.empty(b, h, device=dev).half()
        kernels.decode_attention(q, pages, out, wsb, b, 12, 64, s)
    torch.cuda.synchronize()
    print("ok")
    sys.exit(0)
b, h, l, s = 32, 4096, 882, 1025
pages = torch.randn(1056, 2, b, h, device=dev).half()
if which == "k1chunk":  # one of the runtime's wave-aligned X chunks at config 2 (runtime.wave_positions: 296)
    l = 296
if which in ("k1", "k1chunk", "all"):
    x = torch.randn(l, b, h, device=dev).half()
    w = (torch.randn(2 * h, h, device=dev) * 0.02).half()
    bias = torch.zeros(2 * h, device=dev).half()
    for _ in range(2):
        kernels.recompute_kv(x, w, bias, pages, b, 0, l)
if which in ("k2", "all"):
    q = torch.randn(b, h, device=dev).half()
    out = torch.empty(b, h, device=dev).half()
    ws = torch.empty(16 << 20, dtype=torch.uint8, device=dev)
    for _ in range(2):
        kernels.decode_attention(q, pages, out, ws, b, 32, 128, s)
if which in ("dec", "all"):  # decode projections as the executor issues them (swap-AB; split-K with ws)
    wsb = torch.empty(16 << 20, dtype=torch.uint8, device=dev)
    for n, k, use_ws in ((3 * h, h, False), (h, h, True), (4 * h, h, True), (h, 4 * h, True)):
        a = torch.randn(b, k, device=dev).half()
        wt = (torch.randn(n, k, device=dev) * 0.02).half()
        o = torch.empty(b, n, device=dev).half()
        for _ in range(2):
            kernels.linear_simple(a, wt, None, o, ws=wsb if use_ws else None)
torch.cuda.synchronize()
print("ok")
