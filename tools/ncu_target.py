"""Short, ncu-friendly driver: the hot kernels once each at the OPT-6.7B config-2 shapes.

    ncu --set full -k regex:gemm_tcgen05 -c 1 python tools/ncu_target.py k1
    ncu --set full -k regex:decode_attn -c 1 python tools/ncu_target.py k2
"""
import sys

sys.path.insert(0, ".")
import torch

from paper_2411_17089_b200 import kernels

which = sys.argv[1] if len(sys.argv) > 1 else "all"
dev = torch.device("cuda:0")
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
