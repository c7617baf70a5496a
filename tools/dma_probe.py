"""What slows HBM-bound kernels while PCIe traffic is in flight?  K2 (config-2 shape) timed as single
launches (median of 9) alone and next to: a copy-engine H2D, a copy-engine D2H, a copy-engine D2D, and
an H2D pulled by SM loads from page-locked host memory (zero-copy, kvpr_debug_sm_pull) on 8/16/32 CTAs.

    python tools/dma_probe.py > gpurun_out/dma_probe.json
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2411_17089_b200 import _lib, kernels  # noqa: E402

dev = torch.device("cuda")
b, h, s = 32, 4096, 1025
pages = torch.randn(1056, 2, b, h, device=dev).half()
q = torch.randn(b, h, device=dev).half()
out = torch.empty(b, h, device=dev).half()
ws = torch.empty(16 << 20, dtype=torch.uint8, device=dev)
main = torch.cuda.Stream()
side = torch.cuda.Stream()
N = 1 << 30
from paper_2411_17089_b200.hostmem import mode, pinned_empty  # noqa: E402

host = pinned_empty((N,), torch.uint8)  # KVPR_HOST_ALLOC=register|hostalloc (the host stores' allocation)
dbuf = torch.empty(N, dtype=torch.uint8, device=dev)
dbuf2 = torch.empty(N, dtype=torch.uint8, device=dev)


def k2():
    kernels.decode_attention(q, pages, out, ws, b, 32, 128, s, stream=main)


def single(reps=9):
    ts = []
    for _ in range(reps):
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(main)
        k2()
        e.record(main)
        e.synchronize()
        ts.append(a.elapsed_time(e) * 1e3)
    return sorted(ts)[len(ts) // 2]


def with_bg(start_bg):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    start_bg()
    time.sleep(0.002)
    us = single()
    span = time.perf_counter() - t0
    side.synchronize()
    bg = time.perf_counter() - t0
    return {"k2_us": round(us, 1), "bg_outlasted": bool(bg > span)}


for _ in range(5):
    k2()
torch.cuda.synchronize()
res = {"alone_us": round(single(), 1)}
res["ce_h2d"] = with_bg(lambda: _lib.call("kvpr_copy_async", dbuf.data_ptr(), host.data_ptr(), N, side.cuda_stream))
res["ce_d2h"] = with_bg(lambda: _lib.call("kvpr_copy_async", host.data_ptr(), dbuf.data_ptr(), N, side.cuda_stream))
res["ce_d2d"] = with_bg(lambda: _lib.call("kvpr_copy_async", dbuf2.data_ptr(), dbuf.data_ptr(), N, side.cuda_stream))
for ctas in (8, 16, 32):
    # pull alone: bandwidth
    torch.cuda.synchronize()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(side)
    _lib.call("kvpr_debug_sm_pull", host.data_ptr(), dbuf.data_ptr(), N, ctas, side.cuda_stream)
    e.record(side)
    e.synchronize()
    gbs = N / (a.elapsed_time(e) / 1e3) / 1e9
    r = with_bg(lambda: _lib.call("kvpr_debug_sm_pull", host.data_ptr(), dbuf.data_ptr(), N, ctas,
                                  side.cuda_stream))
    r["pull_gbs_alone"] = round(gbs, 1)
    res[f"sm_pull_{ctas}ctas"] = r
res["host_alloc"] = mode()
print(json.dumps(res))
