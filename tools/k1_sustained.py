"""K1 (the recompute GEMM) at the row schedule's launch shape (OPT-6.7B, b32, l = 888 -> M = 28416,
N = 8192, K = 4096), back to back for a few hundred launches: the burst rate (first 10) vs the
sustained rate (last 100), alone and with a pinned H2D copy loop running on another stream (the
row schedule's KV[l:s'-1] DMA).  Is the in-step K1 slower than K1 alone at its sustained clock?

    python tools/k1_sustained.py > gpurun_out/k1_sustained.json
"""
from __future__ import annotations

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2411_17089_b200 import hostmem, kernels  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    b, h, l = 32, 4096, 888
    x = (torch.randn(l, b, h, device=dev) * 0.5).half()
    w = (torch.randn(2 * h, h, device=dev) * 0.02).half()
    bias = torch.zeros(2 * h, device=dev).half()
    pages = torch.empty(l + 8, 2, b, h, device=dev, dtype=torch.float16)
    flops = 4.0 * b * l * h * h
    host = hostmem.pinned_empty((256 << 20,), torch.uint8)
    dbuf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    cs, hs = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    out = {"M": b * l, "N": 2 * h, "K": h, "flops_per_launch": flops}
    import threading

    import pynvml

    pynvml.nvmlInit()
    hnd = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    a8 = torch.randn(8192, 8192, device=dev).half()
    b8 = torch.randn(8192, 8192, device=dev).half()
    c8 = torch.empty(8192, 8192, device=dev).half()
    for dma in (False, True, "cublas"):
        samples, stop = [], threading.Event()

        def sample():
            while not stop.is_set():
                samples.append((pynvml.nvmlDeviceGetClockInfo(hnd, pynvml.NVML_CLOCK_SM),
                                pynvml.nvmlDeviceGetPowerUsage(hnd) / 1e3,
                                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(hnd)))
                stop.wait(0.02)

        th = threading.Thread(target=sample, daemon=True)
        th.start()
        n = 300
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(n + 1)]
        torch.cuda.synchronize()
        if dma is True:  # keep the copy engine busy for the whole loop (~55 GB/s H2D)
            with torch.cuda.stream(hs):
                for _ in range(int(n * 1.6e-3 * 55e9 / (256 << 20)) + 4):
                    dbuf.copy_(host, non_blocking=True)
        ev[0].record(cs)
        for i in range(n):
            if dma == "cublas":  # the MEASURED_PEAKS sustained reference: fp16 8192^3 through cuBLAS
                with torch.cuda.stream(cs):
                    torch.mm(a8, b8, out=c8)
            else:
                kernels.recompute_kv(x, w, bias, pages, b, 0, l, stream=cs)
            ev[i + 1].record(cs)
        torch.cuda.synchronize()
        stop.set()
        th.join()
        us = [ev[i].elapsed_time(ev[i + 1]) * 1e3 for i in range(n)]
        key = {False: "alone", True: "with_h2d", "cublas": "cublas_8192"}[dma]
        fl = 2.0 * 8192 ** 3 if dma == "cublas" else flops
        out[key] = {"first10_us": sum(us[:10]) / 10, "last100_us": sum(us[-100:]) / 100,
                    "first10_tflops": fl / (sum(us[:10]) / 10) / 1e6,
                    "last100_tflops": fl / (sum(us[-100:]) / 100) / 1e6,
                    "sm_mhz_last_half": sorted(c for c, _, _ in samples[len(samples) // 2:])[len(samples) // 4]
                    if samples else None,
                    "power_w_max": max((p for _, p, _ in samples), default=None),
                    "throttle_reasons": sorted({r for _, _, r in samples})}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
