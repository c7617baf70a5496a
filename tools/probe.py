"""One-shot GPU-box probe: host/PCIe facts plus first kernel timings.

    python tools/probe.py > gpurun_out/probe.json

Times (CUDA events, warm): K1 at the OPT-6.7B config-2 shape, K2 decode
attention at b32/s'1025, pinned H2D/D2H bandwidth at 16 MiB..1 GiB.
"""

from __future__ import annotations

import json
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2411_17089_b200 import kernels  # noqa: E402


def sh(cmd):
    try:
        return subprocess.run(cmd, shell=True, capture_output=True, text=True, timeout=30).stdout.strip()
    except Exception as e:  # pragma: no cover
        return str(e)


def timeit(fn, iters=10, warm=3):
    for _ in range(warm):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters / 1e3


def main():
    res = {
        "nvidia_smi": sh("nvidia-smi --query-gpu=name,pci.bus_id,clocks.max.sm,memory.total --format=csv,noheader"),
        "topo": sh("nvidia-smi topo -m | head -12"),
        "pcie": sh("nvidia-smi --query-gpu=pcie.link.gen.max,pcie.link.width.max,pcie.link.gen.current --format=csv"),
        "cpu": sh("lscpu | grep -E 'Model name|^CPU\\(s\\)|Socket|NUMA node'"),
        "mem": sh("free -g | head -2"),
        "nproc": os.cpu_count(),
    }
    dev = torch.device("cuda:0")
    # --- K1 at OPT-6.7B b32, l=882 ---
    b, h, l = 32, 4096, 882
    x = torch.randn(l + 1, b, h, device=dev).half()
    w = (torch.randn(2 * h, h, device=dev) * 0.02).half()
    bias = (torch.randn(2 * h, device=dev) * 0.02).half()
    pages = torch.empty(1056, 2, b, h, dtype=torch.float16, device=dev)
    t = timeit(lambda: kernels.recompute_kv(x, w, bias, pages, b, 0, l))
    flops = 4 * b * l * h * h
    res["k1_ms"] = t * 1e3
    res["k1_tflops"] = flops / t / 1e12
    ref = x[:l].float() @ w.float().T + bias.float()
    res["k1_maxerr"] = (pages[:l, 0].float() - ref[..., :h]).abs().max().item()
    del ref
    # --- K2 ---
    q = torch.randn(b, h, device=dev).half()
    out = torch.empty(b, h, dtype=torch.float16, device=dev)
    ws = torch.empty(64 << 20, dtype=torch.uint8, device=dev)
    s = 1025
    t2 = timeit(lambda: kernels.decode_attention(q, pages, out, ws, b, 32, 128, s), iters=20)
    res["k2_us"] = t2 * 1e6
    res["k2_gbs"] = 2 * b * s * h * 2 / t2 / 1e9
    # --- decode GEMMs ---
    xa = torch.randn(b, h, device=dev).half()
    for name, n, k in [("qkv", 3 * h, h), ("out", h, h), ("fc1", 4 * h, h), ("fc2", h, 4 * h)]:
        wt = (torch.randn(n, k, device=dev) * 0.02).half()
        o = torch.empty(b, n, dtype=torch.float16, device=dev)
        a_in = xa if k == h else torch.randn(b, k, device=dev).half()
        tt = timeit(lambda: kernels.linear_simple(a_in, wt, None, o), iters=20)
        res[f"dec_{name}_us"] = tt * 1e6
        res[f"dec_{name}_gbs"] = n * k * 2 / tt / 1e9
    # --- pinned copies ---
    bw = {}
    for mib in (16, 64, 256, 1024):
        nb = mib << 20
        hbuf = torch.empty(nb, dtype=torch.uint8).pin_memory()
        dbuf = torch.empty(nb, dtype=torch.uint8, device=dev)
        th = timeit(lambda: dbuf.copy_(hbuf, non_blocking=True), iters=5, warm=2)
        td = timeit(lambda: hbuf.copy_(dbuf, non_blocking=True), iters=5, warm=2)
        bw[mib] = {"h2d_gbs": nb / th / 1e9, "d2h_gbs": nb / td / 1e9, "h2d_s": th, "d2h_s": td}
        del hbuf, dbuf
    res["pinned"] = bw
    # cudaHostRegister of a pageable buffer (what the runtime uses for exact-size stores)
    t0 = time.perf_counter()
    big = torch.empty(4 << 30, dtype=torch.uint8)
    big.fill_(0)
    t1 = time.perf_counter()
    rc = torch.cuda.cudart().cudaHostRegister(big.data_ptr(), big.numel(), 0)
    t2r = time.perf_counter()
    dbig = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
    tr = timeit(lambda: dbig.copy_(big[: 1 << 30], non_blocking=True), iters=5, warm=2)
    res["host_register"] = {"rc": int(rc), "fill_s": t1 - t0, "register_4g_s": t2r - t1, "h2d_1g_gbs": (1 << 30) / tr / 1e9}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
