"""Time the tcgen05 GEMM variants at the K1 shapes (CUDA events, warm, L2-cold inputs > L2).

    python tools/gemm_bench.py        # prints JSON lines: shape, bn, us, TFLOP/s
"""
import json
import sys

sys.path.insert(0, ".")
import torch

from paper_2411_17089_b200 import kernels


def bench(M, N, K, bn, reps=10):
    dev = torch.device("cuda")
    a = (torch.randn(M, K, device=dev) * 0.5).half()
    w = (torch.randn(N, K, device=dev) * 0.02).half()
    o = torch.empty(M, N, device=dev, dtype=torch.float16)
    for _ in range(3):
        kernels.linear_simple(a, w, None, o, bn=bn)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        kernels.linear_simple(a, w, None, o, bn=bn)
    e.record()
    torch.cuda.synchronize()
    t = s.elapsed_time(e) / reps / 1e3
    return t, 2 * M * N * K / t / 1e12


for M, N, K in ((32, 12288, 4096), (32, 4096, 4096), (32, 16384, 4096), (32, 4096, 16384), (32, 50272, 4096)):
    for bn in (64, 128, 256, 0):
        t, tf = bench(M, N, K, bn, reps=50)
        print(json.dumps({"M": M, "N": N, "K": K, "bn": bn, "us": t * 1e6, "weight_gbs": N * K * 2 / t / 1e9}),
              flush=True)

shapes = [(28224, 8192, 4096), (32 * 220, 8192, 4096), (64 * 1596, 1792, 7168), (32 * 1024, 12288, 4096),
          (8192, 8192, 8192)]
for M, N, K in shapes:
    for bn in (256, 512):
        t, tf = bench(M, N, K, bn)
        print(json.dumps({"M": M, "N": N, "K": K, "bn": bn, "us": t * 1e6, "tflops": tf}), flush=True)

ws = torch.empty(16 << 20, dtype=torch.uint8, device="cuda")
for M, N, K in ((32, 4096, 4096), (32, 4096, 16384), (32, 16384, 4096), (32, 12288, 4096)):
    dev = torch.device("cuda")
    a = (torch.randn(M, K, device=dev) * 0.5).half()
    w = (torch.randn(N, K, device=dev) * 0.02).half()
    o = torch.empty(M, N, device=dev, dtype=torch.float16)
    for _ in range(3):
        kernels.linear_simple(a, w, None, o, ws=ws)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(50):
        kernels.linear_simple(a, w, None, o, ws=ws)
    e.record()
    torch.cuda.synchronize()
    t = s.elapsed_time(e) / 50 / 1e3
    print(json.dumps({"M": M, "N": N, "K": K, "bn": "auto+splitK", "us": t * 1e6, "weight_gbs": N * K * 2 / t / 1e9}),
          flush=True)
