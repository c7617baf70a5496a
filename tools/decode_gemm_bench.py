"""Decode-GEMM (M = batch rows, weight streaming) timings as the executor sees them.

    python tools/decode_gemm_bench.py > gpurun_out/decode_gemm.jsonl

Unlike tools/gemm_bench.py (Python issue per launch, weights L2-hot), every launch here is
queued behind a GPU spin first, so the host issue cost is hidden exactly as in the C executor,
and the weights rotate over enough copies (> 2x L2) that each launch streams them from HBM,
as in a decode step (13 GB of weights per step).  Reports us per launch and weight GB/s.
"""

from __future__ import annotations

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2411_17089_b200 import kernels  # noqa: E402

L2_ROTATE_BYTES = 320 << 20


def run(M, N, K, bn, ws=None, reps=40, f32=False):
    dev = torch.device("cuda")
    n_copies = max(2, -(-L2_ROTATE_BYTES // (N * K * 2)))
    ws_ = [(torch.randn(N, K, device=dev) * 0.02).half() for _ in range(n_copies)]
    a = (torch.randn(M, K, device=dev) * 0.5).half()
    bias = (torch.randn(N, device=dev) * 0.02).half()
    o = torch.empty(M, N, device=dev, dtype=torch.float32 if f32 else torch.float16)
    for i in range(3):
        kernels.linear_simple(a, ws_[i % n_copies], bias, o, bn=bn, ws=ws)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(int(2e8))  # ~0.1 s: all launches below queue behind it
    s.record()
    for i in range(reps):
        kernels.linear_simple(a, ws_[i % n_copies], bias, o, bn=bn, ws=ws)
    e.record()
    torch.cuda.synchronize()
    t = s.elapsed_time(e) / reps / 1e3
    return t


def main():
    wsb = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
    shapes = [
        # config 1 (OPT-125M shape, b4): qkv, out-proj, fc1, fc2, LM head
        (4, 2304, 768), (4, 768, 768), (4, 3072, 768), (4, 768, 3072), (4, 50272, 768),
        # config 2 (OPT-6.7B, b32)
        (32, 12288, 4096), (32, 4096, 4096), (32, 16384, 4096), (32, 4096, 16384), (32, 50272, 4096),
    ]
    # K1 at small models: M = b * l rows (config 1: b4, l ~ 250), N = 2h, K = h; every tile shape
    # accumulates K in the same order (bit-identical), so the choice is free
    for M, N, K in (() if "--swap-only" in sys.argv else
                    ((1000, 1536, 768), (4 * 64, 1536, 768), (32 * 250, 1536, 768), (4 * 880, 8192, 4096))):
        for bn in (512, 256, 128, 64, 32):
            t = run(M, N, K, bn)
            print(json.dumps({"M": M, "N": N, "K": K, "bn": bn, "k1": True, "us": round(t * 1e6, 2),
                              "tflops": round(2 * M * N * K / t / 1e12, 1)}), flush=True)
    if "--k1-only" in sys.argv:
        return
    if "--gemv" in sys.argv:
        # CUDA-core decode projection (bn -2) vs the swap-AB tensor-core kernel (with its split-K
        # workspace) at batch <= 8: config-1 shapes, then OPT-6.7B / 13B shapes at b4 / b8
        gshapes = [(m, n, k) for m in (1, 4, 8) for (n, k) in ((768, 768), (3072, 768), (768, 3072), (50272, 768))]
        gshapes += [(m, n, k) for m in (4, 8) for (n, k) in ((4096, 4096), (16384, 4096), (4096, 16384),
                                                             (5120, 5120), (20480, 5120), (5120, 20480))]
        for M, N, K in gshapes:
            for bn in ((-2, -1) if M * K * 2 <= 96 * 1024 else (-1,)):  # gemv stages M x K of A in smem
                t = run(M, N, K, bn, ws=wsb)
                print(json.dumps({"M": M, "N": N, "K": K, "bn": bn, "split_ws": True, "us": round(t * 1e6, 2),
                                  "weight_gbs": round(N * K * 2 / t / 1e9, 1)}), flush=True)
        return
    for M, N, K in shapes:
        for bn in ((-1,) if "--swap-only" in sys.argv else (-1, 32, 128, 0)):
            for split in (False, True):
                t = run(M, N, K, bn, ws=wsb if split else None)
                print(json.dumps({"M": M, "N": N, "K": K, "bn": bn, "split_ws": split, "us": round(t * 1e6, 2),
                                  "kbox": os.environ.get("KVPR_SWAP_KBOX", "default"),
                                  "weight_gbs": round(N * K * 2 / t / 1e9, 1)}), flush=True)


if __name__ == "__main__":
    main()
