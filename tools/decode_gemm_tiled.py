"""Decode-GEMM weight streaming: row-major vs box-tiled weights (kvpr_tile_weight), unsplit vs stream-K.

    python tools/decode_gemm_tiled.py > gpurun_out/decode_gemm_tiled.jsonl

Each launch queues behind a GPU spin (host issue hidden, as in the C executor) and the weights
rotate over copies totalling > 2x L2, so every launch streams its weights from HBM.  Reports
us per launch and weight GB/s (weight bytes / time)."""

from __future__ import annotations

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2411_17089_b200 import kernels  # noqa: E402

ROTATE = 320 << 20


def run(M, N, K, tiled, ws, reps=40):
    dev = torch.device("cuda")
    n = max(2, -(-ROTATE // (N * K * 2)))
    mats = [(torch.randn(N, K, device=dev) * 0.02).half() for _ in range(n)]
    if tiled:
        mats = [kernels.tile_weight(m) for m in mats]
    a = (torch.randn(M, K, device=dev) * 0.5).half()
    o = torch.empty(M, N, device=dev)
    for i in range(3):
        kernels.linear_simple(a, mats[i % n], None, o, bn=-1, ws=ws)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(int(2e8))
    s.record()
    for i in range(reps):
        kernels.linear_simple(a, mats[i % n], None, o, bn=-1, ws=ws)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps / 1e3


def main():
    ws = torch.empty(16 << 20, dtype=torch.uint8, device="cuda")
    shapes = [(32, 12288, 4096), (32, 4096, 4096), (32, 16384, 4096), (32, 4096, 16384), (32, 50272, 4096),
              (16, 5120, 5120), (4, 4096, 4096), (64, 7168, 7168)]
    for M, N, K in shapes:
        for tiled in (False, True):
            for sk in (False, True):
                t = run(M, N, K, tiled, ws if sk else None)
                print(json.dumps({"M": M, "N": N, "K": K, "tiled": tiled, "stream_k": sk, "us": round(t * 1e6, 2),
                                  "weight_gbs": round(N * K * 2 / t / 1e9, 1)}), flush=True)


if __name__ == "__main__":
    main()
