"""Causal prefill attention (csrc/prefill_attn.cu) at the benchmarked prompt shapes: device time per
launch (CUDA events, after warm-up) and the tensor throughput it reaches on the causal FLOPs
(2 GEMMs x 2 flops x b x heads x S(S+1)/2 x head_dim).  One JSON line per shape.

    python tools/prefill_bench.py > gpurun_out/prefill_bench.jsonl
"""
from __future__ import annotations

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2411_17089_b200 import kernels  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    for batch, heads, d, seq in [(32, 32, 128, 1024), (32, 32, 128, 2048), (8, 32, 128, 8192), (4, 12, 64, 256),
                                 (32, 40, 128, 1024)]:
        h = heads * d
        g = torch.Generator(device=dev).manual_seed(0)
        pages = torch.randn(seq, 2, batch, h, generator=g, device=dev).half()
        q = torch.randn(seq, batch, h, generator=g, device=dev).half()
        out = torch.empty(seq, batch, h, dtype=torch.float16, device=dev)
        for _ in range(3):
            kernels.prefill_attention(q, pages, out, batch, heads, d, seq)
        torch.cuda.synchronize()
        reps = 10
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            kernels.prefill_attention(q, pages, out, batch, heads, d, seq)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        flops = 4.0 * batch * heads * d * seq * (seq + 1) / 2
        print(json.dumps({"batch": batch, "heads": heads, "head_dim": d, "seq": seq, "ms": round(ms, 4),
                          "tflops": round(flops / ms / 1e9, 1)}), flush=True)
        del pages, q, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
