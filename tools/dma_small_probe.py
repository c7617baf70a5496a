"""Copy-engine cost of the per-layer DMAs of a small model (config 1: X[:, :l] ~1.6 MB and the KV tail
~100 KB host -> device, the new X row 6 KB + K,V page 12 KB device -> host), alone and combined:
one vs two H2D streams, with and without the concurrent D2H traffic of the step.

    python tools/dma_small_probe.py > gpurun_out/dma_small_probe.json
"""
from __future__ import annotations

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2411_17089_b200 import hostmem  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    X, KV, DX, DKV = 1_600_000, 98_304, 6_144, 12_288
    reps = 50
    # the runtime's host stores are exact-size cudaHostAlloc (hostmem.py)
    hx = hostmem.pinned_empty((X * reps,), torch.uint8)
    hk = hostmem.pinned_empty((KV * reps,), torch.uint8)
    hd = hostmem.pinned_empty(((DX + DKV) * reps,), torch.uint8)
    dx = torch.empty(X * 2, dtype=torch.uint8, device=dev)
    dk = torch.empty(KV * 2, dtype=torch.uint8, device=dev)
    dd = torch.empty(DX + DKV, dtype=torch.uint8, device=dev)
    s1, s2, s3 = torch.cuda.Stream(dev), torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    out = {}

    def timed(name, body):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cur = torch.cuda.current_stream()
        e0.record(cur)
        for s in (s1, s2, s3):
            s.wait_stream(cur)
        body()
        for s in (s1, s2, s3):
            cur.wait_stream(s)
        e1.record(cur)
        torch.cuda.synchronize()
        out[name] = e0.elapsed_time(e1) * 1e3 / reps

    def x_only():
        with torch.cuda.stream(s1):
            for i in range(reps):
                dx[(i % 2) * X:(i % 2 + 1) * X].copy_(hx[i * X:(i + 1) * X], non_blocking=True)

    def kv_only():
        with torch.cuda.stream(s1):
            for i in range(reps):
                dk[(i % 2) * KV:(i % 2 + 1) * KV].copy_(hk[i * KV:(i + 1) * KV], non_blocking=True)

    def x_kv_one_stream():
        with torch.cuda.stream(s1):
            for i in range(reps):
                dx[(i % 2) * X:(i % 2 + 1) * X].copy_(hx[i * X:(i + 1) * X], non_blocking=True)
                dk[(i % 2) * KV:(i % 2 + 1) * KV].copy_(hk[i * KV:(i + 1) * KV], non_blocking=True)

    def x_kv_two_streams():
        for i in range(reps):
            with torch.cuda.stream(s1):
                dx[(i % 2) * X:(i % 2 + 1) * X].copy_(hx[i * X:(i + 1) * X], non_blocking=True)
            with torch.cuda.stream(s2):
                dk[(i % 2) * KV:(i % 2 + 1) * KV].copy_(hk[i * KV:(i + 1) * KV], non_blocking=True)

    def with_d2h(body):
        def f():
            body()
            with torch.cuda.stream(s3):
                for i in range(reps):
                    hd[i * (DX + DKV):i * (DX + DKV) + DX].copy_(dd[:DX], non_blocking=True)
                    hd[i * (DX + DKV) + DX:(i + 1) * (DX + DKV)].copy_(dd[DX:], non_blocking=True)
        return f

    def d2h_only():
        with torch.cuda.stream(s3):
            for i in range(reps):
                hd[i * (DX + DKV):i * (DX + DKV) + DX].copy_(dd[:DX], non_blocking=True)
                hd[i * (DX + DKV) + DX:(i + 1) * (DX + DKV)].copy_(dd[DX:], non_blocking=True)

    import ctypes

    from paper_2411_17089_b200 import _lib

    lib = _lib.load()
    lib.kvpr_copy_batch_async.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_size_t, ctypes.c_void_p]

    def x_kv_one_call():
        dsts = (ctypes.c_void_p * 2)()
        srcs = (ctypes.c_void_p * 2)()
        sizes = (ctypes.c_size_t * 2)(X, KV)
        for i in range(reps):
            dsts[0], dsts[1] = dx[(i % 2) * X:].data_ptr(), dk[(i % 2) * KV:].data_ptr()
            srcs[0], srcs[1] = hx[i * X:].data_ptr(), hk[i * KV:].data_ptr()
            rc = lib.kvpr_copy_batch_async(dsts, srcs, sizes, 2, ctypes.c_void_p(s1.cuda_stream))
            if rc:
                raise RuntimeError(_lib.last_error())

    for _ in range(2):
        timed("x_kv_one_call_us", x_kv_one_call)
        timed("x_kv_one_call_with_d2h_us", with_d2h(x_kv_one_call))
        timed("x_only_us", x_only)
        timed("kv_only_us", kv_only)
        timed("d2h_pair_only_us", d2h_only)
        timed("x_then_kv_one_stream_us", x_kv_one_stream)
        timed("x_kv_two_streams_us", x_kv_two_streams)
        timed("x_then_kv_one_stream_with_d2h_us", with_d2h(x_kv_one_stream))
        timed("x_kv_two_streams_with_d2h_us", with_d2h(x_kv_two_streams))
    out["x_only_gbs"] = X / out["x_only_us"] / 1e3
    print(json.dumps(out))


if __name__ == "__main__":
    main()
