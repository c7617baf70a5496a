"""Copy-engine cost of config 1's per-layer H2D DMAs when several layers' copies go as ONE strided
(2-D) submission: X[j][0:l] (~1.6 MB) and KV[j][l:s'-1] (~100 KB) for G consecutive layers j, host
pitch = one layer's store, device pitch = one staging buffer (kvpr_copy_2d_async).  Per-layer cost in
us for G = 1, 2, 3, 4, 6, 12, X alone, KV alone and X + KV back to back on one stream.

    python tools/dma_2d_probe.py > gpurun_out/dma_2d_probe.json
"""
from __future__ import annotations

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2411_17089_b200 import _lib, hostmem  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    L, X, KV = 12, 1_600_000, 98_304
    HP, DP = 4 * X, 2 * X  # host layer stride (store of S positions), device staging-buffer stride
    hx = hostmem.pinned_empty((L * HP,), torch.uint8)
    dx = torch.empty(L * DP, dtype=torch.uint8, device=dev)
    hx.fill_(1)
    s = torch.cuda.Stream(dev)
    lib = _lib.load()
    out = {}

    def timed(name, body, reps=20):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(reps):
            body()
        e1.record(s)
        torch.cuda.synchronize()
        out[name] = round(e0.elapsed_time(e1) * 1e3 / (reps * L), 3)  # us per layer

    def run(width_x, width_kv, g):
        def body():
            for j0 in range(0, L, g):
                h = min(g, L - j0)
                if width_x:
                    _lib.call("kvpr_copy_2d_async", dx.data_ptr() + j0 * DP, DP, hx.data_ptr() + j0 * HP, HP,
                              width_x, h, s.cuda_stream)
                if width_kv:  # the KV tail sits past X in both pitches (a different region of the same store)
                    _lib.call("kvpr_copy_2d_async", dx.data_ptr() + j0 * DP + X, DP, hx.data_ptr() + j0 * HP + 2 * X,
                              HP, width_kv, h, s.cuda_stream)
        return body

    s2 = torch.cuda.Stream(dev)

    def two_streams(width_x, width_kv):  # layer j's copies on stream j % 2 (two copy engines in flight)
        def body():
            for j in range(L):
                st = s if j % 2 == 0 else s2
                if width_x:
                    _lib.call("kvpr_copy_async", dx.data_ptr() + j * DP, hx.data_ptr() + j * HP, width_x, st.cuda_stream)
                if width_kv:
                    _lib.call("kvpr_copy_async", dx.data_ptr() + j * DP + X, hx.data_ptr() + j * HP + 2 * X, width_kv,
                              st.cuda_stream)
        return body

    def timed2(name, body, reps=20):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        s2.wait_stream(s)
        for _ in range(reps):
            body()
        s.wait_stream(s2)
        e1.record(s)
        torch.cuda.synchronize()
        out[name] = round(e0.elapsed_time(e1) * 1e3 / (reps * L), 3)

    def split_rows(rows):  # one layer's X as ONE 2-D submission of `rows` contiguous rows (pitch = width)
        w = X // rows

        def body():
            for j in range(L):
                _lib.call("kvpr_copy_2d_async", dx.data_ptr() + j * DP, w, hx.data_ptr() + j * HP, w, w, rows,
                          s.cuda_stream)
        return body

    for _ in range(2):
        for rows in (1, 4, 16, 64):
            timed(f"x_rows{rows}_us", split_rows(rows))
        timed2("x_2streams_us", two_streams(X, 0))
        timed2("x_kv_2streams_us", two_streams(X, KV))
        for g in (1, 2, 3, 4, 6, 12):
            timed(f"x_g{g}_us", run(X, 0, g))
            timed(f"kv_g{g}_us", run(0, KV, g))
            timed(f"x_kv_g{g}_us", run(X, KV, g))
    out["x_bytes"], out["kv_bytes"] = X, KV
    out["x_g1_gbs"] = X / out["x_g1_us"] / 1e3
    out["x_g12_gbs"] = X / out["x_g12_us"] / 1e3
    print(json.dumps(out))


if __name__ == "__main__":
    main()
