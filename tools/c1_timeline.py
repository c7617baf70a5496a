"""Device timeline of a config-1 decode (OPT-125M shape, b4, prompt 256) through the native executor,
recorded with the CUDA profiler interface torch.profiler exposes (CUPTI activity records: every
kernel and copy with its stream and device start / end).  Prints per-stream busy time, the
per-layer period and the first events in order; writes the Chrome trace next to it.

    python tools/c1_timeline.py [--steps 4] [--x-resident] > gpurun_out/c1_timeline.json
"""
from __future__ import annotations

import argparse
import json
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2411_17089_b200.costmodel import WorkloadSpec  # noqa: E402
from paper_2411_17089_b200.hwprofile import HardwareProfile  # noqa: E402
from paper_2411_17089_b200.runtime import KVPRRuntime  # noqa: E402
from paper_2411_17089_b200.scheduler import plan_generation  # noqa: E402
from paper_2411_17089_b200.weights import OPTWeights, preset  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="opt-125m")
    ap.add_argument("--batch", type=int, default=4)
    ap.add_argument("--prompt", type=int, default=256)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--x-resident", action="store_true")
    ap.add_argument("--events", type=int, default=120, help="events listed in order (events_head)")
    ap.add_argument("--trace-out", default="gpurun_out/c1_timeline_trace.json")
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    cfg = preset(args.model).with_positions(args.prompt + 4 * args.steps + 8)
    wl = WorkloadSpec(args.batch, args.prompt, 4 * args.steps)
    prof = HardwareProfile(gpu_flops=1391.2e12, h2d_bandwidth=55e9, d2h_bandwidth=55e9)
    splits = plan_generation(cfg.spec(), wl, prof, "row" if args.x_resident else "column").splits
    w = OPTWeights.random(cfg, seed=0, device=dev)
    prompt = torch.randint(0, cfg.vocab, (args.batch, args.prompt), generator=torch.Generator().manual_seed(1))
    rt = KVPRRuntime(w, args.batch, args.prompt + 4 * args.steps + 1, device=dev, x_resident=args.x_resident)
    first = rt.prefill(prompt)
    K = args.steps
    rt.decode(splits[:K], tokens=first)
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CUDA]) as p:
        rt.decode(splits[K:2 * K])
        torch.cuda.synchronize()
    os.makedirs(os.path.dirname(args.trace_out) or ".", exist_ok=True)
    p.export_chrome_trace(args.trace_out)
    ev = json.load(open(args.trace_out))["traceEvents"]
    gpu = [e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
    gpu.sort(key=lambda e: e["ts"])
    t0 = gpu[0]["ts"]
    t1 = max(e["ts"] + e["dur"] for e in gpu)
    span = t1 - t0
    by_stream = defaultdict(float)
    by_name = defaultdict(lambda: [0, 0.0])
    for e in gpu:
        st = e.get("args", {}).get("stream")
        by_stream[st] += e["dur"]
        n = e["name"].split("(")[0][:60]
        if e["cat"] == "gpu_memcpy":
            n = "memcpy " + e["name"]
        by_name[n][0] += 1
        by_name[n][1] += e["dur"]
    units = K * cfg.layers
    out = {"model": args.model, "batch": args.batch, "prompt": args.prompt, "steps": K, "x_resident": args.x_resident,
           "fused_tail": rt.fused_tail, "span_us": span, "us_per_layer": span / units,
           "busy_us_per_stream": {str(k): v for k, v in by_stream.items()},
           "per_name": {k: {"n": v[0], "us_total": v[1], "us_avg": v[1] / v[0]} for k, v in
                        sorted(by_name.items(), key=lambda kv: -kv[1][1])}}
    out["events_head"] = [[e["name"].split("(")[0][:50], e.get("args", {}).get("stream"), round(e["ts"] - t0, 2),
                           round(e["ts"] + e["dur"] - t0, 2)] for e in gpu[:args.events]]
    rt.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
