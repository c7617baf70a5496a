"""Config 1 (OPT-125M shape, b4, prompt 256, 16 tokens): is the step bound by the copy stream?  One
timed native decode with every H2D DMA bracketed by CUDA events (kvpr_decoder_kernel_stats kind 2):
copy-stream busy time per step vs the step, achieved GB/s inside the copies, and K1 / K2 launch times.
Variants by environment as in tools/c1_modes.py.

    python tools/c1_h2d.py [--env NAME:K=V,...] > gpurun_out/c1_h2d.jsonl
"""
from __future__ import annotations

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2411_17089_b200.costmodel import WorkloadSpec  # noqa: E402
from paper_2411_17089_b200.hwprofile import HardwareProfile  # noqa: E402
from paper_2411_17089_b200.runtime import DecodeTiming, KVPRRuntime  # noqa: E402
from paper_2411_17089_b200.scheduler import plan_generation  # noqa: E402
from paper_2411_17089_b200.weights import OPTWeights, preset  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--env", action="append", default=[])
    ap.add_argument("--steps", type=int, default=16)
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    cfg, b, S0, gen = preset("opt-125m"), 4, 256, args.steps
    wl = WorkloadSpec(batch_size=b, prompt_len=S0, gen_len=gen)
    prof = HardwareProfile(gpu_flops=1391.2e12, h2d_bandwidth=55.5e9, d2h_bandwidth=55e9)
    splits = plan_generation(cfg.spec(), wl, prof, "column").splits
    w = OPTWeights.random(cfg, seed=0, device=dev)
    prompt = torch.randint(0, cfg.vocab, (b, S0), generator=torch.Generator().manual_seed(1))
    variants = [("default", {})] + [(s.partition(":")[0], dict(kv.split("=", 1) for kv in s.partition(":")[2].split(",") if kv))
                                    for s in args.env]
    keys = set(k for _, m in variants for k in m)
    for name, env in variants:
        for k in keys:
            os.environ.pop(k, None)
        os.environ.update(env)
        rt = KVPRRuntime(w, b, S0 + gen + 1, device=dev)
        first = rt.prefill(prompt)
        rt.decode(splits[:4], tokens=first)
        for timed in (False, True):
            rt.reset(S0)
            rt.kernel_timing = [] if timed else None
            tim = DecodeTiming()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(dev)
            e0.record(rt.cs)
            rt.decode(splits, tokens=first, timing=tim if timed else None)
            e1.record(rt.cs)
            torch.cuda.synchronize(dev)
            ms = e0.elapsed_time(e1) / gen
            if not timed:
                plain = ms
        st = rt.kernel_stats()
        rec = {"mode": name, "ms_per_step": round(plain, 4), "ms_per_step_timed": round(ms, 4),
               "dma_group": rt.dma_group, "nbuf": rt.nbuf}
        if "h2d" in st:
            n, t, u = st["h2d"]
            rec["h2d"] = {"dmas_per_step": n / gen, "us_per_dma": round(t * 1e6, 2), "mb_per_dma": round(u / 1e6, 3),
                          "gbs_in_copy": round(u / t / 1e9, 2), "busy_ms_per_step": round(n * t / gen * 1e3, 4)}
        for k in ("k1", "k2"):
            if k in st:
                rec[k + "_us"] = round(st[k][1] * 1e6, 2)
        rt.close()
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
