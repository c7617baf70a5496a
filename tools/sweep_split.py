"""BASELINE config 5: split-point sweep l in [0, s'] at prompts 512..8192 on the
OPT-6.7B geometry — measured per-layer decode latency vs the overlap roofline,
and the scheduler's l vs the measured optimum.

    python tools/sweep_split.py [--layers 4] [--prompts 512,1024,2048,4096,8192] > sweep.jsonl

Per-layer latency is what is swept, so a reduced layer count (default 4 of the
32 OPT-6.7B layers, identical per-layer shapes) keeps host stores within the
box's DRAM at prompt 8192.  Each point = median layer time over `steps`
decode steps at a constant split (the runtime rewinds the cache between
points so s' is the same for every l).
"""

from __future__ import annotations

import argparse
import json
import statistics
import sys

sys.path.insert(0, ".")

import torch  # noqa: E402

from paper_2411_17089_b200 import profiler  # noqa: E402
from paper_2411_17089_b200.costmodel import WorkloadSpec  # noqa: E402
from paper_2411_17089_b200.runtime import DecodeTiming, KVPRRuntime  # noqa: E402
from paper_2411_17089_b200.scheduler import layer_time, overlap_roofline, solve_split  # noqa: E402
from paper_2411_17089_b200.weights import OPTConfig, OPTWeights, preset  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--prompts", default="512,1024,2048,4096,8192")
    ap.add_argument("--points", type=int, default=11)
    ap.add_argument("--steps", type=int, default=3)
    args = ap.parse_args()
    base = preset("opt-6.7b")
    peaks = json.load(open("MEASURED_PEAKS.json")) if __import__("os").path.exists("MEASURED_PEAKS.json") else \
        {"bf16_tflops_sustained": 1400.0}
    f_peak = peaks["bf16_tflops_sustained"] * 1e12
    b = args.batch
    calib, recs = profiler.measure(base.hidden, b)
    prof = calib.profile
    bw = profiler.peak_h2d(recs)
    print(json.dumps({"profile": prof.to_dict(), "bw_peak": bw, "f_peak": f_peak}), flush=True)
    for P in [int(x) for x in args.prompts.split(",")]:
        cfg = OPTConfig(base.hidden, args.layers, base.heads, base.ffn, base.vocab, max(base.max_pos, P + 16))
        w = OPTWeights.random(cfg, seed=0, device="cuda")
        prompt = torch.randint(0, cfg.vocab, (b, P), generator=torch.Generator().manual_seed(1))
        steps = args.steps
        rt = KVPRRuntime(w, b, P + steps + 1)
        first = rt.prefill(prompt)
        s1 = P + 1
        spec = cfg.spec()
        wl = WorkloadSpec(batch_size=b, prompt_len=P, gen_len=steps)
        l_sched = solve_split(spec, wl, prof, s1, "column").recompute_len
        grid = sorted({round(i * s1 / (args.points - 1)) for i in range(args.points)} | {l_sched})
        rows = []
        for l in grid:
            rt.reset(P)
            tim = DecodeTiming()
            rt.decode([min(l, P + 1 + i) for i in range(steps)], tokens=first, timing=tim)
            per_layer = [x for row in tim.layer_ms for x in row[1:]]
            med = statistics.median(per_layer)
            troof = overlap_roofline(spec, wl, s1, l, bw, f_peak) * 1e3
            pred = layer_time(spec, wl, prof, s1, l, "column").total * 1e3
            row = {"prompt": P, "l": l, "layer_ms": med, "troof_ms": troof, "pred_column_ms": pred,
                   "frac": troof / med, "sched": l == l_sched}
            rows.append(row)
            print(json.dumps(row), flush=True)
        best = min(rows, key=lambda r: r["layer_ms"])
        at = next(r for r in rows if r["sched"])
        print(json.dumps({"prompt": P, "summary": True, "l_sched": l_sched, "layer_ms_at_sched": at["layer_ms"],
                          "troof_ms_at_sched": at["troof_ms"], "l_measured_opt": best["l"],
                          "layer_ms_at_opt": best["layer_ms"], "troof_min_ms": min(r["troof_ms"] for r in rows)}),
              flush=True)
        rt.close()
        del rt, w
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
