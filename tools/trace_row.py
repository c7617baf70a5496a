"""Measured timeline of a few decode steps (row or column schedule) at the config-2 shape:
per-lane busy fractions and the mean duration of each operation kind per layer.

    python tools/trace_row.py [--row] [--layers 32] [--steps 3] [--trace out.json]
"""
import argparse
import json
import statistics
import sys

sys.path.insert(0, ".")
import torch

from paper_2411_17089_b200 import profiler, trace
from paper_2411_17089_b200.costmodel import WorkloadSpec
from paper_2411_17089_b200.runtime import KVPRRuntime
from paper_2411_17089_b200.scheduler import plan_generation
from paper_2411_17089_b200.weights import OPTConfig, preset, OPTWeights

ap = argparse.ArgumentParser()
ap.add_argument("--row", action="store_true")
ap.add_argument("--layers", type=int, default=32)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--trace")
a = ap.parse_args()
base = preset("opt-6.7b")
cfg = OPTConfig(base.hidden, a.layers, base.heads, base.ffn, max_pos=2048)
b, P = 32, 1024
calib, recs = profiler.measure(cfg.hidden, b)
wl = WorkloadSpec(batch_size=b, prompt_len=P, gen_len=a.steps + 1)
plan = plan_generation(cfg.spec(), wl, calib.profile, "row" if a.row else "column")
w = OPTWeights.random(cfg, seed=0, device="cuda")
rt = KVPRRuntime(w, b, P + a.steps + 2, x_resident=a.row)
first = rt.prefill(torch.randint(0, cfg.vocab, (b, P), generator=torch.Generator().manual_seed(1)))
rt.decode(plan.splits[:1], tokens=first)
tr = trace.Tracer()
rt.decode(plan.splits[1:], trace=tr)
torch.cuda.synchronize()
ents = tr.entries()
rep = trace.report(ents, b * a.steps)
by = {}
for e in ents:
    by.setdefault((e.kind, e.part[:1] if e.kind != "compute_mha" else e.part), []).append((e.end - e.start) * 1e3)
print(json.dumps({"row": a.row, "splits": plan.splits[1:], "ms_per_step": rep["makespan_s"] / a.steps * 1e3,
                  "lane_busy": rep["lane_busy"], "gpu_util": rep["gpu_util"],
                  "mean_ms": {f"{k}:{p}": statistics.mean(v) for (k, p), v in by.items()},
                  "sum_ms_per_layer": {f"{k}:{p}": sum(v) / (a.steps * a.layers) for (k, p), v in by.items()}},
                 indent=1))
if a.trace:
    trace.write_trace(ents, a.trace)
rt.close()
