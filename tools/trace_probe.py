"""Where does a config-1 layer's time go?  Prequeued (GPU spin first) Python-loop decode with the
measured-timeline tracer: mean duration per traced group and lane busy fractions.  (Events between
the groups cost the PDL overlap at group edges, so totals run above the native executor's.)

    python tools/trace_probe.py [--x-resident]
"""
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
from paper_2411_17089_b200.trace import Tracer, report  # noqa: E402
from paper_2411_17089_b200.weights import OPTWeights, preset  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--x-resident", action="store_true")
args = ap.parse_args()
b, S0, K = 4, 256, 8
cfg = preset("opt-125m").with_positions(S0 + 3 * K + 8)
prof = HardwareProfile(gpu_flops=1391.2e12, h2d_bandwidth=55e9, d2h_bandwidth=55e9)
splits = plan_generation(cfg.spec(), WorkloadSpec(b, S0, 3 * K), prof, "row" if args.x_resident else "column").splits
w = OPTWeights.random(cfg, seed=0, device="cuda")
prompt = torch.randint(0, cfg.vocab, (b, S0), generator=torch.Generator().manual_seed(1))
rt = KVPRRuntime(w, b, S0 + 3 * K + 1, x_resident=args.x_resident)
first = rt.prefill(prompt)
rt.decode(splits[:K], tokens=first, native=False)
torch.cuda.synchronize()
torch.cuda._sleep(int(2e9))
tr = Tracer()
rt.decode(splits[K:2 * K], trace=tr, native=False)
ents = tr.entries()
rt.close()
dur = defaultdict(list)
for e in ents:
    dur[(e.lane, e.kind, e.part.rstrip("0123456789") if e.kind != "compute_mha" else e.part)].append(e.end - e.start)
L = cfg.layers
out = {"layers": L, "steps": K, "x_resident": args.x_resident,
       "per_layer_us": {f"{k[0]}:{k[1]}:{k[2]}": round(sum(v) / (K * L) * 1e6, 2) for k, v in sorted(dur.items())},
       "report": {k: v for k, v in report(ents, b * K).items() if k != "breakdown"}}
out["makespan_per_layer_us"] = round(out["report"]["makespan_s"] / (K * L) * 1e6, 2)
print(json.dumps(out))
