"""Row schedule (X resident in HBM, reference solver mode "row") at config 2: per-layer time and the
in-step K1 / K2 launch times from an instrumented replay.  KVPR_K1_STREAM=0/1 A/B via the env.

    python tools/row_probe.py > gpurun_out/row_probe.jsonl
"""
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

b, S0, W, K = 32, 1024, 3, 8
cfg = preset("opt-6.7b").with_positions(S0 + W + K + 8)
prof = HardwareProfile(gpu_flops=1391.2e12, h2d_bandwidth=55e9, d2h_bandwidth=55e9)
splits = plan_generation(cfg.spec(), WorkloadSpec(b, S0, W + K), prof, "row").splits
w = OPTWeights.random(cfg, seed=0, device="cuda")
prompt = torch.randint(0, cfg.vocab, (b, S0), generator=torch.Generator().manual_seed(1))
rt = KVPRRuntime(w, b, S0 + W + K + 1, x_resident=True)
first = rt.prefill(prompt)
rt.decode(splits[:W], tokens=first)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(rt.cs)
rt.decode(splits[W:])
e.record(rt.cs)
torch.cuda.synchronize()
plain = s.elapsed_time(e) / K
rt.reset(S0 + W)
rt.kernel_timing = []
tim = DecodeTiming()
rt.decode(splits[W:], timing=tim)
torch.cuda.synchronize()
ks = rt.kernel_stats()
lay = sorted(x for row in tim.layer_ms for x in row[1:])
print(json.dumps({"k1_stream": rt.k1_stream, "ms_per_step": plain, "tok_s": b / plain * 1e3,
                  "layer_ms_median": lay[len(lay) // 2], "splits": splits[W:],
                  "kernel_stats": {k: [v[0], v[1] * 1e6] for k, v in ks.items()}}), flush=True)
rt.close()
