"""Is a small-model decode (BASELINE config 1) host-issue bound or GPU-latency bound?

    python tools/issue_probe.py [--model opt-125m --batch 4 --prompt 256 --steps 8] > gpurun_out/issue_probe.json

Three timings of the same K decode steps through the native executor:
  normal     device time of decode() issued while the GPU is idle (what bench.py measures)
  prequeued  device time when every op is already queued behind a long spin on the
             GPU (host issue cost hidden): the pure GPU-side chain of launches, copies and waits
  issue      host wall time of the decode() call in the prequeued run
normal ~ issue >> prequeued  => host-issue bound;  normal ~ prequeued  => GPU-latency bound.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

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
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--graph", type=int, default=-1, help="force executor graph mode (0/1); -1 = runtime default")
    ap.add_argument("--x-resident", action="store_true", help="row schedule: X resident in HBM (no X H2D)")
    ap.add_argument("--nbuf", type=int, default=None, help="device staging buffers per category (default: the runtime's)")
    ap.add_argument("--split", type=int, default=-2, help=">= 0: constant split l; -1: l = s' (all recompute)")
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    cfg = preset(args.model).with_positions(args.prompt + 4 * args.steps + 8)
    wl = WorkloadSpec(args.batch, args.prompt, 4 * args.steps)
    prof = HardwareProfile(gpu_flops=1391.2e12, h2d_bandwidth=55e9, d2h_bandwidth=55e9)
    splits = plan_generation(cfg.spec(), wl, prof, "row" if args.x_resident else "column").splits
    if args.split >= 0:
        splits = [min(args.split, args.prompt + i + 1) for i in range(len(splits))]
    elif args.split == -1:
        splits = [args.prompt + i + 1 for i in range(len(splits))]
    w = OPTWeights.random(cfg, seed=0, device=dev)
    prompt = torch.randint(0, cfg.vocab, (args.batch, args.prompt), generator=torch.Generator().manual_seed(1))
    rt = KVPRRuntime(w, args.batch, args.prompt + 4 * args.steps + 1, device=dev, x_resident=args.x_resident,
                     nbuf=args.nbuf)
    if args.graph >= 0 and hasattr(rt, "graph"):
        rt.graph = bool(args.graph)
    first = rt.prefill(prompt)
    K = args.steps
    rt.decode(splits[:K], tokens=first)  # warm-up
    torch.cuda.synchronize()
    out = {"model": args.model, "batch": args.batch, "prompt": args.prompt, "steps": K, "layers": cfg.layers,
           "x_resident": args.x_resident, "split": args.split, "nbuf": args.nbuf, "pdl": os.environ.get("KVPR_PDL", "1"),
           "splits": splits[K:2 * K]}

    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cur = torch.cuda.current_stream()
    e0.record(cur)
    t0 = time.perf_counter()
    rt.decode(splits[K:2 * K])
    issue_normal = time.perf_counter() - t0
    e1.record(cur)
    torch.cuda.synchronize()
    out["normal_ms_per_step"] = e0.elapsed_time(e1) / K
    out["normal_issue_ms_per_step"] = issue_normal * 1e3 / K

    torch.cuda._sleep(int(2e9))  # ~1 s of spin at ~2 GHz: every op below queues behind it
    e0.record(cur)
    t0 = time.perf_counter()
    rt.decode(splits[2 * K:3 * K])
    issue = time.perf_counter() - t0
    e1.record(cur)
    torch.cuda.synchronize()
    out["prequeued_ms_per_step"] = e0.elapsed_time(e1) / K
    out["issue_ms_per_step"] = issue * 1e3 / K
    out["issue_hidden"] = bool(issue < 0.9)
    out["tok_s_normal"] = args.batch / (out["normal_ms_per_step"] / 1e3)
    out["tok_s_prequeued"] = args.batch / (out["prequeued_ms_per_step"] / 1e3)
    out["launches_per_step"] = rt.launches / (3 * K)
    rt.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
