"""Config 1 (OPT-125M shape, b4, prompt 256, 16 tokens) through bench.run_config1 under runtime
variants selected by environment (read when the runtime is built): default, one DMA per layer (KVPR_DMA_GROUP=1) or per 2 / 3 layers,
zero-copy reads of the KV tail by the fused layer tail (KVPR_TAIL_ZC=r), zero-copy writes of the new X row / K,V page (w),
both, the unfused multi-kernel layer (KVPR_FUSED_TAIL=0).  One JSON line per variant and repeat.

    python tools/c1_modes.py [--reps 3] [--modes default,zc_r,...] > gpurun_out/c1_modes.jsonl
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402

MODES = {
    "default": {},
    "group1": {"KVPR_DMA_GROUP": "1"},
    "group2": {"KVPR_DMA_GROUP": "2"},
    "group3": {"KVPR_DMA_GROUP": "3"},
    "zc_r": {"KVPR_TAIL_ZC": "r"},
    "zc_w": {"KVPR_TAIL_ZC": "w"},
    "zc_rw": {"KVPR_TAIL_ZC": "rw"},
    "unfused": {"KVPR_FUSED_TAIL": "0"},
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--modes", default=",".join(MODES))
    ap.add_argument("--env", action="append", default=[],
                    help="extra variant as NAME:K=V[,K=V...] (e.g. tail116:KVPR_TAIL_CTAS=116,KVPR_DMA_GROUP=1)")
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    peaks = bench.load_peaks()
    modes = dict(MODES)
    for spec in args.env:
        name, _, kvs = spec.partition(":")
        modes[name] = dict(kv.split("=", 1) for kv in kvs.split(",") if kv)
    names = [n for n in args.modes.split(",") if n] + [spec.partition(":")[0] for spec in args.env]
    keys = set(k for m in modes.values() for k in m)
    for rep in range(args.reps):
        for name in names:
            for k in keys:
                os.environ.pop(k, None)
            os.environ.update(modes[name])
            r = bench.run_config1(None, dev, peaks)
            print(json.dumps({"mode": name, "rep": rep, "ms_per_step": round(r["ms_per_step"], 4),
                              "tok_s": round(r["value"], 1), "frac": round(r["overlap_roofline_frac"], 4),
                              "e2e_tok_s": round(r["e2e"]["value"], 1), "launches_per_step": r["launches_per_step"]}),
                  flush=True)


if __name__ == "__main__":
    main()
