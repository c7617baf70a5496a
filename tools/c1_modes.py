"""Config 1 (OPT-125M shape, b4, prompt 256, 16 tokens) through bench.run_config1 under runtime
variants selected by environment (read when the runtime is built): default, zero-copy reads of the
KV tail by the fused layer tail (KVPR_TAIL_ZC=r), zero-copy writes of the new X row / K,V page (w),
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
    "zc_r": {"KVPR_TAIL_ZC": "r"},
    "zc_w": {"KVPR_TAIL_ZC": "w"},
    "zc_rw": {"KVPR_TAIL_ZC": "rw"},
    "unfused": {"KVPR_FUSED_TAIL": "0"},
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--modes", default=",".join(MODES))
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    peaks = bench.load_peaks()
    keys = set(k for m in MODES.values() for k in m)
    for rep in range(args.reps):
        for name in args.modes.split(","):
            for k in keys:
                os.environ.pop(k, None)
            os.environ.update(MODES[name])
            r = bench.run_config1(None, dev, peaks)
            print(json.dumps({"mode": name, "rep": rep, "ms_per_step": round(r["ms_per_step"], 4),
                              "tok_s": round(r["value"], 1), "frac": round(r["overlap_roofline_frac"], 4),
                              "e2e_tok_s": round(r["e2e"]["value"], 1), "launches_per_step": r["launches_per_step"]}),
                  flush=True)


if __name__ == "__main__":
    main()
