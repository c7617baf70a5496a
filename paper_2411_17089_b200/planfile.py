"""Plan documents: the JSON a planning run hands to the runtime (or to another process).

Wire format of the reference's plan export (/root/reference/pkg/src/kvoverlap/scheduler.py:233-288),
byte-identical for the same plan (`plan_to_json` is checked against the reference CLI's stdout in
tests/golden/scheduler_golden.json):

    {"mode", "model": ModelSpec fields, "workload": WorkloadSpec fields, "profile": HardwareProfile
     fields, "decisions": [{"step", "seq_len", "l", "t_total_s", "t_recomp_s", "t_kv_s", "t_act_s"}]}

`scheduler` re-exports these three functions, so `scheduler.export_plan` etc. keep the reference's
module layout.
"""

from __future__ import annotations

import json
from dataclasses import asdict

from .costmodel import ModelSpec, WorkloadSpec
from .hwprofile import HardwareProfile

# decision field  <->  document key (document order = reference order)
_KEYS = (("step", "step"), ("seq_len", "seq_len"), ("recompute_len", "l"), ("t_total", "t_total_s"),
         ("t_recompute", "t_recomp_s"), ("t_kv", "t_kv_s"), ("t_act", "t_act_s"))


def export_plan(plan, spec: ModelSpec, wl: WorkloadSpec, profile: HardwareProfile) -> dict:
    return {
        "mode": plan.mode,
        "model": asdict(spec),
        "workload": asdict(wl),
        "profile": profile.to_dict(),
        "decisions": [{key: getattr(dec, field) for field, key in _KEYS} for dec in plan.decisions],
    }


def import_plan(doc: dict):
    """Inverse of export_plan with the reference's checks: every l within [0, s'], one decision per
    generated token, steps numbered 1..gen_len with s' = prompt_len + step."""
    from .scheduler import SplitDecision, SplitPlan

    spec, wl = ModelSpec(**doc["model"]), WorkloadSpec(**doc["workload"])
    profile = HardwareProfile.from_dict(doc["profile"])
    rows = []
    for entry in doc["decisions"]:
        dec = SplitDecision(**{field: entry[key] for field, key in _KEYS})
        if dec.recompute_len < 0 or dec.recompute_len > dec.seq_len:
            raise ValueError(f"step {dec.step}: split {dec.recompute_len} out of range")
        rows.append(dec)
    plan = SplitPlan(mode=doc["mode"], decisions=tuple(rows))
    if len(rows) != wl.gen_len:
        raise ValueError("plan length does not match workload gen_len")
    for expect, dec in enumerate(rows, start=1):
        if (dec.step, dec.seq_len) != (expect, wl.prompt_len + expect):
            raise ValueError(f"plan step {expect} inconsistent with workload")
    return plan, spec, wl, profile


def plan_to_json(plan, spec: ModelSpec, wl: WorkloadSpec, profile: HardwareProfile) -> str:
    return json.dumps(export_plan(plan, spec, wl, profile), indent=2, sort_keys=True)
