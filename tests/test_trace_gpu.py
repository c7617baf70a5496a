"""Measured timelines (paper_2411_17089_b200.trace) of a real decode run:
schema of the reference's Chrome trace (pipesim/trace.py:30-43), and the
simulator's timeline invariants (engine.py:103-119) — lane exclusivity and
task-graph dependencies (graph.py:266-347) — hold on the measured data."""

from __future__ import annotations

import json

import pytest
import torch

from paper_2411_17089_b200 import trace
from paper_2411_17089_b200.runtime import KVPRRuntime
from paper_2411_17089_b200.weights import OPTConfig, OPTWeights

pytestmark = pytest.mark.gpu


def test_measured_trace_schema_and_invariants(tmp_path, criterion):
    cfg = OPTConfig(hidden=1024, layers=4, heads=8, ffn=4096, vocab=4096)
    b, S0, steps = 8, 300, 3
    w = OPTWeights.random(cfg, seed=0, device="cuda")
    prompt = torch.randint(0, cfg.vocab, (b, S0), generator=torch.Generator().manual_seed(0))
    rt = KVPRRuntime(w, b, S0 + steps + 1)
    first = rt.prefill(prompt)
    tr = trace.Tracer()
    rt.decode([150, 0, S0 + 3], tokens=first, trace=tr)
    torch.cuda.synchronize()
    rt.close()
    ents = tr.entries()
    kinds = {e.kind for e in ents}
    # step 2 has l = 0 (no activation loads / recompute), step 3 has l = s' (no KV load)
    assert {"load_activation_recompute", "load_cache", "compute_recompute", "compute_mha", "compute_ffn",
            "store_cache", "store_activation"} <= kinds
    assert not any(e.kind == "compute_recompute" and e.step == 2 for e in ents)
    assert not any(e.kind == "load_cache" and e.step == 3 for e in ents)
    bad = trace.check_invariants(ents, cfg.layers)
    doc = trace.export_trace(ents)
    assert all(set(d) == {"name", "cat", "ph", "ts", "dur", "pid", "tid"} and d["ph"] == "X" for d in doc)
    assert {d["tid"] for d in doc} == {0, 1, 2}
    p = tmp_path / "t.json"
    trace.write_trace(ents, str(p))
    assert json.loads(p.read_text()) == json.loads(json.dumps(doc))
    rep = trace.report(ents, tokens=b * steps)
    assert rep["makespan_s"] > 0 and 0 < rep["gpu_util"] <= 1
    criterion("T1", f"measured timeline satisfies lane exclusivity + DAG dependencies ({len(ents)} ops)", not bad)
    assert not bad, bad[:5]
