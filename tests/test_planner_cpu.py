"""Split points bit-exact with the reference (no GPU).

The product solver (paper_2411_17089_b200.scheduler) is compared, float for
float, with decisions the LIVE reference produced (tests/golden/
scheduler_golden.json, made by tests/golden/make_golden.py): the frozen
goldens of pkg/tests/test_scheduler.py:52-65, the 1000-config harness of
test_acceptance.py:73-108, full generation plans at every BASELINE config
under three profiles, and calibrate() fits.  The oracle scan
(oracle/scheduler_ref.py) is a second, independent route.
"""

from __future__ import annotations

import json
import math

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from oracle import scheduler_ref
from paper_2411_17089_b200 import costmodel as cm
from paper_2411_17089_b200 import hwprofile as hp
from paper_2411_17089_b200 import scheduler as sc

from .conftest import GOLDEN

GIB = 2**30
G = json.loads((GOLDEN / "scheduler_golden.json").read_text())


def _objs(c):
    spec = cm.ModelSpec(**c["spec"])
    wl = cm.WorkloadSpec(**c["wl"])
    prof = hp.HardwareProfile.from_dict(c["profile"])
    return spec, wl, prof


def _same(d, g):
    return (d.step, d.seq_len, d.recompute_len, d.t_total, d.t_recompute, d.t_kv, d.t_act) == (
        g["step"], g["seq_len"], g["l"], g["t_total"], g["t_recompute"], g["t_kv"], g["t_act"])


def test_frozen_goldens(criterion):
    # pkg/tests/test_scheduler.py:52-65
    spec = cm.ModelSpec(hidden_dim=4096, num_layers=1, num_heads=32, ffn_dim=16384)
    wl = cm.WorkloadSpec(batch_size=32, prompt_len=1023, gen_len=1)
    p = hp.HardwareProfile(gpu_flops=312e12, h2d_bandwidth=32 * GIB, d2h_bandwidth=32 * GIB)
    row = sc.solve_split(spec, wl, p, 1024, "row")
    col = sc.solve_split(spec, wl, p, 1024, "column")
    ok = (row.recompute_len == 706 and row.t_total == 0.004859370049641026 and row.t_act == 0.0
          and col.recompute_len == 706 and col.t_total == 0.010245722588703526
          and col.t_act == 0.0053863525390625 and col.t_kv == 0.004852294921875
          and col.t_recompute == 0.004859370049641026)
    criterion("S0", "frozen reference goldens l=706 (row/column) reproduced bit-exactly", ok)
    assert ok
    for c in G["frozen"]:
        spec, wl, prof = _objs(c)
        assert _same(sc.solve_split(spec, wl, prof, c["seq_len"], c["mode"]), c["solve"])
        assert _same(sc.scan_split(spec, wl, prof, c["seq_len"], c["mode"]), c["scan"])


def test_acceptance_1000_configs_bit_exact(criterion):
    bad = []
    for i, c in enumerate(G["acceptance02"]):
        spec, wl, prof = _objs(c)
        d = sc.solve_split(spec, wl, prof, c["seq_len"], c["mode"])
        if not _same(d, c["solve"]):
            bad.append(i)
    criterion("S1", f"solve_split bit-exact vs live reference on {len(G['acceptance02'])} random configs", not bad)
    assert not bad, bad[:10]


def test_baseline_plans_bit_exact(criterion):
    bad = []
    for c in G["plans"]:
        spec, wl, prof = _objs(c)
        plan = sc.plan_generation(spec, wl, prof, c["mode"])
        if len(plan.decisions) != len(c["decisions"]) or not all(
                _same(d, g) for d, g in zip(plan.decisions, c["decisions"])):
            bad.append((c["name"], c["profile_name"], c["mode"]))
        elif sc.plan_to_json(plan, spec, wl, prof) != c["json"]:
            bad.append((c["name"], "json"))
    criterion("S2", f"plan_generation bit-exact (l and times, JSON bytes) on {len(G['plans'])} BASELINE plans",
              not bad)
    assert not bad, bad


def test_appendix_a_values():
    # SURVEY.md Appendix A spot values: opt-6.7b b32 s1024 B200-guess column l=882, paper l=706
    by = {(c["name"], c["profile_name"], c["mode"]): c for c in G["plans"]}
    assert by[("opt6.7b_b32_s1024", "b200_guess", "column")]["decisions"][0]["l"] == 882
    assert by[("opt6.7b_b32_s1024", "paper", "column")]["decisions"][0]["l"] == 706
    assert by[("opt6.7b_b32_s1024", "paper", "row")]["decisions"][0]["l"] == 707


def test_layer_time_every_split_bit_exact():
    c = G["layer_time_cfg"]
    spec = cm.ModelSpec(**c["spec"])
    wl = cm.WorkloadSpec(**c["wl"])
    prof = hp.HardwareProfile.from_dict(c["profile"])
    for g in G["layer_time"]:
        lt = sc.layer_time(spec, wl, prof, c["seq_len"], g["split"], g["mode"])
        assert (lt.total, lt.t_recompute, lt.t_kv, lt.t_act) == (g["total"], g["t_recompute"], g["t_kv"], g["t_act"])


def test_latency_cases_bit_exact():
    for c in G["latency"]:
        spec, wl, prof = _objs(c)
        assert _same(sc.solve_split(spec, wl, prof, c["seq_len"], c["mode"]), c["solve"])
        assert _same(sc.scan_split(spec, wl, prof, c["seq_len"], c["mode"]), c["scan"])


def test_calibrate_matches_reference():
    for c in G["calibrate"]:
        recs = [hp.Measurement(k, float(s), float(e)) for k, s, e in c["records"]]
        res = hp.calibrate(recs)
        assert res.profile.to_dict() == c["profile"], c["name"]
        assert res.residual_rms == c["residual_rms"]


def test_calibrate_csv_round_trip(tmp_path):
    c = G["calibrate"][1]
    recs = [hp.Measurement(k, float(s), float(e)) for k, s, e in c["records"]]
    p = tmp_path / "m.csv"
    hp.write_measurements_csv(recs, str(p))
    back = hp.read_measurements_csv(str(p))
    assert back == recs
    assert hp.calibrate(back).profile.to_dict() == c["profile"]


def test_calibrate_errors():
    with pytest.raises(hp.CalibrationError, match="at least 2"):
        hp.calibrate([hp.Measurement("h2d", 1.0, 1.0)])
    recs = [hp.Measurement(k, 8.0, 1.0) for k in ("h2d", "h2d", "d2h", "d2h", "gemm", "gemm")]
    with pytest.raises(hp.CalibrationError, match="degenerate"):
        hp.calibrate(recs)
    with pytest.raises(ValueError):
        hp.Measurement("pcie", 1.0, 1.0)


# ---------------------------------------------------------------------------
# solver == independent scan oracle (test_scheduler.py:100-117 style)

@settings(max_examples=80, deadline=None)
@given(
    seq=st.integers(0, 300),
    b=st.integers(1, 64),
    hidden=st.sampled_from([256, 768, 1024, 4096]),
    v=st.sampled_from([1e11, 1e13, 312e12, 1391.2e12]),
    bw=st.sampled_from([2 * GIB, 32 * GIB, 55e9]),
    lat=st.sampled_from([0.0, 1e-6, 1e-5, 1e-4]),
    q=st.sampled_from([None, 2.0, 1.0, 0.5625]),
    mode=st.sampled_from(["row", "column"]),
)
def test_solver_matches_oracle_scan(seq, b, hidden, v, bw, lat, q, mode):
    spec = cm.ModelSpec(hidden_dim=hidden, num_layers=1, num_heads=8, ffn_dim=4 * hidden)
    wl = cm.WorkloadSpec(batch_size=b, prompt_len=seq, gen_len=1, kv_bytes_per_element=q)
    p = hp.HardwareProfile(gpu_flops=v, h2d_bandwidth=bw, d2h_bandwidth=bw, transfer_latency=lat)
    got = sc.solve_split(spec, wl, p, seq, mode)
    want = scheduler_ref.scan(hidden, b, 2, cm.kv_element_bytes(spec, wl), seq, v, 1.0, bw, lat, mode)
    assert (got.recompute_len, got.t_total, got.t_recompute, got.t_kv, got.t_act) == want


def test_degenerate_rates_and_zero_length():
    spec = cm.ModelSpec(hidden_dim=4096, num_layers=1, num_heads=32, ffn_dim=16384)
    wl = cm.WorkloadSpec(batch_size=32, prompt_len=1023, gen_len=1)
    slow = hp.HardwareProfile(gpu_flops=0.0, h2d_bandwidth=GIB, d2h_bandwidth=GIB)
    assert sc.solve_split(spec, wl, slow, 512, "row").recompute_len == 0
    fast = hp.HardwareProfile(gpu_flops=math.inf, h2d_bandwidth=GIB, d2h_bandwidth=GIB)
    assert sc.solve_split(spec, wl, fast, 512, "row").recompute_len == 512
    z = sc.solve_split(spec, wl, fast, 0, "row")
    assert z.recompute_len == 0 and z.t_total == 0.0


def test_plan_io_and_validation():
    spec = cm.ModelSpec(hidden_dim=1024, num_layers=1, num_heads=8, ffn_dim=4096)
    wl = cm.WorkloadSpec(batch_size=4, prompt_len=50, gen_len=3, kv_bytes_per_element=0.5625)
    p = hp.HardwareProfile(gpu_flops=1e14, h2d_bandwidth=GIB, d2h_bandwidth=GIB, transfer_latency=1e-6)
    plan = sc.plan_generation(spec, wl, p, "column")
    assert sc.import_plan(sc.export_plan(plan, spec, wl, p)) == (plan, spec, wl, p)
    doc = sc.export_plan(plan, spec, wl, p)
    with pytest.raises(ValueError, match="gen_len"):
        sc.import_plan(dict(doc, decisions=doc["decisions"][:1]))
    with pytest.raises(ValueError, match="out of range"):
        sc.import_plan(dict(doc, decisions=[dict(doc["decisions"][0], l=999)] + doc["decisions"][1:]))
    with pytest.raises(ValueError, match="mode"):
        sc.layer_time(spec, wl, p, 10, 0, "diagonal")
    with pytest.raises(ValueError):
        sc.SplitPlan(mode="spiral", decisions=())
    cp = sc.constant_plan(cm.WorkloadSpec(batch_size=1, prompt_len=2, gen_len=4), "column", 5)
    assert cp.splits == [3, 4, 5, 5]


def test_costmodel_tables():
    # pkg/tests/test_costmodel.py:55-65 per-layer KV at b32 s'=1024 fp16
    wl = cm.WorkloadSpec(batch_size=32, prompt_len=1023, gen_len=1)
    want = {"opt-6.7b": 536_870_912, "opt-13b": 671_088_640, "opt-30b": 939_524_096}
    for name, nbytes in want.items():
        assert cm.kv_cache_bytes(cm.opt_preset(name), wl, 1024) == nbytes
    spec = cm.opt_preset("opt-6.7b")
    assert cm.recompute_flops(spec, cm.WorkloadSpec(batch_size=32, prompt_len=1, gen_len=1), 882) == 1_894_080_577_536
    assert cm.groupwise_quant_bytes_per_element() == 0.5625
    with pytest.raises(ValueError, match="split"):
        cm.kv_remainder_bytes(spec, wl, 10, 11)
    with pytest.raises(ValueError, match="divisible"):
        cm.ModelSpec(hidden_dim=100, num_layers=1, num_heads=3, ffn_dim=4)
    with pytest.raises(ValueError, match="unknown preset"):
        cm.opt_preset("opt-175b")


def test_monotone_split(criterion):
    rng = np.random.default_rng(3)
    bad = 0
    for _ in range(30):
        spec = cm.ModelSpec(hidden_dim=int(rng.choice([1024, 4096])), num_layers=1, num_heads=8,
                            ffn_dim=4096)
        wl = cm.WorkloadSpec(batch_size=int(rng.integers(1, 65)), prompt_len=int(rng.integers(0, 1024)),
                             gen_len=int(rng.integers(2, 65)))
        p = hp.HardwareProfile(gpu_flops=float(rng.uniform(1e12, 5e14)),
                               h2d_bandwidth=float(rng.uniform(2, 64)) * GIB, d2h_bandwidth=GIB)
        ls = sc.plan_generation(spec, wl, p, "row").splits
        bad += ls != sorted(ls)
    assert bad == 0


def test_overlap_roofline_appendix_a():
    # T_roof(882) = 5.567 ms at OPT-6.7B b32 s'=1025, 55e9 B/s, 1391.2 TF/s
    spec = cm.opt_preset("opt-6.7b")
    wl = cm.WorkloadSpec(batch_size=32, prompt_len=1024, gen_len=1)
    t = sc.overlap_roofline(spec, wl, 1025, 882, 55e9, 1391.2e12)
    assert abs(t - 5.567e-3) < 1e-6


@settings(max_examples=60, deadline=None)
@given(
    seq=st.integers(0, 400),
    b=st.integers(1, 64),
    hidden=st.sampled_from([256, 768, 4096]),
    v=st.sampled_from([1e11, 1e13, 1.19e15, math.inf]),
    bw=st.sampled_from([2 * GIB, 55e9]),
    lat=st.sampled_from([0.0, 1e-5, 1e-3]),
    q=st.sampled_from([None, 1.0, 0.5625]),
)
def test_overlap_solver_matches_scan(seq, b, hidden, v, bw, lat, q):
    """Extension objective max(t_act + t_kv, t_rec): closed-form candidates == exhaustive scan."""
    spec = cm.ModelSpec(hidden_dim=hidden, num_layers=1, num_heads=8, ffn_dim=4 * hidden)
    wl = cm.WorkloadSpec(batch_size=b, prompt_len=seq, gen_len=1, kv_bytes_per_element=q)
    p = hp.HardwareProfile(gpu_flops=v, h2d_bandwidth=bw, d2h_bandwidth=bw, transfer_latency=lat)
    got = sc.solve_split_overlap(spec, wl, p, seq)
    best = min(range(seq + 1), key=lambda l: (sc.overlap_layer_time(spec, wl, p, seq, l).total, l))
    assert got.recompute_len == best
    assert got.t_total == sc.overlap_layer_time(spec, wl, p, seq, best).total


def test_overlap_mode_prefers_full_recompute_on_b200():
    # SURVEY.md Appendix A finding: with X chunked under K1, l = s' minimises the per-layer time
    spec = cm.opt_preset("opt-6.7b")
    wl = cm.WorkloadSpec(batch_size=32, prompt_len=1024, gen_len=2)
    p = hp.HardwareProfile(gpu_flops=1.19e15, h2d_bandwidth=55.3e9, d2h_bandwidth=55e9)
    assert [d.recompute_len for d in sc.plan_generation_overlap(spec, wl, p).decisions] == [1025, 1026]
