"""paper_2411_17089_b200.pipesim against the live reference (no GPU).

tests/golden/pipesim_golden.json holds kvoverlap.pipesim's task graphs and
simulated timelines for 48 random configs (tests/golden/make_golden.py): every
task (kind, cost, deps, priority), every start / end and the report must come
out bit-identical.  Plus the reference's own simulator criteria
(/root/reference/pkg/tests/test_acceptance.py): 04 (simulated cache-ready time
== analytic layer model), 05b (fine weight loads never lose to coarse, with the
frozen witness makespans) and 06 (zero split == naive pipeline bit for bit).
"""

from __future__ import annotations

import json

import numpy as np
import pytest

from paper_2411_17089_b200 import pipesim as ps
from paper_2411_17089_b200.costmodel import ModelSpec, WorkloadSpec
from paper_2411_17089_b200.hwprofile import HardwareProfile
from paper_2411_17089_b200.scheduler import constant_plan, layer_time, plan_generation, solve_split

from .conftest import GOLDEN

GIB = 2**30
CASES = json.loads((GOLDEN / "pipesim_golden.json").read_text())


def _plan(c):
    spec, wl = ModelSpec(**c["spec"]), WorkloadSpec(**c["wl"])
    prof = HardwareProfile(**c["profile"])
    pol = ps.Policy(*c["policy"])
    plan = plan_generation(spec, wl, prof, pol.schedule)
    if [d.recompute_len for d in plan.decisions] != c["splits"]:
        assert len(set(c["splits"])) == 1, "golden plan is neither the solver's nor constant"
        plan = constant_plan(wl, pol.schedule, c["splits"][0])
    return spec, wl, prof, pol, plan


@pytest.mark.parametrize("n", range(len(CASES)))
def test_simulated_timeline_bit_identical_to_reference(n):
    c = CASES[n]
    spec, wl, prof, pol, plan = _plan(c)
    g = ps.build_task_graph(spec, wl, prof, plan, pol)
    got = [[t.kind.value, t.cost, list(t.deps), t.step, t.layer, t.batch, t.priority, t.part] for t in g.tasks]
    assert got == c["tasks"]
    tl, rep = ps.simulate(g, prof)
    assert [e.start for e in tl.entries] == c["start"]
    assert [e.end for e in tl.entries] == c["end"]
    assert [e.name for e in tl.entries] == c["names"]
    r = c["report"]
    assert (rep.makespan, rep.decode_throughput, rep.gpu_utilization, rep.peak_gpu_bytes) == (
        r["makespan"], r["decode_throughput"], r["gpu_utilization"], r["peak_gpu_bytes"])
    assert rep.breakdown == r["breakdown"]
    assert [list(x) for x in rep.utilization_timeline] == r["utilization_timeline"]


def test_golden_grid_covers_every_variant():
    seen = {(c["policy"][0], c["policy"][1], c["policy"][2], c["policy"][3]) for c in CASES}
    assert {p[0] for p in seen} == {"row", "column"}
    assert {p[3] for p in seen} == {True, False}
    assert {(p[2], p[3]) for p in seen} >= {("coarse", False), ("fine", False)}
    assert {c["wl"]["num_batches"] for c in CASES} == {1, 2, 3}
    assert any(max(c["splits"]) > c["wl"]["prompt_len"] for c in CASES)  # rebuilt decode positions


def test_criterion_04_simulated_layer_matches_analytic_model(criterion):
    """test_acceptance.py:150-183 on this restatement: the cache-ready time of a one-layer column
    simulation equals scheduler.layer_time (rel 1e-9)."""
    rng = np.random.default_rng(4)
    bad = []
    for case in range(100):
        h = int(rng.choice([256, 512, 1024, 2048]))
        spec = ModelSpec(hidden_dim=h, num_layers=1, num_heads=8, ffn_dim=4 * h)
        wl = WorkloadSpec(batch_size=int(rng.integers(1, 33)), prompt_len=int(rng.integers(16, 2049)), gen_len=1)
        prof = HardwareProfile(gpu_flops=float(rng.uniform(1e13, 5e14)),
                               h2d_bandwidth=float(rng.uniform(2, 64)) * GIB, d2h_bandwidth=32 * GIB,
                               transfer_latency=float(rng.choice([0.0, 1e-6, 1e-4])))
        s = wl.prompt_len + 1
        solved = solve_split(spec, wl, prof, s, "column", step=1).recompute_len
        for l in {solved, int(rng.integers(0, s + 1)), 0, s}:
            g = ps.build_task_graph(spec, wl, prof, constant_plan(wl, "column", l), ps.Policy("column", True))
            tl, _ = ps.simulate(g, prof)
            ready = max(e.end for e in tl.entries if e.kind in ("compute_recompute", "load_cache"))
            want = layer_time(spec, wl, prof, s, l, "column").total
            if abs(ready - want) > 1e-9 * want:
                bad.append((case, l, ready, want))
    criterion("P04", "pipesim restatement: simulated cache-ready time == analytic layer model (rel 1e-9)", not bad)
    assert not bad, bad[:5]


def test_criterion_05b_fine_never_loses_and_frozen_witness(criterion):
    """test_acceptance.py:223-262: fine-grained weight loads never lose to coarse; the reference's frozen
    witness makespans reproduce exactly."""
    spec = ModelSpec(hidden_dim=4096, num_layers=4, num_heads=32, ffn_dim=16384)
    prof = HardwareProfile(gpu_flops=3.12e14, h2d_bandwidth=32 * GIB, d2h_bandwidth=32 * GIB)
    bad = []
    for b in (1, 2, 4, 8, 16, 32):
        wl = WorkloadSpec(batch_size=b, prompt_len=256, gen_len=2, num_batches=4)
        plan = plan_generation(spec, wl, prof, "column")
        out = {gran: ps.simulate(ps.build_task_graph(spec, wl, prof, plan,
                                                     ps.Policy("column", True, gran, weights_resident=False)),
                                 prof)[1].makespan for gran in ("fine", "coarse")}
        if out["fine"] > out["coarse"]:
            bad.append((b, out))
    wspec = ModelSpec(hidden_dim=4096, num_layers=1, num_heads=32, ffn_dim=16384)
    wwl = WorkloadSpec(batch_size=32, prompt_len=1023, gen_len=1)
    wplan = plan_generation(wspec, wwl, prof, "row")
    wit = {gran: ps.simulate(ps.build_task_graph(wspec, wwl, prof, wplan,
                                                 ps.Policy("row", True, gran, weights_resident=False)),
                             prof)[1].makespan for gran in ("fine", "coarse")}
    ok = not bad and wit == {"fine": 0.008801563424439102, "coarse": 0.008808638552205128}
    criterion("P05b", "pipesim restatement: fine weight loads never lose to coarse; frozen witness exact", ok)
    assert ok, (bad, wit)


def test_criterion_06_zero_split_degenerates_to_naive():
    spec = ModelSpec(hidden_dim=64, num_layers=2, num_heads=4, ffn_dim=256)
    wl = WorkloadSpec(batch_size=2, prompt_len=8, gen_len=2, num_batches=2)
    prof = HardwareProfile(gpu_flops=1e12, h2d_bandwidth=GIB, d2h_bandwidth=GIB, transfer_latency=1e-6)
    for schedule in ("row", "column"):
        plan = constant_plan(wl, schedule, 0)
        a = ps.simulate(ps.build_task_graph(spec, wl, prof, plan, ps.Policy(schedule, False)), prof)
        b = ps.simulate(ps.build_task_graph(spec, wl, prof, plan, ps.Policy(schedule, True)), prof)
        assert a == b


def test_errors_match_reference():
    spec = ModelSpec(hidden_dim=64, num_layers=2, num_heads=4, ffn_dim=256)
    wl = WorkloadSpec(batch_size=2, prompt_len=8, gen_len=2)
    prof = HardwareProfile(gpu_flops=1e12, h2d_bandwidth=GIB, d2h_bandwidth=GIB)
    plan = constant_plan(wl, "row", 3)
    with pytest.raises(ValueError, match="plan mode"):
        ps.build_task_graph(spec, wl, prof, plan, ps.Policy("column"))
    with pytest.raises(ps.GpuMemoryBudgetError):
        ps.build_task_graph(spec, wl, prof, plan, ps.Policy("row"), gpu_mem_budget=1.0)
    with pytest.raises(ValueError):
        ps.Policy("diagonal")
    for engine in ps.available_engines():  # the reference's CSR form: task 0 waits for 1, 1 for 0
        with pytest.raises(ps.DependencyCycleError):
            ps.run_schedule([0, 0], [1.0, 1.0], [0, 0], [0, 1, 2], [1, 0], 3, engine=engine)
    with pytest.raises(ValueError):
        ps.simulate(ps.build_task_graph(spec, wl, prof, constant_plan(wl, "row", 0), ps.Policy("row")), prof,
                    engine="fortran")


def test_compiled_engine_bit_identical():
    """The compiled engine (kvpr_list_schedule, csrc/sched_engine.cu) schedules exactly like the Python one:
    every golden case's timeline and report, and 200 random DAGs with tied priorities and durations."""
    assert ps.available_engines() == ("py", "c") and ps.active_engine() == "c"
    for c in CASES:
        spec, wl, prof, pol, plan = _plan(c)
        g = ps.build_task_graph(spec, wl, prof, plan, pol)
        assert ps.simulate(g, prof, engine="py") == ps.simulate(g, prof, engine="c")
    rng = np.random.default_rng(5)
    for _ in range(200):
        n = int(rng.integers(0, 150))
        res = rng.integers(0, 3, size=n)
        dur = rng.integers(0, 4, size=n) * 0.25  # ties in completion times
        pri = rng.integers(0, 10, size=n)        # ties in priority: id breaks them
        deps = [rng.choice(i, size=int(rng.integers(0, min(i, 4) + 1)), replace=False) if i else np.empty(0, int)
                for i in range(n)]
        indptr = np.zeros(n + 1, dtype=np.int64)
        indptr[1:] = np.cumsum([len(d) for d in deps])
        idx = np.concatenate(deps).astype(np.int64) if n else np.empty(0, np.int64)
        a = ps.run_schedule(res, dur, pri, indptr, idx, 3, engine="py")
        b = ps.run_schedule(res, dur, pri, indptr, idx, 3, engine="c")
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
