"""The reference's acceptance gate (/root/reference/pkg/tests/test_acceptance.py), restated against
this package's cost model, scheduler and pipesim restatement with the reference's own frozen
constants -- golden vectors of the path's planning side, no GPU.  Criteria 02 / 04 / 05b / 06 live in
test_planner_cpu.py (S1) and test_pipesim_cpu.py (P04, P05b); 07's split-rebuild exactness in
test_oracle_cpu.py (oracle) and on the device in test_numerics_gpu.py / cli validate (N1)."""

from __future__ import annotations

import numpy as np
import pytest

from paper_2411_17089_b200.costmodel import ModelSpec, WorkloadSpec, kv_cache_bytes, opt_preset
from paper_2411_17089_b200.hwprofile import HardwareProfile, transfer_time
from paper_2411_17089_b200.pipesim import Policy, compare
from paper_2411_17089_b200.scheduler import plan_generation

GIB = 2**30

# pkg/configs/demo.json of the reference (OPT-6.7B, b32, prompt 1024, 8 tokens, 312 TFLOP/s, 32 GiB/s, row)
DEMO_SPEC = opt_preset("opt-6.7b")
DEMO_WL = WorkloadSpec(batch_size=32, prompt_len=1024, gen_len=8)
DEMO_PROFILE = HardwareProfile(gpu_flops=3.12e14, h2d_bandwidth=34359738368, d2h_bandwidth=34359738368)


def test_criterion_01_cache_footprints_and_transfer_times(criterion):
    """test_acceptance.py:47-70: fp16 cache bytes of the three presets at b32 x 1024 positions, and
    their 32 GiB/s transfer times within 0.5% of the paper's table."""
    profile = HardwareProfile(gpu_flops=1e15, h2d_bandwidth=32 * GIB, d2h_bandwidth=32 * GIB)
    wl = WorkloadSpec(batch_size=32, prompt_len=1023, gen_len=1)
    bad = []
    for preset, want_bytes, want_time in (("opt-6.7b", 536_870_912, 0.0156), ("opt-13b", 671_088_640, 0.0195),
                                          ("opt-30b", 939_524_096, 0.0273)):
        got = kv_cache_bytes(opt_preset(preset), wl, 1024)
        t = transfer_time(profile, got, "h2d")
        if got != want_bytes or abs(t - want_time) / want_time > 0.005 or not t < 1.0:
            bad.append((preset, got, t))
    assert criterion("A01", "cache footprints and 32 GiB/s transfer times of the three presets (reference "
                            "criterion 01)", not bad), bad


def test_criterion_03_split_monotone_across_generation(criterion):
    """test_acceptance.py:111-147 (seed 3, 100 cases): the per-step split never decreases as the cache
    grows (unique-optimum configurations, as the reference restricts them)."""
    rng = np.random.default_rng(3)
    bad = []
    for case in range(100):
        h = int(rng.choice([512, 1024, 2048, 4096]))
        spec = ModelSpec(hidden_dim=h, num_layers=2, num_heads=8, ffn_dim=4 * h)
        q = [None, 1.0, 0.5625][int(rng.integers(0, 3))]
        profile = HardwareProfile(gpu_flops=float(rng.uniform(1e12, 5e14)),
                                  h2d_bandwidth=float(rng.uniform(1, 64)) * GIB, d2h_bandwidth=32 * GIB,
                                  transfer_latency=float(rng.choice([0.0, 1e-6, 1e-4])))
        mode = ("row", "column")[int(rng.integers(0, 2))]
        if mode == "column" and profile.transfer_latency == 0 and q == 1.0:
            q = None  # flat column objective: the argmin is not unique (the reference's own exclusion)
        wl = WorkloadSpec(batch_size=int(rng.integers(1, 33)), prompt_len=int(rng.integers(0, 513)),
                          gen_len=int(rng.integers(1, 257)), kv_bytes_per_element=q)
        splits = [d.recompute_len for d in plan_generation(spec, wl, profile, mode).decisions]
        if any(b < a for a, b in zip(splits, splits[1:])):
            bad.append(case)
    assert criterion("A03", "per-step split monotone non-decreasing over generation (reference criterion 03, "
                            "100 cases)", not bad), bad


def test_criterion_05a_recompute_never_loses_when_transfer_bound(criterion):
    """test_acceptance.py:186-220 (seed 55, 40 cases): the KVPR pipeline never has a longer simulated
    makespan than the naive one when the decode is transfer-bound."""
    rng = np.random.default_rng(55)
    bad = []
    for case in range(40):
        h = int(rng.choice([1024, 2048, 4096]))
        spec = ModelSpec(hidden_dim=h, num_layers=int(rng.integers(1, 5)), num_heads=8, ffn_dim=4 * h)
        wl = WorkloadSpec(batch_size=int(rng.integers(8, 65)), prompt_len=int(rng.integers(512, 4096)),
                          gen_len=int(rng.integers(1, 5)), num_batches=int(rng.integers(1, 3)))
        profile = HardwareProfile(gpu_flops=float(rng.uniform(1e14, 5e14)),
                                  h2d_bandwidth=float(rng.uniform(8, 64)) * GIB, d2h_bandwidth=32 * GIB,
                                  transfer_latency=float(rng.choice([0.0, 1e-6])))
        mode = ("row", "column")[int(rng.integers(0, 2))]
        rows = compare(spec, wl, profile, [("naive", Policy(mode, False)), ("kvpr", Policy(mode, True))])
        if rows[1]["makespan_s"] > rows[0]["makespan_s"]:
            bad.append((case, mode))
    assert criterion("A05a", "recomputation never loses to naive when transfer-bound (reference criterion 05a, "
                             "40 cases)", not bad), bad


def test_criteria_08_09_10_demo_frozen_values(criterion):
    """test_acceptance.py:331-397: on the reference's demo config, the simulated GPU utilisation, the
    4-bit-cache throughput and the naive-vs-KVPR speedup reproduce the reference's frozen floats
    exactly (speedup at rel 1e-12, as there)."""
    pol = [("naive", Policy("row", False)), ("kvpr", Policy("row", True))]
    rows = compare(DEMO_SPEC, DEMO_WL, DEMO_PROFILE, pol)
    wl4 = WorkloadSpec(batch_size=32, prompt_len=1024, gen_len=8, kv_bytes_per_element=0.5625)
    tp16 = compare(DEMO_SPEC, DEMO_WL, DEMO_PROFILE, pol[1:])[0]["throughput_tok_s"]
    tp4 = compare(DEMO_SPEC, wl4, DEMO_PROFILE, pol[1:])[0]["throughput_tok_s"]
    checks = {
        "08 naive util": rows[0]["gpu_util"] == 0.0027415906225959027,
        "08 kvpr util": rows[1]["gpu_util"] == 1.0,
        "09 fp16 tput": tp16 == 203.12631734187744,
        "09 kv4 tput": tp4 == 362.19613267549335 and tp4 > tp16,
        "10 naive makespan": rows[0]["makespan_s"] == 4.017621156945847,
        "10 kvpr makespan": rows[1]["makespan_s"] == 1.2602995187922008,
        "10 speedup": rows[1]["speedup_vs_first"] == pytest.approx(3.1878304300204015, rel=1e-12),
    }
    bad = [k for k, v in checks.items() if not v]
    assert criterion("A08-10", "demo config: utilisation lift, 4-bit cache throughput, 3.19x speedup -- the "
                               "reference's frozen values reproduced exactly (criteria 08 / 09 / 10)", not bad), bad
