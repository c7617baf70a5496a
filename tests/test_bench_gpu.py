"""bench.py end to end on the B200 in its N > 1 form: two ranks under torchrun (sharing cuda:0 and one
PCIe link: KVPR_BENCH_SHARE_GPU=1, gloo reductions -- NCCL refuses two ranks on one device) print ONE
JSON line from rank 0 with the whole-job value, n_gpus 2, each rank's timed window (they must overlap:
max over ranks of concurrent work), e2e and launches -- the driver's SCALE command, at reduced size."""

from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

from .conftest import ROOT

pytestmark = pytest.mark.gpu


def test_bench_two_ranks_json_line():
    env = dict(os.environ, KVPR_BENCH_SHARE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", "29517", str(ROOT / "bench.py"), "--gpus", "2", "--steps", "3", "--warmup", "3",
           "--model", "opt-125m", "--batch", "8", "--prompt", "128", "--no-cpu-baseline"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["metric"] == "decode_tokens_per_s" and d["value"] > 0 and d["steps"] == 3
    assert d["config"]["batch"] == 8 and d["config"]["batch_per_gpu"] == 4
    w = d["rank_windows"]
    assert [r["rank"] for r in w] == [0, 1] and all(r["batch"] == 4 for r in w)
    assert max(r["start_s"] for r in w) < min(r["end_s"] for r in w)  # the ranks' timed regions overlap
    assert d["gpu_launches"] > 0 and d["e2e"]["value"] > 0


def test_bench_one_gpu_json_contract():
    """The N = 1 line at reduced size carries every key of the contract: roofline (bound / achieved /
    peak / unit / frac / traffic), overlap roofline with the copy-stream measurement, cpu_baseline,
    e2e with its copy bytes, gpu_launches and the clocks sampled during the timed region."""
    cmd = [sys.executable, str(ROOT / "bench.py"), "--steps", "3", "--warmup", "3", "--model", "opt-125m", "--batch",
           "4", "--prompt", "128", "--no-alt", "--cpu-budget", "1"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    r = d["roofline"]
    assert r["bound"] in ("tensor", "hbm") and r["achieved"] > 0 and r["peak"] > 0 and r["frac"] > 0
    assert {"value", "unit", "cores", "kind", "sample"} <= set(d["cpu_baseline"])
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0 and d["clocks"]["sm_max_mhz"] > 0
    assert d["overlap_roofline"]["copy_stream"]["gbs_in_copy"] > 0
