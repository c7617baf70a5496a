"""CLI subcommands that execute on the B200: run (plan -> real decode, measured
report + trace in the reference schema) and validate (device exactness)."""

from __future__ import annotations

import json

import pytest

from paper_2411_17089_b200 import cli

from .conftest import ROOT

pytestmark = pytest.mark.gpu


def test_cli_run_reports_measured_pipeline(tmp_path, capsys):
    tr = tmp_path / "t.json"
    mx = tmp_path / "m.csv"
    rc = cli.main(["run", "--config", str(ROOT / "configs" / "opt125m_b4_s256.json"), "--trace", str(tr),
                   "--metrics", str(mx)])
    out = capsys.readouterr().out
    assert rc == 0, out
    kv = dict(line.split("=", 1) for line in out.strip().splitlines())
    assert float(kv["decode_throughput_tok_s"]) > 0 and 0 < float(kv["gpu_utilization"]) <= 1
    doc = json.loads(tr.read_text())
    assert {e["tid"] for e in doc} == {0, 1, 2}
    assert mx.read_text().splitlines()[0].startswith("policy,schedule")
    assert float(kv["simulated_makespan_s"]) > 0 and float(kv["replay_over_measured"]) > 0


@pytest.mark.parametrize("policy,workload", [
    ({"schedule": "column", "weights_resident": False, "granularity": "fine"}, {"num_batches": 2}),
    ({"schedule": "column"}, {"kv_bytes_per_element": 0.5625}),
    ({"schedule": "row"}, {}),
])
def test_cli_run_policies(tmp_path, capsys, policy, workload):
    """run executes what the config plans: streamed weights x 2 GPU batches (StreamedRuntime), 4-bit KV
    pages, the row schedule (X resident)."""
    doc = {"model": {"hidden_dim": 256, "num_layers": 2, "num_heads": 4, "ffn_dim": 1024},
           "workload": {"batch_size": 2, "prompt_len": 40, "gen_len": 3, **workload},
           "hardware": {"gpu_flops": 1e15, "h2d_bw": 5e10, "d2h_bw": 5e10}, "policy": policy}
    p = tmp_path / "c.json"
    p.write_text(json.dumps(doc))
    rc = cli.main(["run", "--config", str(p)])
    out = capsys.readouterr()
    assert rc == 0, out.err
    kv = dict(line.split("=", 1) for line in out.out.strip().splitlines() if "=" in line and " " not in line)
    assert float(kv["makespan_s"]) > 0


def test_cli_validate_device_exactness(capsys):
    rc = cli.main(["validate", "--cases", "4", "--seed", "1"])
    assert rc == 0, capsys.readouterr().err
