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


def test_cli_validate_device_exactness(capsys):
    rc = cli.main(["validate", "--cases", "4", "--seed", "1"])
    assert rc == 0, capsys.readouterr().err
