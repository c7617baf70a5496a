"""CLI contract (no GPU): byte-identical plan / calibrate / simulate / sweep documents vs the
reference CLI's stdout (tests/golden/scheduler_golden.json["cli"], produced by
running `kvoverlap plan|calibrate` on the same files), config validation and
the exit-code contract of pkg/src/kvoverlap/cli.py:45-48."""

from __future__ import annotations

import hashlib
import json

import pytest

from paper_2411_17089_b200 import cli

from .conftest import GOLDEN, ROOT

G = json.loads((GOLDEN / "scheduler_golden.json").read_text())["cli"]


@pytest.mark.parametrize("name", sorted(G))
def test_cli_output_identical_to_reference(name, capsys, monkeypatch, tmp_path):
    """plan / calibrate / simulate / sweep: stdout byte-identical to the reference CLI's, and simulate's
    --trace (sha256) and --metrics files too."""
    monkeypatch.chdir(ROOT)
    case = G[name]
    rc = cli.main([a.replace("@TMP", str(tmp_path)) for a in case["argv"]])
    out = capsys.readouterr().out
    assert rc == case["rc"] == 0
    assert out == case["stdout"]
    if "trace_sha256" in case:
        data = (tmp_path / "t.json").read_bytes()
        assert (len(data), hashlib.sha256(data).hexdigest()) == (case["trace_bytes"], case["trace_sha256"])
        assert (tmp_path / "m.csv").read_text() == case["metrics"]


def test_sweep_and_simulate_errors(tmp_path, capsys):
    cfg = _cfg(tmp_path, BASE)
    assert cli.main(["sweep", "--config", cfg, "--vary", "nope=1,2"]) == cli.EXIT_INVALID
    assert cli.main(["sweep", "--config", cfg, "--vary", "prompt_len"]) == cli.EXIT_INVALID
    assert cli.main(["sweep", "--config", cfg, "--vary", "prompt_len=8", "--policies", "kvpr:sideways"]) == \
        cli.EXIT_INVALID
    assert cli.main(["sweep", "--config", cfg, "--vary", "prompt_len=8", "--policies", "greedy"]) == cli.EXIT_INVALID
    assert cli.main(["sweep", "--config", cfg, "--vary", "prompt_len=x"]) == cli.EXIT_INVALID
    tight = dict(BASE, hardware=dict(BASE["hardware"], gpu_mem_budget_bytes=1e6))
    assert cli.main(["simulate", "--config", _cfg(tmp_path, tight)]) == cli.EXIT_BUDGET
    capsys.readouterr()


def _cfg(tmp_path, doc):
    p = tmp_path / "c.json"
    p.write_text(json.dumps(doc))
    return str(p)


BASE = {"model": {"preset": "opt-6.7b"}, "workload": {"batch_size": 4, "prompt_len": 8, "gen_len": 2},
        "hardware": {"gpu_flops": 1e15, "h2d_bw": 5e10, "d2h_bw": 5e10}}


def test_exit_codes(tmp_path, capsys):
    assert cli.main(["plan", "--config", _cfg(tmp_path, BASE)]) == cli.EXIT_OK
    bad = dict(BASE, model={"preset": "opt-6.7b", "bogus": 1})
    assert cli.main(["plan", "--config", _cfg(tmp_path, bad)]) == cli.EXIT_INVALID
    assert "unknown model keys" in capsys.readouterr().err
    assert cli.main(["plan", "--config", _cfg(tmp_path, {"model": BASE["model"]})]) == cli.EXIT_INVALID
    assert cli.main(["plan", "--config", _cfg(tmp_path, BASE), "--l", "-1"]) == cli.EXIT_INVALID
    assert cli.main(["plan"]) == cli.EXIT_INVALID  # argparse usage error is 1, not 2
    assert cli.main(["validate", "--cases", "0"]) == cli.EXIT_INVALID
    p = tmp_path / "x.json"
    p.write_text("{not json")
    assert cli.main(["plan", "--config", str(p)]) == cli.EXIT_INVALID
    budget = dict(BASE, hardware=dict(BASE["hardware"], gpu_mem_budget_bytes=1e6))
    assert cli.main(["run", "--config", _cfg(tmp_path, budget)]) == cli.EXIT_BUDGET


def test_plan_round_trip_through_file(tmp_path, capsys):
    out = tmp_path / "plan.json"
    assert cli.main(["plan", "--config", _cfg(tmp_path, BASE), "--out", str(out)]) == 0
    doc = json.loads(out.read_text())
    assert [d["seq_len"] for d in doc["decisions"]] == [9, 10]
    assert doc["mode"] == "row"


def test_plan_accepts_streamed_weights_like_the_reference(tmp_path, capsys):
    """policy.weights_resident=false is a valid plan config in the reference CLI (exit 0); only `run`
    decides how to execute it (streamed.StreamedRuntime)."""
    doc = dict(BASE, policy={"schedule": "column", "weights_resident": False, "granularity": "fine"})
    assert cli.main(["plan", "--config", _cfg(tmp_path, doc)]) == cli.EXIT_OK
    assert json.loads(capsys.readouterr().out)["mode"] == "column"


def test_run_rejects_plan_of_the_other_mode(tmp_path, capsys):
    """A plan made for the row schedule (t_act = 0) must not drive the column runtime, and vice versa."""
    out = tmp_path / "plan.json"
    assert cli.main(["plan", "--config", _cfg(tmp_path, BASE), "--out", str(out)]) == 0  # row (default)
    col = dict(BASE, policy={"schedule": "column"})
    assert cli.main(["run", "--config", _cfg(tmp_path, col), "--plan", str(out)]) == cli.EXIT_INVALID
    assert "plan mode 'row'" in capsys.readouterr().err
