"""bench.py's reference arm (CPU only: the reference's split_merge_kv + decode_attention, restated in
oracle/numerics_ref.py, on the host cores) prints the contract's JSON line: same metric / unit / config
keys as the kvpr arm, impl "reference", a cpu_baseline and an e2e object with zero copy bytes."""

from __future__ import annotations

import json
import subprocess
import sys

from .conftest import ROOT


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "2", "--warmup",
                          "1", "--model", "opt-125m", "--batch", "4", "--prompt", "64"], capture_output=True,
                         text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["metric"] == "decode_tokens_per_s" and d["unit"] == "tok/s"
    assert d["value"] > 0 and d["higher_is_better"] is True and d["steps"] == 2 and d["warmup"] == 1
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": "tok/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["batch"] == 4 and d["config"]["prompt_len"] == 64 and d["extrapolated"] is True
    assert len(d["run"]["splits_timed"]) == 2
