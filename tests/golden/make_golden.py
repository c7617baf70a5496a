"""Generate the golden fixtures from the LIVE reference (run in the build
container only — /root/reference does not exist on the GPU box).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes
  scheduler_golden.json  solve_split / scan_split / plan_generation / layer_time
                         decisions of kvoverlap for: the frozen goldens of
                         test_scheduler.py:52-65, the 1000-config harness of
                         test_acceptance.py:73-108 (seed 20260816), the BASELINE
                         configs under the paper and B200-guess profiles
                         (SURVEY.md Appendix A), plus calibrate() fits.
  pipesim_golden.json    kvoverlap.pipesim timelines (every task's start / end) and
                         reports for row / column, recompute on / off, resident /
                         streamed (coarse, fine) weights, 1-3 GPU batches, with and
                         without transfer latency (pins paper_2411_17089_b200.pipesim).
  cli_small.json         a small streamed-weights config for the CLI cases (simulate --trace/--metrics, sweep)
  numerics_golden.npz    fp64 split_merge_kv / decode_attention / append_token_kv
                         outputs of kvoverlap.numerics on seeded small cases
                         (pins oracle/numerics_ref.py).
Floats are stored with repr round-trip (json) / raw fp64 (npz): bit-exact.
"""

from __future__ import annotations

import json
import math
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from kvoverlap import costmodel as rc  # noqa: E402
from kvoverlap import hwprofile as rh  # noqa: E402
from kvoverlap import numerics as rn  # noqa: E402
from kvoverlap import scheduler as rs  # noqa: E402

OUT = Path(__file__).resolve().parent
# the reference's shipped calibration sample (pkg/configs/measurements.csv), as data
SAMPLE = [("h2d", 16777216, 0.000503), ("h2d", 67108864, 0.001967), ("h2d", 268435456, 0.007826),
          ("h2d", 1073741824, 0.031262), ("d2h", 16777216, 0.000524), ("d2h", 67108864, 0.002041),
          ("d2h", 268435456, 0.008103), ("d2h", 1073741824, 0.032391), ("gemm", 1099511627776, 0.004405),
          ("gemm", 4398046511104, 0.017612), ("gemm", 17592186044416, 0.070442)]
GIB = 2**30


def dec(d):
    return {"step": d.step, "seq_len": d.seq_len, "l": d.recompute_len, "t_total": d.t_total,
            "t_recompute": d.t_recompute, "t_kv": d.t_kv, "t_act": d.t_act}


def case(spec, wl, prof, seq, mode, scan=True):
    c = {
        "spec": dict(hidden_dim=spec.hidden_dim, num_layers=spec.num_layers, num_heads=spec.num_heads,
                     ffn_dim=spec.ffn_dim, precision_bytes=spec.precision_bytes),
        "wl": dict(batch_size=wl.batch_size, prompt_len=wl.prompt_len, gen_len=wl.gen_len,
                   num_batches=wl.num_batches, kv_bytes_per_element=wl.kv_bytes_per_element),
        "profile": prof.to_dict(),
        "seq_len": seq,
        "mode": mode,
        "solve": dec(rs.solve_split(spec, wl, prof, seq, mode)),
    }
    if scan:
        c["scan"] = dec(rs.scan_split(spec, wl, prof, seq, mode))
    return c


def scheduler_cases():
    out = {"frozen": [], "acceptance02": [], "baseline": [], "plans": [], "layer_time": [], "calibrate": [],
           "latency": []}
    spec = rc.ModelSpec(hidden_dim=4096, num_layers=1, num_heads=32, ffn_dim=16384)
    wl = rc.WorkloadSpec(batch_size=32, prompt_len=1023, gen_len=1)
    prof = rh.HardwareProfile(gpu_flops=312e12, h2d_bandwidth=32 * GIB, d2h_bandwidth=32 * GIB)
    for mode in ("row", "column"):
        out["frozen"].append(case(spec, wl, prof, 1024, mode))

    rng = np.random.default_rng(20260816)
    for _ in range(1000):
        h = int(rng.choice([512, 1024, 2048, 4096, 5120, 7168]))
        sp = rc.ModelSpec(hidden_dim=h, num_layers=2, num_heads=8, ffn_dim=4 * h)
        w = rc.WorkloadSpec(batch_size=int(rng.integers(1, 65)), prompt_len=1, gen_len=1,
                            kv_bytes_per_element=[None, 2.0, 1.0, 0.5625][int(rng.integers(0, 4))])
        p = rh.HardwareProfile(gpu_flops=float(rng.uniform(1e12, 5e14)),
                               h2d_bandwidth=float(rng.uniform(1, 64)) * GIB, d2h_bandwidth=32 * GIB,
                               transfer_latency=float(rng.choice([0.0, 1e-6, 1e-4])))
        seq = int(rng.integers(0, 4097))
        mode = ("row", "column")[int(rng.integers(0, 2))]
        out["acceptance02"].append(case(sp, w, p, seq, mode, scan=False))

    # BASELINE configs: paper profile, B200-guess, B200-guess + 10us
    paper = rh.HardwareProfile(gpu_flops=312e12, h2d_bandwidth=32 * GIB, d2h_bandwidth=32 * GIB)
    guess = rh.HardwareProfile(gpu_flops=1391.2e12, h2d_bandwidth=55e9, d2h_bandwidth=55e9)
    guess_lat = rh.HardwareProfile(gpu_flops=1391.2e12, h2d_bandwidth=55e9, d2h_bandwidth=55e9,
                                   transfer_latency=1e-5)
    c1 = rc.ModelSpec(hidden_dim=768, num_layers=12, num_heads=12, ffn_dim=3072)
    cfgs = [
        ("opt125m_b4_s256", c1, rc.WorkloadSpec(batch_size=4, prompt_len=256, gen_len=16)),
        ("opt6.7b_b32_s1024", rc.opt_preset("opt-6.7b"), rc.WorkloadSpec(batch_size=32, prompt_len=1024, gen_len=32)),
        ("opt13b_b32_s1024", rc.opt_preset("opt-13b"), rc.WorkloadSpec(batch_size=32, prompt_len=1024, gen_len=32)),
        ("opt13b_b4_s1024", rc.opt_preset("opt-13b"), rc.WorkloadSpec(batch_size=4, prompt_len=1024, gen_len=32)),
        ("opt30b_b64_s2048", rc.opt_preset("opt-30b"), rc.WorkloadSpec(batch_size=64, prompt_len=2048, gen_len=32)),
    ] + [
        (f"opt6.7b_b32_s{s}", rc.opt_preset("opt-6.7b"), rc.WorkloadSpec(batch_size=32, prompt_len=s, gen_len=64))
        for s in (512, 2048, 4096, 8192)
    ]
    for name, sp, w in cfgs:
        for pname, p in (("paper", paper), ("b200_guess", guess), ("b200_guess_lat10us", guess_lat)):
            for mode in ("row", "column"):
                plan = rs.plan_generation(sp, w, p, mode)
                out["plans"].append({
                    "name": name, "profile_name": pname, "mode": mode,
                    "spec": {k: getattr(sp, k) for k in ("hidden_dim", "num_layers", "num_heads", "ffn_dim",
                                                          "precision_bytes")},
                    "wl": {k: getattr(w, k) for k in ("batch_size", "prompt_len", "gen_len", "num_batches",
                                                       "kv_bytes_per_element")},
                    "profile": p.to_dict(),
                    "decisions": [dec(d) for d in plan.decisions],
                    "json": rs.plan_to_json(plan, sp, w, p),
                })

    # layer_time at every split of a small config, both modes, with latency
    sp = rc.ModelSpec(hidden_dim=1024, num_layers=1, num_heads=8, ffn_dim=4096)
    w = rc.WorkloadSpec(batch_size=7, prompt_len=60, gen_len=1, kv_bytes_per_element=0.5625)
    p = rh.HardwareProfile(gpu_flops=2.5e14, h2d_bandwidth=25e9, d2h_bandwidth=20e9, transfer_latency=3e-6)
    for mode in ("row", "column"):
        for split in range(0, 62):
            lt = rs.layer_time(sp, w, p, 61, split, mode)
            out["layer_time"].append({"mode": mode, "split": split, "total": lt.total, "t_recompute": lt.t_recompute,
                                      "t_kv": lt.t_kv, "t_act": lt.t_act})
    out["layer_time_cfg"] = {"spec": {"hidden_dim": 1024, "num_layers": 1, "num_heads": 8, "ffn_dim": 4096},
                             "wl": {"batch_size": 7, "prompt_len": 60, "gen_len": 1, "kv_bytes_per_element": 0.5625},
                             "profile": p.to_dict(), "seq_len": 61}

    # latency-aware and degenerate profiles
    for lat in (5e-4, 1e-6, 1e-4):
        pl = rh.HardwareProfile(gpu_flops=312e12, h2d_bandwidth=32 * GIB, d2h_bandwidth=32 * GIB,
                                transfer_latency=lat)
        for mode in ("row", "column"):
            out["latency"].append(case(spec, wl, pl, 1024, mode))

    # calibrate(): the shipped sample CSV (values inlined) and a synthetic noisy set
    sample = SAMPLE
    rng = np.random.default_rng(5)
    synth = []
    for kind, rate, lat in (("h2d", 53e9, 8e-6), ("d2h", 55e9, 9e-6), ("gemm", 1.3e15, 2e-5)):
        for size in (2**24, 2**26, 2**28, 2**30) if kind != "gemm" else (1e12, 4e12, 16e12):
            synth.append((kind, float(size), lat + size / rate * (1 + 0.01 * rng.standard_normal())))
    for name, recs in (("sample_csv", sample), ("synthetic_b200", synth)):
        ms = [rh.Measurement(k, float(s), float(e)) for k, s, e in recs]
        res = rh.calibrate(ms)
        out["calibrate"].append({"name": name, "records": [list(r) for r in recs], "profile": res.profile.to_dict(),
                                 "residual_rms": res.residual_rms})
    return out


def pipesim_cases():
    """Simulated timelines of the live reference for a grid of policies / workloads / profiles."""
    from kvoverlap.pipesim import Policy, build_task_graph, simulate

    out = []
    rng = np.random.default_rng(17)
    profiles = [rh.HardwareProfile(gpu_flops=312e12, h2d_bandwidth=32 * GIB, d2h_bandwidth=32 * GIB),
                rh.HardwareProfile(gpu_flops=1391.2e12, h2d_bandwidth=55e9, d2h_bandwidth=51e9,
                                   transfer_latency=1e-6),
                rh.HardwareProfile(gpu_flops=2e13, h2d_bandwidth=8 * GIB, d2h_bandwidth=8 * GIB,
                                   transfer_latency=1e-4, gpu_efficiency=0.8)]
    for n in range(48):
        h = int(rng.choice([256, 1024, 4096]))
        sp = rc.ModelSpec(hidden_dim=h, num_layers=int(rng.integers(1, 4)), num_heads=8, ffn_dim=4 * h)
        wl = rc.WorkloadSpec(batch_size=int(rng.integers(1, 33)), prompt_len=int(rng.integers(4, 300)),
                             gen_len=int(rng.integers(1, 4)), num_batches=int(rng.integers(1, 4)),
                             kv_bytes_per_element=[None, 0.5625][int(rng.integers(0, 2))])
        prof = profiles[n % 3]
        pol = Policy(("row", "column")[n % 2], bool(rng.integers(0, 4)), ("coarse", "fine")[(n // 2) % 2],
                     bool((n // 4) % 2))
        if n % 5 == 4:  # constant plans, including splits past the prompt (rebuilt decode positions)
            plan = rs.constant_plan(wl, pol.schedule, int(rng.integers(0, wl.prompt_len + wl.gen_len + 1)))
        else:
            plan = rs.plan_generation(sp, wl, prof, pol.schedule)
        g = build_task_graph(sp, wl, prof, plan, pol)
        tl, rep = simulate(g, prof)
        out.append({
            "spec": {k: getattr(sp, k) for k in ("hidden_dim", "num_layers", "num_heads", "ffn_dim", "precision_bytes")},
            "wl": {k: getattr(wl, k) for k in ("batch_size", "prompt_len", "gen_len", "num_batches",
                                               "kv_bytes_per_element")},
            "profile": prof.to_dict(), "policy": [pol.schedule, pol.recompute, pol.granularity, pol.weights_resident],
            "splits": [d.recompute_len for d in plan.decisions],
            "tasks": [[t.kind.value, t.cost, list(t.deps), t.step, t.layer, t.batch, t.priority, t.part]
                      for t in g.tasks],
            "start": [e.start for e in tl.entries], "end": [e.end for e in tl.entries],
            "names": [e.name for e in tl.entries],
            "report": {"makespan": rep.makespan, "decode_throughput": rep.decode_throughput,
                       "gpu_utilization": rep.gpu_utilization, "breakdown": rep.breakdown,
                       "utilization_timeline": [list(x) for x in rep.utilization_timeline],
                       "peak_gpu_bytes": rep.peak_gpu_bytes},
        })
    return out


def numerics_cases():
    arrs = {}
    meta = []
    rng = np.random.default_rng(7)
    for i in range(24):
        heads = int(rng.choice([1, 2, 4]))
        d = int(rng.integers(1, 9))
        h = heads * d
        seq = int(rng.integers(1, 33))
        x = rng.standard_normal((seq, h))
        w_k, w_v, w_o = (rng.standard_normal((h, h)) for _ in range(3))
        q = rng.standard_normal(h)
        split = int(rng.integers(0, seq + 1))
        full = rn.build_kv(x, w_k, w_v, heads)
        suffix = rn.KVState(keys=full.keys[:, split:, :], values=full.values[:, split:, :])
        merged = rn.split_merge_kv(x, split, w_k, w_v, suffix)
        att = rn.decode_attention(q, merged, w_o)
        x_new = rng.standard_normal(h)
        grown = rn.append_token_kv(full, x_new, w_k, w_v)
        for k, v in dict(x=x, w_k=w_k, w_v=w_v, w_o=w_o, q=q, x_new=x_new, keys=merged.keys, values=merged.values,
                         att=att, grown_keys=grown.keys, grown_values=grown.values).items():
            arrs[f"c{i}_{k}"] = v
        meta.append({"i": i, "heads": heads, "split": split})
    arrs["meta"] = np.array(json.dumps(meta))
    return arrs


CLI_SMALL = {"model": {"hidden_dim": 768, "num_layers": 4, "num_heads": 12, "ffn_dim": 3072}, "workload": {"batch_size": 4, "prompt_len": 64, "gen_len": 2,
                                                          "num_batches": 2},
             "hardware": {"gpu_flops": 1.19e15, "h2d_bw": 55.3e9, "d2h_bw": 55.3e9, "transfer_latency_s": 2e-6},
             "policy": {"schedule": "column", "granularity": "fine", "weights_resident": False}}


def cli_cases():
    """stdout (and --trace / --metrics files) of the reference CLI (`kvoverlap plan | calibrate |
    simulate | sweep`) for configs shipped with this repo."""
    import contextlib
    import hashlib
    import io
    import tempfile

    from kvoverlap import cli as rcli

    root = OUT.parents[1]
    (OUT / "cli_small.json").write_text(json.dumps(CLI_SMALL, sort_keys=True) + "\n")
    big = str(root / "configs" / "opt6.7b_b32_s1024.json")
    small = str(OUT / "cli_small.json")
    tmp = Path(tempfile.mkdtemp())
    out = {}
    for name, argv in (
        ("plan_opt6.7b", ["plan", "--config", big]),
        ("plan_opt6.7b_l500", ["plan", "--config", big, "--l", "500"]),
        ("calibrate_sample", ["calibrate", "--measurements", str(OUT / "measurements_sample.csv")]),
        ("simulate_opt6.7b", ["simulate", "--config", big]),
        ("simulate_opt6.7b_l500", ["simulate", "--config", big, "--l", "500"]),
        ("simulate_small_files", ["simulate", "--config", small, "--trace", "@TMP/t.json", "--metrics", "@TMP/m.csv"]),
        ("sweep_prompt", ["sweep", "--config", big, "--vary", "prompt_len=512,2048",
                          "--policies", "naive,kvpr,kvpr:row,kvpr:fine:offloaded"]),
        ("sweep_h2d_bw", ["sweep", "--config", big, "--vary", "h2d_bw=25e9,64e9"]),
        ("sweep_small_batches", ["sweep", "--config", small, "--vary", "num_batches=1,3",
                                 "--policies", "kvpr,kvpr:coarse,naive:row:resident"]),
    ):
        buf = io.StringIO()
        real = [a.replace("@TMP", str(tmp)) for a in argv]
        with contextlib.redirect_stdout(buf):
            rc = rcli.main(real)
        case = {"argv": argv[:1] + [a.replace(str(root) + "/", "") for a in argv[1:]], "rc": rc,
                "stdout": buf.getvalue()}
        assert rc == 0, (name, rc)
        if "--trace" in argv:
            data = (tmp / "t.json").read_bytes()
            case["trace_sha256"], case["trace_bytes"] = hashlib.sha256(data).hexdigest(), len(data)
            case["metrics"] = (tmp / "m.csv").read_text()
        out[name] = case
    return out


def main():
    (OUT / "measurements_sample.csv").write_text(
        "kind,size,elapsed_s\n" + "".join(f"{k},{s},{e}\n" for k, s, e in SAMPLE))
    doc = scheduler_cases()
    doc["cli"] = cli_cases()
    (OUT / "scheduler_golden.json").write_text(json.dumps(doc, sort_keys=True) + "\n")
    (OUT / "pipesim_golden.json").write_text(json.dumps(pipesim_cases(), sort_keys=True) + "\n")
    np.savez_compressed(OUT / "numerics_golden.npz", **numerics_cases())
    print("wrote", OUT / "scheduler_golden.json", OUT / "numerics_golden.npz")


if __name__ == "__main__":
    main()
