"""Operator front end (§8f rank 4), mirroring ``kvoverlap``'s CLI contract
(/root/reference/pkg/src/kvoverlap/cli.py): one JSON config with
model / workload / hardware / policy sections (unknown keys rejected,
cli.py:73-164), plan JSON on stdout or --out, exit codes 0 ok, 1 invalid
input, 2 GPU memory budget exceeded, 3 validation failure (cli.py:45-48).

    python -m paper_2411_17089_b200 plan      --config cfg.json [--l N] [--out plan.json]
    python -m paper_2411_17089_b200 simulate  --config cfg.json [--plan p.json | --l N] [--trace t.json] [--metrics m.csv]
    python -m paper_2411_17089_b200 sweep     --config cfg.json --vary AXIS=V1,V2 [--policies naive,kvpr:column]
    python -m paper_2411_17089_b200 calibrate --measurements m.csv
    python -m paper_2411_17089_b200 profile   [--hidden 4096 --batch 32] [--out m.csv]   (GPU)
    python -m paper_2411_17089_b200 run       --config cfg.json [--plan plan.json] [--trace t.json] (GPU)
    python -m paper_2411_17089_b200 validate  [--cases N] [--seed S]                       (GPU)

`plan` / `calibrate` / `simulate` / `sweep` print byte-identical documents to
the reference's for the same config (simulate / sweep through the pipesim
restatement; its --trace / --metrics files are byte-identical too).  `run` executes the plan on the B200 (random-init weights,
synthetic prompt) instead of simulating it and prints the reference's
`key=value` report style with measured numbers.  An optional "runtime"
section adds {"seed", "weights_std", "chunks", "device"}.
"""

from __future__ import annotations

import argparse
import copy
import json
import logging
import os
import re
import sys
from dataclasses import dataclass

from .costmodel import ModelSpec, WorkloadSpec, opt_preset
from .hwprofile import HardwareProfile, calibrate, profile_to_json, read_measurements_csv
from .pipesim import GpuMemoryBudgetError  # the reference's class (graph.py:70), raised by the residency check
from .scheduler import SplitPlan, constant_plan, import_plan, plan_generation, plan_to_json

log = logging.getLogger("paper_2411_17089_b200")

EXIT_OK, EXIT_INVALID, EXIT_BUDGET, EXIT_VALIDATION = 0, 1, 2, 3


class ConfigError(ValueError):
    """Configuration file or flag value is invalid."""


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # argparse would exit 2, which the contract reserves
        raise ConfigError(message)


@dataclass(frozen=True)
class Setup:
    spec: ModelSpec
    wl: WorkloadSpec
    profile: HardwareProfile
    schedule: str
    recompute: bool
    budget: float | None
    runtime: dict
    weights_resident: bool = True
    granularity: str = "coarse"


def _only(section: str, given: dict, allowed) -> None:
    extra = sorted(set(given) - set(allowed))
    if extra:
        raise ConfigError(f"unknown {section} keys: {', '.join(extra)}")


def _sec(doc, name, required):
    if name not in doc:
        if required:
            raise ConfigError(f"config missing required section {name!r}")
        return {}
    if not isinstance(doc[name], dict):
        raise ConfigError(f"config section {name!r} must be an object")
    return doc[name]


_WORKLOAD_AXES = ("batch_size", "num_batches", "prompt_len", "gen_len", "kv_bytes_per_element")
_HARDWARE_AXES = ("gpu_flops", "h2d_bw", "d2h_bw", "transfer_latency_s", "gpu_efficiency")


def load_config_doc(path: str) -> dict:
    try:
        with open(path) as fh:
            doc = json.load(fh)
    except json.JSONDecodeError as exc:
        raise ConfigError(f"{path}: not valid JSON ({exc})") from exc
    if not isinstance(doc, dict):
        raise ConfigError(f"{path}: config must be a JSON object")
    _only("config", doc, ("model", "workload", "hardware", "policy", "runtime"))
    return doc


def load_config(path: str) -> Setup:
    return setup_from_doc(load_config_doc(path))


def setup_from_doc(doc: dict) -> Setup:
    try:
        m = _sec(doc, "model", True)
        fields = ("hidden_dim", "num_layers", "num_heads", "ffn_dim", "precision_bytes")
        _only("model", m, fields + ("preset",))
        if "preset" in m:
            base = opt_preset(m["preset"])
            spec = ModelSpec(**{**{f: getattr(base, f) for f in fields}, **{k: v for k, v in m.items() if k != "preset"}})
        else:
            missing = [f for f in fields[:-1] if f not in m]
            if missing:
                raise ConfigError(f"model section missing: {', '.join(missing)}")
            spec = ModelSpec(**m)
        w = _sec(doc, "workload", True)
        _only("workload", w, _WORKLOAD_AXES)
        wl = WorkloadSpec(**w)
        hw = _sec(doc, "hardware", True)
        _only("hardware", hw, _HARDWARE_AXES + ("gpu_mem_budget_bytes",))
        for k in ("gpu_flops", "h2d_bw", "d2h_bw"):
            if k not in hw:
                raise ConfigError(f"hardware section missing {k!r}")
        prof = HardwareProfile(gpu_flops=hw["gpu_flops"], h2d_bandwidth=hw["h2d_bw"], d2h_bandwidth=hw["d2h_bw"],
                               transfer_latency=hw.get("transfer_latency_s", 0.0),
                               gpu_efficiency=hw.get("gpu_efficiency", 1.0))
        pol = _sec(doc, "policy", False)
        _only("policy", pol, ("schedule", "recompute", "granularity", "weights_resident"))
        rec = pol.get("recompute", "on")
        if isinstance(rec, str):
            if rec not in ("on", "off"):
                raise ConfigError("policy.recompute must be 'on' or 'off'")
            rec = rec == "on"
        if pol.get("granularity", "coarse") not in ("coarse", "fine"):
            raise ConfigError("policy.granularity must be 'coarse' or 'fine'")
        schedule = pol.get("schedule", "row")
        if schedule not in ("row", "column"):
            raise ConfigError("policy.schedule must be 'row' or 'column'")
        rt = _sec(doc, "runtime", False)
        _only("runtime", rt, ("seed", "weights_std", "chunks", "device"))
    except ConfigError:
        raise
    except (ValueError, TypeError) as exc:
        raise ConfigError(str(exc)) from exc
    return Setup(spec, wl, prof, schedule, bool(rec), hw.get("gpu_mem_budget_bytes"), rt,
                 bool(pol.get("weights_resident", True)), pol.get("granularity", "coarse"))


def _plan(s: Setup, l_override: int | None) -> SplitPlan:
    if l_override is not None:
        if l_override < 0:
            raise ConfigError("--l must be nonnegative")
        return constant_plan(s.wl, s.schedule, l_override)
    if not s.recompute:
        return constant_plan(s.wl, s.schedule, 0)
    return plan_generation(s.spec, s.wl, s.profile, s.schedule)


def _out(text: str, path: str | None) -> None:
    if path:
        with open(path, "w") as fh:
            fh.write(text)
    else:
        sys.stdout.write(text)


def cmd_plan(a) -> int:
    s = load_config(a.config)
    _out(plan_to_json(_plan(s, a.l), s.spec, s.wl, s.profile) + "\n", a.out)
    return EXIT_OK


def _sim_policy(s: Setup):
    from .pipesim import Policy

    return Policy(schedule=s.schedule, recompute=s.recompute, granularity=s.granularity,
                  weights_resident=s.weights_resident)


def _import_plan_for(s: Setup, path: str) -> SplitPlan:
    with open(path) as fh:
        doc = json.load(fh)
    plan, spec, wl, prof = import_plan(doc)
    if (spec, wl, prof) != (s.spec, s.wl, s.profile):
        raise ConfigError("--plan document does not match the config")
    return plan


def cmd_simulate(a) -> int:
    """The reference's prediction for one policy (cli.py:195-230): task DAG + list scheduler
    (pipesim restatement), `key=value` report, optional Chrome trace and metrics CSV."""
    from . import pipesim

    s = load_config(a.config)
    if a.l is not None:
        plan = _plan(s, a.l)
    elif a.plan:
        plan = _import_plan_for(s, a.plan)
    else:
        plan = _plan(s, None)
    policy = _sim_policy(s)
    graph = pipesim.build_task_graph(s.spec, s.wl, s.profile, plan, policy, s.budget)
    timeline, rep = pipesim.simulate(graph, s.profile)
    label = "kvpr" if policy.recompute else "naive"
    lines = [f"policy={label} schedule={policy.schedule} granularity={policy.granularity} "
             f"recompute={'on' if policy.recompute else 'off'} weights_resident={policy.weights_resident}",
             f"tasks={len(graph)}", f"makespan_s={rep.makespan!r}", f"throughput_tok_s={rep.decode_throughput!r}",
             f"gpu_utilization={rep.gpu_utilization!r}", f"peak_gpu_bytes={rep.peak_gpu_bytes!r}"]
    lines += [f"breakdown.{k}={v!r}" for k, v in rep.breakdown.items()]
    _out("".join(x + "\n" for x in lines), a.out)
    if a.trace:
        pipesim.write_trace(timeline, a.trace)
    if a.metrics:
        with open(a.metrics, "w") as fh:
            pipesim.write_metrics_csv([pipesim.metrics_row(label, policy, rep)], fh)
    return EXIT_OK


_POLICY_MODIFIERS = {"row": ("schedule", "row"), "column": ("schedule", "column"),
                     "coarse": ("granularity", "coarse"), "fine": ("granularity", "fine"),
                     "resident": ("weights_resident", True), "offloaded": ("weights_resident", False)}


def parse_policy_token(token: str, base):
    """'naive' / 'kvpr' plus ':'-separated modifiers over the config's policy (cli.py:243-262)."""
    from .pipesim import Policy

    head, *mods = token.strip().split(":")
    if head not in ("naive", "kvpr"):
        raise ConfigError(f"unknown policy {head!r} (use naive or kvpr)")
    values = {"recompute": head == "kvpr", "schedule": base.schedule, "granularity": base.granularity,
              "weights_resident": base.weights_resident}
    for mod in mods:
        if mod not in _POLICY_MODIFIERS:
            raise ConfigError(f"unknown policy modifier {mod!r}")
        field_, value = _POLICY_MODIFIERS[mod]
        values[field_] = value
    return token.strip(), Policy(**values)


def _number(text: str):
    if re.fullmatch(r"[+-]?\d+", text):
        return int(text)
    try:
        return float(text)
    except ValueError as exc:
        raise ConfigError(f"not a number: {text!r}") from exc


def parse_axis(vary: str):
    if "=" not in vary:
        raise ConfigError("--vary expects AXIS=V1,V2,...")
    axis, _, rest = vary.partition("=")
    axis = axis.strip()
    values = [v for v in (x.strip() for x in rest.split(",")) if v]
    if not values:
        raise ConfigError("--vary axis has no values")
    if axis not in _WORKLOAD_AXES and axis not in _HARDWARE_AXES:
        raise ConfigError(f"unknown sweep axis {axis!r}; known: {', '.join(_WORKLOAD_AXES + _HARDWARE_AXES)}")
    return axis, [_number(v) for v in values]


_SWEEP_COLS = ("policy", "schedule", "granularity", "recompute", "makespan_s", "throughput_tok_s", "gpu_util",
               "peak_gpu_bytes", "speedup_vs_first")


def cmd_sweep(a) -> int:
    """One axis across policies, one CSV row per (value, policy) (cli.py:287-318)."""
    from . import pipesim

    doc = load_config_doc(a.config)
    base = _sim_policy(setup_from_doc(doc))
    axis, values = parse_axis(a.vary)
    policies = [parse_policy_token(t, base) for t in a.policies.split(",") if t.strip()]
    if not policies:
        raise ConfigError("--policies is empty")
    section = "workload" if axis in _WORKLOAD_AXES else "hardware"
    rows = [",".join(pipesim.cell(c) for c in ("axis", "value") + _SWEEP_COLS)]
    for value in values:
        point = copy.deepcopy(doc)
        point.setdefault(section, {})[axis] = value
        s = setup_from_doc(point)
        for row in pipesim.compare(s.spec, s.wl, s.profile, policies, s.budget):
            rows.append(",".join(pipesim.cell(c) for c in [axis, value] + [row[k] for k in _SWEEP_COLS]))
    _out("".join(r + "\n" for r in rows), a.out)
    return EXIT_OK


def cmd_calibrate(a) -> int:
    _out(profile_to_json(calibrate(read_measurements_csv(a.measurements))) + "\n", a.out)
    return EXIT_OK


def cmd_profile(a) -> int:
    from . import profiler
    from .hwprofile import write_measurements_csv

    res, recs = profiler.measure(a.hidden, a.batch)
    if a.out:
        write_measurements_csv(recs, a.out)
    sys.stdout.write(profile_to_json(res) + "\n")
    return EXIT_OK


def _device_bytes(s: Setup, capacity: int) -> float:
    h, L, f, b = s.spec.hidden_dim, s.spec.num_layers, s.spec.ffn_dim, s.wl.batch_size
    resident_layers = L if s.weights_resident and s.wl.num_batches == 1 else 2  # streamed: two layer slots
    weights = resident_layers * (4 * h * h + 2 * h * f) * 2 + 2 * 50272 * h * 2
    buffers = 2 * capacity * 3 * b * h * 2 + b * 50272 * 4
    return float(weights + buffers)


def cmd_run(a) -> int:
    import torch

    from . import trace as tr
    from .runtime import KVPRRuntime
    from .weights import OPTConfig, OPTWeights

    s = load_config(a.config)
    if a.plan:
        with open(a.plan) as fh:
            plan, pspec, pwl, _ = import_plan(json.load(fh))
        if (pspec, pwl) != (s.spec, s.wl):
            raise ConfigError("plan context does not match the config")
        if plan.mode != s.schedule:
            raise ConfigError(f"plan mode {plan.mode!r} does not match policy.schedule {s.schedule!r}")
    else:
        plan = _plan(s, a.l)
    cap = s.wl.prompt_len + s.wl.gen_len + 1
    need = _device_bytes(s, cap)
    if s.budget is not None and need > s.budget:
        raise GpuMemoryBudgetError(f"estimated device residency {need:.0f} B exceeds budget {s.budget:.0f} B")
    rt_cfg = s.runtime
    dev = torch.device(rt_cfg.get("device", "cuda:0"))
    cfg = OPTConfig(s.spec.hidden_dim, s.spec.num_layers, s.spec.num_heads, s.spec.ffn_dim,
                    max_pos=max(2048, cap + 8))
    w = OPTWeights.random(cfg, seed=int(rt_cfg.get("seed", 0)), device=dev, std=float(rt_cfg.get("weights_std", 0.02)))
    prompt = torch.randint(0, cfg.vocab, (s.wl.batch_size, s.wl.prompt_len),
                           generator=torch.Generator().manual_seed(int(rt_cfg.get("seed", 0)) + 1))
    kv_bits = _kv_bits(s)
    if not s.weights_resident or s.wl.num_batches > 1:
        return _run_streamed(a, s, plan, w, cap, dev, need)
    # the row schedule keeps X resident in HBM (t_act = 0 in its plan); column streams X over PCIe
    rt = KVPRRuntime(w, s.wl.batch_size, cap, device=dev, chunks=int(rt_cfg.get("chunks", 4)),
                     x_resident=s.schedule == "row", kv_bits=kv_bits)
    first = rt.prefill(prompt)
    tracer = tr.Tracer()
    rt.decode(plan.splits, tokens=first, trace=tracer)
    torch.cuda.synchronize(dev)
    ents = tracer.entries()
    rep = tr.report(ents, s.wl.batch_size * s.wl.gen_len)
    rt.close()
    if a.trace:
        tr.write_trace(ents, a.trace)
    if a.metrics:
        with open(a.metrics, "w") as fh:
            tr.write_metrics_csv([tr.metrics_row("kvpr" if s.recompute else "naive", rep, s.schedule, need)], fh)
    lines = [f"makespan_s={rep['makespan_s']!r}", f"decode_throughput_tok_s={rep['throughput_tok_s']!r}",
             f"gpu_utilization={rep['gpu_util']!r}", f"peak_gpu_bytes={need!r}",
             f"splits={','.join(str(x) for x in plan.splits)}"]
    lines += [f"busy_{k}={v!r}" for k, v in sorted(rep["breakdown"].items())]
    # the reference's prediction for the same plan and profile (pipesim restatement), §8f rank 2
    cmp = tr.compare_with_model(ents, s.spec, s.wl, s.profile, plan, s.schedule)
    lines += [f"simulated_makespan_s={cmp['makespan']['simulated_s']!r}",
              f"measured_over_simulated={cmp['makespan']['measured_over_simulated']!r}",
              f"replay_over_measured={cmp['makespan']['replay_over_measured']!r}"]
    sys.stdout.write("\n".join(lines) + "\n")
    return EXIT_OK


def _kv_bits(s: Setup) -> int | None:
    """fp16 pages for q = p (or None); 4-bit groupwise pages for q = 0.5625 (costmodel.py:109-118)."""
    q = s.wl.kv_bytes_per_element
    if q is None or q == s.spec.precision_bytes:
        return None
    if q == 0.5625:
        return 4
    raise ConfigError(f"workload.kv_bytes_per_element={q!r}: the B200 runtime stores fp16 pages or 4-bit "
                      "groupwise pages (0.5625)")


def _run_streamed(a, s: Setup, plan: SplitPlan, w, cap: int, dev, need: float) -> int:
    """policy.weights_resident=false or num_batches > 1: the throughput-oriented column schedule with
    layer weights streamed from host (streamed.StreamedRuntime, §8f rank 1).  Timed with CUDA events;
    it has no per-task trace, so --trace / --metrics are rejected."""
    import torch

    from .streamed import StreamedRuntime

    if s.schedule != "column":
        raise ConfigError("streamed weights / num_batches > 1 run the column schedule (policy.schedule='column')")
    if _kv_bits(s) is not None:
        raise ConfigError("streamed weights run fp16 KV pages")
    if a.trace or a.metrics:
        raise ConfigError("--trace / --metrics need resident weights (the streamed runtime has no task trace)")
    K = s.wl.num_batches
    g = torch.Generator().manual_seed(int(s.runtime.get("seed", 0)) + 1)
    prompts = [torch.randint(0, w.cfg.vocab, (s.wl.batch_size, s.wl.prompt_len), generator=g) for _ in range(K)]
    rt = StreamedRuntime(w, s.wl.batch_size, K, cap, device=dev, granularity=s.granularity,
                         chunks=int(s.runtime.get("chunks", 4)))
    first = rt.prefill(prompts)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(rt.cs)
    rt.decode(plan.splits, tokens=first)
    e1.record(rt.cs)
    torch.cuda.synchronize(dev)
    rt.close()
    makespan = e0.elapsed_time(e1) / 1e3
    lines = [f"makespan_s={makespan!r}",
             f"decode_throughput_tok_s={s.wl.batch_size * K * s.wl.gen_len / makespan!r}",
             f"peak_gpu_bytes={need!r}", f"splits={','.join(str(x) for x in plan.splits)}",
             f"weights=streamed granularity={s.granularity} num_batches={K}"]
    sys.stdout.write("\n".join(lines) + "\n")
    return EXIT_OK


def run_validation_cases(seed: int, cases: int) -> list[str]:
    """Randomized split/merge exactness on the device (cli.py:343-377 analogue); returns failure lines.

    Per case: K1-rebuilt pages == the prefill's stored pages, bit for bit, and the decode output is
    identical for every split, on randomized small geometries."""
    import random

    import torch

    from . import kernels
    from .runtime import KVPRRuntime
    from .weights import OPTConfig, OPTWeights

    rng = random.Random(seed)
    failures = []
    for case in range(cases):
        heads = rng.choice([1, 2, 4, 8])
        d = rng.choice([64, 128])
        h = heads * d
        b = rng.randint(1, 4)
        S0 = rng.randint(1, 48)
        cfg = OPTConfig(hidden=h, layers=2, heads=heads, ffn=4 * h, vocab=256, max_pos=128)
        w = OPTWeights.random(cfg, seed=case, device="cuda", std=0.1, emb_std=0.1)
        prompt = torch.randint(0, 256, (b, S0), generator=torch.Generator().manual_seed(case))
        outs = []
        for l in sorted({0, rng.randint(0, S0 + 1), S0 + 1}):
            rt = KVPRRuntime(w, b, S0 + 2)
            first = rt.prefill(prompt)
            if not outs:
                for j in range(cfg.layers):
                    pages = torch.zeros(S0 + 2, 2, b, h, dtype=torch.float16, device="cuda")
                    kernels.recompute_kv(rt.stores.x[j].cuda(), w.layers[j].w_kv, w.layers[j].b_kv, pages, b, 0, S0)
                    if not torch.equal(pages[:S0].cpu(), rt.stores.kv[j][:S0]):
                        failures.append(f"case={case} layer={j} h={h} b={b} s={S0}: rebuilt pages differ")
            rt.decode([l], tokens=first, keep_logits=True)
            torch.cuda.synchronize()
            outs.append((l, rt.last_logits.cpu()))
            rt.close()
        for l, lg in outs[1:]:
            if not torch.equal(lg, outs[0][1]):
                failures.append(f"case={case} h={h} b={b} s'={S0 + 1} l={l}: logits differ from l=0")
    return failures


def cmd_validate(a) -> int:
    failures = run_validation_cases(a.seed, a.cases)
    if failures:
        for f in failures:
            print(f"FAIL {f}", file=sys.stderr)
        print(f"validation failed: {len(failures)} case(s)", file=sys.stderr)
        return EXIT_VALIDATION
    print(f"ok: {a.cases} cases, rebuilt pages and decode logits bit-exact for every split")
    return EXIT_OK


def build_parser() -> argparse.ArgumentParser:
    p = _Parser(prog="paper_2411_17089_b200", description="KVPR decode path on B200")
    sub = p.add_subparsers(dest="command", required=True)
    sp = sub.add_parser("plan")
    sp.add_argument("--config", required=True)
    sp.add_argument("--l", type=int, default=None)
    sp.add_argument("--out")
    sp.set_defaults(fn=cmd_plan)
    sp = sub.add_parser("simulate")
    sp.add_argument("--config", required=True)
    sp.add_argument("--plan")
    sp.add_argument("--out")
    sp.add_argument("--trace")
    sp.add_argument("--metrics")
    sp.add_argument("--l", type=int, default=None)
    sp.set_defaults(fn=cmd_simulate)
    sp = sub.add_parser("sweep")
    sp.add_argument("--config", required=True)
    sp.add_argument("--vary", required=True)
    sp.add_argument("--policies", default="naive,kvpr")
    sp.add_argument("--out")
    sp.set_defaults(fn=cmd_sweep)
    sp = sub.add_parser("calibrate")
    sp.add_argument("--measurements", required=True)
    sp.add_argument("--out")
    sp.set_defaults(fn=cmd_calibrate)
    sp = sub.add_parser("profile")
    sp.add_argument("--hidden", type=int, default=4096)
    sp.add_argument("--batch", type=int, default=32)
    sp.add_argument("--out")
    sp.set_defaults(fn=cmd_profile)
    sp = sub.add_parser("run")
    sp.add_argument("--config", required=True)
    sp.add_argument("--plan")
    sp.add_argument("--l", type=int, default=None)
    sp.add_argument("--trace")
    sp.add_argument("--metrics")
    sp.set_defaults(fn=cmd_run)
    sp = sub.add_parser("validate")
    sp.add_argument("--cases", type=int, default=20)
    sp.add_argument("--seed", type=int, default=0)
    sp.set_defaults(fn=cmd_validate)
    return p


def main(argv=None) -> int:
    level = os.environ.get("KVPR_LOG", "error").upper()
    logging.basicConfig(level=getattr(logging, level, logging.ERROR), stream=sys.stderr)
    try:
        args = build_parser().parse_args(argv)
        if getattr(args, "cases", 1) < 1:
            raise ConfigError("--cases must be >= 1")
        return args.fn(args)
    except GpuMemoryBudgetError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_BUDGET
    except (ConfigError, ValueError, OSError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_INVALID
