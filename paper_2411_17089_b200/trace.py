"""Measured timelines of the B200 runtime in the reference simulator's schema.

The reference exports *simulated* timelines (pipesim/trace.py:16, 30-49):
Chrome trace "X" events with lanes h2d=0 / gpu=1 / d2h=2, microsecond
timestamps, task names "<kind>[ <part>] i<step> j<layer>" (tasks.py:73-82),
and a metrics row (trace.py:18-27, 52-62).  Here the same documents are
produced from CUDA events recorded around every transfer and kernel group
of a real decode run (KVPRRuntime.decode(..., trace=Tracer())), so a measured
run can be compared line by line with a simulated one.  ``check_invariants``
restates the simulator's timeline checks (engine.py:103-119) on the measured
data: one operation at a time per lane, and every dependency of the task
graph (graph.py:266-347) honoured.
"""

from __future__ import annotations

import csv
import json
from dataclasses import dataclass, field

import torch

TRACE_LANES = {"h2d": 0, "gpu": 1, "d2h": 2}

KIND_LANE = {
    "load_activation_recompute": "h2d",
    "load_cache": "h2d",
    "compute_recompute": "gpu",
    "compute_mha": "gpu",
    "compute_ffn": "gpu",
    "store_cache": "d2h",
    "store_activation": "d2h",
}

METRICS_COLUMNS = ("policy", "schedule", "granularity", "recompute", "makespan_s", "throughput_tok_s", "gpu_util",
                   "peak_gpu_bytes")


@dataclass
class _Span:
    kind: str
    part: str
    step: int
    layer: int
    start: torch.cuda.Event
    end: torch.cuda.Event


@dataclass(frozen=True)
class Entry:
    kind: str
    part: str
    step: int
    layer: int
    start: float  # seconds since the run's first event
    end: float

    @property
    def lane(self) -> str:
        return KIND_LANE[self.kind]

    @property
    def name(self) -> str:
        bits = [self.kind] + ([self.part] if self.part else []) + [f"i{self.step}", f"j{self.layer}"]
        return " ".join(bits)


@dataclass
class Tracer:
    """Collects (start, end) CUDA events around runtime operations."""

    spans: list[_Span] = field(default_factory=list)
    origin: torch.cuda.Event | None = None

    def begin(self, stream: torch.cuda.Stream, kind: str, step: int, layer: int, part: str = "") -> _Span:
        if kind not in KIND_LANE:
            raise ValueError(f"unknown task kind {kind!r}")
        if self.origin is None:
            self.origin = torch.cuda.Event(enable_timing=True)
            self.origin.record(stream)
        sp = _Span(kind, part, step, layer, torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        sp.start.record(stream)
        return sp

    def end(self, stream: torch.cuda.Stream, sp: _Span) -> None:
        sp.end.record(stream)
        self.spans.append(sp)

    def entries(self) -> list[Entry]:
        """Resolve events (synchronises) into entries sorted by start time."""
        if self.origin is None:
            return []
        for sp in self.spans:
            sp.end.synchronize()
        out = [Entry(sp.kind, sp.part, sp.step, sp.layer, self.origin.elapsed_time(sp.start) / 1e3,
                     self.origin.elapsed_time(sp.end) / 1e3) for sp in self.spans]
        t0 = min(e.start for e in out)
        out = [Entry(e.kind, e.part, e.step, e.layer, e.start - t0, e.end - t0) for e in out]
        return sorted(out, key=lambda e: (e.start, TRACE_LANES[e.lane]))


def export_trace(entries: list[Entry]) -> list[dict]:
    """Chrome trace-event document in the reference's schema (trace.py:30-43)."""
    return [{"name": e.name, "cat": e.kind, "ph": "X", "ts": e.start * 1e6, "dur": (e.end - e.start) * 1e6, "pid": 0,
             "tid": TRACE_LANES[e.lane]} for e in entries]


def write_trace(entries: list[Entry], path: str) -> None:
    with open(path, "w") as fh:
        json.dump(export_trace(entries), fh, sort_keys=True, separators=(",", ":"))
        fh.write("\n")


def _union(intervals):
    tot, cur_s, cur_e = 0.0, None, None
    for s, e in sorted(intervals):
        if cur_e is None or s > cur_e:
            if cur_e is not None:
                tot += cur_e - cur_s
            cur_s, cur_e = s, e
        else:
            cur_e = max(cur_e, e)
    if cur_e is not None:
        tot += cur_e - cur_s
    return tot


def report(entries: list[Entry], tokens: int) -> dict:
    """Measured analogue of SimReport (tasks.py:113-122): makespan, tok/s, GPU busy fraction, per-kind share."""
    if not entries:
        return {"makespan_s": 0.0, "throughput_tok_s": 0.0, "gpu_util": 0.0, "breakdown": {}}
    makespan = max(e.end for e in entries) - min(e.start for e in entries)
    gpu = _union([(e.start, e.end) for e in entries if e.lane == "gpu"])
    lanes = {lane: _union([(e.start, e.end) for e in entries if e.lane == lane]) / makespan for lane in TRACE_LANES}
    kinds = {}
    for k in KIND_LANE:
        kinds[k] = sum(e.end - e.start for e in entries if e.kind == k) / makespan
    return {"makespan_s": makespan, "throughput_tok_s": tokens / makespan if makespan > 0 else 0.0,
            "gpu_util": gpu / makespan, "lane_busy": lanes, "breakdown": kinds}


def metrics_row(label: str, rep: dict, schedule: str = "column", peak_gpu_bytes: float = 0.0) -> dict:
    return {"policy": label, "schedule": schedule, "granularity": "coarse", "recompute": "on",
            "makespan_s": rep["makespan_s"], "throughput_tok_s": rep["throughput_tok_s"], "gpu_util": rep["gpu_util"],
            "peak_gpu_bytes": peak_gpu_bytes}


def write_metrics_csv(rows, fh) -> None:
    w = csv.writer(fh, lineterminator="\n")
    w.writerow(METRICS_COLUMNS)
    for r in rows:
        w.writerow([repr(r[c]) if isinstance(r[c], float) else str(r[c]) for c in METRICS_COLUMNS])


def check_invariants(entries: list[Entry], layers: int, tol: float = 2e-6) -> list[str]:
    """Lane exclusivity and the task-graph dependencies on a measured timeline.

    Returns a list of violations (empty = consistent).  Dependencies checked
    (graph.py:266-347): recompute chunk c after its activation chunk landed;
    MHA after the KV load and after every recompute chunk; the KV load of
    (i, j) after the cache store of (i-1, j); FFN after MHA; stores after the
    MHA that produced them.
    """
    bad = []
    # transfers on one copy engine never overlap (the GPU lane may overlap across streams? no: one compute stream)
    for lane in TRACE_LANES:
        es = sorted((e for e in entries if e.lane == lane), key=lambda e: e.start)
        for a, b in zip(es, es[1:]):
            if b.start < a.end - tol:
                bad.append(f"{lane}: {b.name} starts before {a.name} ends")
    by = {}
    for e in entries:
        by.setdefault((e.kind, e.step, e.layer), []).append(e)

    def ends(kind, i, j, part=None):
        return [e.end for e in by.get((kind, i, j), []) if part is None or e.part == part]

    for (kind, i, j), es in by.items():
        if kind == "compute_recompute":
            for e in es:
                src = ends("load_activation_recompute", i, j, e.part)
                if src and e.start < max(src) - tol:
                    bad.append(f"{e.name} starts before its activation chunk landed")
        if kind == "compute_mha":
            attn = [x for x in es if x.part == "attn"]
            if not attn:
                continue
            e = attn[0]
            for dep in ("load_cache", "compute_recompute"):
                d = ends(dep, i, j)
                if d and e.start < max(d) - tol:
                    bad.append(f"{e.name} starts before {dep} i{i} j{j} finished")
        if kind == "compute_ffn":
            d = ends("compute_mha", i, j, "attn")
            if d and es[0].start < max(d) - tol:
                bad.append(f"{es[0].name} starts before compute_mha")
        if kind == "load_cache" and i > 1:
            d = ends("store_cache", i - 1, j)
            if d and es[0].start < max(d) - tol:
                bad.append(f"{es[0].name} starts before store_cache i{i - 1} j{j} finished")
    return bad


# ---------------------------------------------------------------------------
# measured vs simulated

def _med(xs):
    xs = sorted(xs)
    return xs[len(xs) // 2] if xs else 0.0


def compare_with_model(entries: list[Entry], spec, wl, profile, plan, schedule: str = "column") -> dict:
    """Lay a measured decode next to the reference's prediction for the same plan and profile.

    The reference predicts a run by list-scheduling its task DAG (pipesim.build_task_graph +
    simulate, graph.py:176-355, engine.py:140-204) with durations from the profile.  Returned:

    * ``kinds``: per task kind, total measured busy time vs the simulated total (ratio = measured /
      simulated).  Transfers and the recompute are what the profile models (calibrated bandwidths,
      the profiled K1 rate); the reference prices MHA / FFN at the GEMM FLOP rate, which a decode
      step (HBM-bound) does not run at, so those ratios are reported, not expected to be 1;
    * ``makespan``: measured vs simulated, and vs a *replay*: the same DAG and scheduler fed the
      measured per-task durations.  replay / measured >= 1 means the runtime realised at least the
      overlap the DAG allows (it pipelines X chunks under K1, which the DAG's recompute-after-all-of-X
      edge does not);
    * ``layer``: steady-state per-layer time (median spacing of consecutive FFN ends) both ways.
    The DAG's token-activation loads (column mode's per-unit X row, graph.py:295-304) are modeled but
    not executed: the runtime keeps the residual stream in HBM, so they replay as zero.
    """
    from . import pipesim as ps

    pol = ps.Policy(schedule, True)
    graph = ps.build_task_graph(spec, wl, profile, plan, pol)
    tl, rep = ps.simulate(graph, profile)
    sim_dur = ps.task_durations(graph, profile).tolist()
    meas: dict[tuple[str, int, int], float] = {}
    for e in entries:
        key = (e.kind, e.step, e.layer)
        meas[key] = meas.get(key, 0.0) + (e.end - e.start)
    kinds: dict[str, dict] = {}
    replay = []
    for t in graph.tasks:
        k = t.kind.value
        m = meas.get((k, t.step, t.layer), 0.0)
        replay.append(m)
        d = kinds.setdefault(k, {"measured_s": 0.0, "simulated_s": 0.0, "tasks": 0})
        d["measured_s"] += m
        d["simulated_s"] += sim_dur[t.id]
        d["tasks"] += 1
    for d in kinds.values():
        d["ratio"] = d["measured_s"] / d["simulated_s"] if d["simulated_s"] > 0 else None
    _, rep_replay = ps.simulate(graph, profile, durations=replay)
    m_span = max(e.end for e in entries) - min(e.start for e in entries)
    m_ffn = sorted(e.end for e in entries if e.kind == "compute_ffn")
    s_ffn = sorted(tl.entries[t.id].end for t in graph.tasks if t.kind is ps.TaskKind.COMPUTE_FFN)
    m_layer = _med([b - a for a, b in zip(m_ffn, m_ffn[1:])])
    s_layer = _med([b - a for a, b in zip(s_ffn, s_ffn[1:])])
    return {
        "kinds": kinds,
        "makespan": {"measured_s": m_span, "simulated_s": rep.makespan, "replay_s": rep_replay.makespan,
                     "measured_over_simulated": m_span / rep.makespan if rep.makespan > 0 else None,
                     "replay_over_measured": rep_replay.makespan / m_span if m_span > 0 else None},
        "layer": {"measured_s": m_layer, "simulated_s": s_layer,
                  "measured_over_simulated": m_layer / s_layer if s_layer > 0 else None},
        "simulated_report": {"decode_throughput": rep.decode_throughput, "gpu_utilization": rep.gpu_utilization},
    }
