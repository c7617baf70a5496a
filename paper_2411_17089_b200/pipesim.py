"""The reference's offload-pipeline model, restated: task DAG + list scheduler.

kvoverlap predicts a decode run by building a task DAG per (step, layer, batch) unit
(pipesim/graph.py:176-355), assigning every task a duration from the hardware
profile (engine.py:81-90) and list-scheduling it onto three exclusive lanes
h2d / gpu / d2h (_engine_py.py:18-90).  The B200 runtime executes the same DAG on
real streams; this module reproduces the prediction so a measured timeline
(trace.py) can be laid next to the simulated one for the same plan and profile
(criterion 04's analytic-vs-simulated check,
test_acceptance.py:150-183, is the template).

Same API and results as the reference, bit for bit (tests/test_pipesim_cpu.py
against timelines produced by the live reference, tests/golden/pipesim_golden.json):
``Policy``, ``build_task_graph``, ``estimate_peak_gpu_bytes``, ``task_durations``,
``run_schedule``, ``simulate`` -> (``Timeline``, ``SimReport``), and the exporters / policy table
of pipesim/trace.py (``export_trace``, ``write_trace``, ``metrics_row``, ``write_metrics_csv``,
``plan_for_policy``, ``compare``) behind the CLI's ``simulate`` and ``sweep``.  Only the pure
Python engine is restated (the Cython twin computes identical schedules).

Per unit the graph holds up to eight tasks (graph.py:1-28):
    h2d  weights (streamed: whole, or K/V half then Q/O half), X[:, :l] for the
         rebuild (column), KV[l:s'], the unit's token activations (column)
    gpu  recompute K,V[0:l), MHA, FFN — one program-ordered compute stream
    d2h  the new K,V page, the new activation row (column)
Ordering: data dependencies for correctness, queue priorities for preference
(h2d: weights-KV < recompute X < weights-QO < KV < token X; earlier units
first), double buffering as a dependency on the consumer two loads back.
"""

from __future__ import annotations

import csv
import heapq
import json
import math
import os
from dataclasses import dataclass, field

import numpy as np
from enum import Enum

from .costmodel import (ModelSpec, WorkloadSpec, activation_bytes, decode_step_flops, kv_remainder_bytes,
                        mha_matrix_bytes, mha_weight_bytes, recompute_flops, token_activation_bytes,
                        token_kv_store_bytes)
from .hwprofile import HardwareProfile, compute_time, transfer_time
from .scheduler import SCHEDULE_MODES, SplitPlan, constant_plan, plan_generation


class TaskKind(str, Enum):
    LOAD_WEIGHT = "load_weight"
    LOAD_CACHE = "load_cache"
    LOAD_ACTIVATION = "load_activation"
    LOAD_ACTIVATION_RECOMPUTE = "load_activation_recompute"
    COMPUTE_RECOMPUTE = "compute_recompute"
    COMPUTE_MHA = "compute_mha"
    COMPUTE_FFN = "compute_ffn"
    STORE_CACHE = "store_cache"
    STORE_ACTIVATION = "store_activation"
    SYNC = "sync"


class Resource(str, Enum):
    H2D = "h2d"
    GPU = "gpu"
    D2H = "d2h"


RESOURCE_INDEX = {Resource.H2D: 0, Resource.GPU: 1, Resource.D2H: 2}  # engine ids == trace lanes

_LANE = {"load": Resource.H2D, "compute": Resource.GPU, "store": Resource.D2H, "sync": Resource.GPU}
KIND_RESOURCE = {k: _LANE[k.value.split("_")[0]] for k in TaskKind}

GRANULARITIES = ("coarse", "fine")


class GpuMemoryBudgetError(RuntimeError):
    """Estimated peak GPU residency exceeds the configured budget (graph.py:70)."""


class DependencyCycleError(ValueError):
    """Some tasks never became ready (_engine_py.py:15)."""


@dataclass(frozen=True)
class Policy:
    """Pipeline variant (graph.py:74-87)."""

    schedule: str = "row"
    recompute: bool = True
    granularity: str = "coarse"
    weights_resident: bool = True

    def __post_init__(self) -> None:
        if self.schedule not in SCHEDULE_MODES:
            raise ValueError(f"schedule must be one of {SCHEDULE_MODES}")
        if self.granularity not in GRANULARITIES:
            raise ValueError(f"granularity must be one of {GRANULARITIES}")


@dataclass(frozen=True)
class Task:
    """One unit of work on one lane; cost = bytes (transfers) or FLOPs (gpu) (tasks.py:45-82)."""

    id: int
    kind: TaskKind
    resource: Resource
    cost: float
    deps: tuple[int, ...]
    step: int
    layer: int
    batch: int
    priority: int
    part: str = ""

    def __post_init__(self) -> None:
        if KIND_RESOURCE[self.kind] is not self.resource:
            raise ValueError(f"{self.kind.value} cannot run on {self.resource.value}")
        if self.cost < 0:
            raise ValueError("cost must be nonnegative")

    @property
    def name(self) -> str:
        """'<kind>[ <part>] i<step> j<layer>[ k<batch>]' (the trace event name)."""
        tail = [f"i{self.step}", f"j{self.layer}"] + ([f"k{self.batch}"] if self.batch >= 0 else [])
        return " ".join([self.kind.value] + ([self.part] if self.part else []) + tail)


@dataclass(frozen=True)
class TaskGraph:
    tasks: tuple[Task, ...]
    tokens_generated: int
    peak_gpu_bytes: float

    def __len__(self) -> int:
        return len(self.tasks)


@dataclass(frozen=True)
class TimelineEntry:
    task_id: int
    kind: str
    resource: str
    start: float
    end: float
    name: str


@dataclass(frozen=True)
class Timeline:
    entries: tuple[TimelineEntry, ...]
    makespan: float


@dataclass(frozen=True)
class SimReport:
    makespan: float
    decode_throughput: float
    gpu_utilization: float
    breakdown: dict[str, float] = field(default_factory=dict)
    utilization_timeline: tuple[tuple[float, float], ...] = ()
    peak_gpu_bytes: float = 0.0


# ---------------------------------------------------------------------------
# graph

# queue classes (smaller first within a unit) and the per-unit priority stride (graph.py:56-67)
_H2D_CLASS = {"w_kv": 0, "x_recompute": 1, "w_qo": 2, "kv": 3, "x_token": 4}
_GPU_CLASS = {"recompute": 0, "mha": 1, "ffn": 2}
_D2H_CLASS = {"kv": 0, "x": 1}
_STRIDE = 8


def _units(wl: WorkloadSpec, layers: int, schedule: str) -> list[tuple[int, int, int]]:
    """(step, layer, batch), 1-based step/layer: row = batch-major, column = layer-major (graph.py:128-134)."""
    if schedule == "row":
        return [(i, j, k) for k in range(wl.num_batches) for i in range(1, wl.gen_len + 1)
                for j in range(1, layers + 1)]
    return [(i, j, k) for i in range(1, wl.gen_len + 1) for j in range(1, layers + 1)
            for k in range(wl.num_batches)]


def _validate(wl: WorkloadSpec, plan: SplitPlan, policy: Policy) -> None:
    if plan.mode != policy.schedule:
        raise ValueError(f"plan mode {plan.mode!r} != policy schedule {policy.schedule!r}")
    if len(plan.decisions) != wl.gen_len:
        raise ValueError("plan does not cover gen_len steps")
    for step, d in enumerate(plan.decisions, start=1):
        if d.step != step or d.seq_len != wl.prompt_len + step:
            raise ValueError(f"plan step {step} inconsistent with workload")
        if not 0 <= d.recompute_len <= d.seq_len:
            raise ValueError(f"plan step {step}: split out of range")


def _splits(plan: SplitPlan, policy: Policy) -> list[int]:
    return [d.recompute_len if policy.recompute else 0 for d in plan.decisions]


def estimate_peak_gpu_bytes(spec: ModelSpec, wl: WorkloadSpec, plan: SplitPlan, policy: Policy) -> float:
    """Resident (or two streamed) layers' weights + two staging buffers of the largest KV tail, and in
    column mode two X staging buffers, two token-activation buffers and the retained rebuild prefixes
    of every batch (graph.py:149-173)."""
    splits = _splits(plan, policy)
    layers = spec.num_layers if policy.weights_resident else 2
    total = float(layers * mha_weight_bytes(spec))
    total += 2 * max(kv_remainder_bytes(spec, wl, wl.prompt_len + s, l) for s, l in enumerate(splits, start=1))
    if policy.schedule == "column":
        x_max = max(activation_bytes(spec, wl, l) for l in splits)
        total += 2 * x_max + 2 * token_activation_bytes(spec, wl) + wl.num_batches * x_max
    return total


class _Graph:
    """Accumulates tasks; ids are positions."""

    def __init__(self) -> None:
        self.tasks: list[Task] = []

    def add(self, kind: TaskKind, cost: float, deps, unit, priority: int, batch=None, part: str = "") -> int:
        i, j, k = unit
        tid = len(self.tasks)
        uniq = tuple(dict.fromkeys(d for d in deps if d is not None))
        self.tasks.append(Task(tid, kind, KIND_RESOURCE[kind], cost, uniq, i, j, k if batch is None else batch,
                               priority, part))
        return tid


def build_task_graph(spec: ModelSpec, wl: WorkloadSpec, profile: HardwareProfile, plan: SplitPlan, policy: Policy,
                     gpu_mem_budget: float | None = None) -> TaskGraph:
    """The decode DAG of one policy (graph.py:176-355).  ``profile`` does not shape it (durations come
    from simulate); GpuMemoryBudgetError when the residency estimate exceeds the budget."""
    del profile
    _validate(wl, plan, policy)
    peak = estimate_peak_gpu_bytes(spec, wl, plan, policy)
    if gpu_mem_budget is not None and peak > gpu_mem_budget:
        raise GpuMemoryBudgetError(f"estimated peak {peak:.0f} B exceeds budget {gpu_mem_budget:.0f} B")
    L = spec.num_layers
    column = policy.schedule == "column"
    splits = _splits(plan, policy)
    flops = {s: decode_step_flops(spec, wl, wl.prompt_len + s) for s in range(1, wl.gen_len + 1)}
    w_bytes = {"half": float(2 * mha_matrix_bytes(spec)), "full": float(mha_weight_bytes(spec))}
    x_tok, kv_tok = float(token_activation_bytes(spec, wl)), float(token_kv_store_bytes(spec, wl))

    g = _Graph()
    prev_gpu = None
    # double buffering: the consumer of each staged load, per category; a load waits for the consumer
    # of the load two before it in its category (graph.py:215-221)
    consumers = {"kv": [], "x": [], "tok": []}
    loads = {"kv": 0, "x": 0, "tok": 0}

    def two_back(cat):
        return consumers[cat][loads[cat] - 2] if loads[cat] >= 2 else None

    groups: dict[tuple, int] = {}             # weight group key -> index (first-use order)
    group_tasks: list[tuple[int, int]] = []   # (K/V-half load, Q/O-half load); one task twice if coarse
    group_done: list[int | None] = []         # last MHA that reads the group
    ffn_of, store_kv_of, store_x_of = {}, {}, {}

    for t, unit in enumerate(_units(wl, L, policy.schedule)):
        i, j, k = unit
        s, l = wl.prompt_len + i, splits[i - 1]
        base = t * _STRIDE

        w_kv = w_qo = gidx = None
        if not policy.weights_resident:
            key = (i, j) if column else (i, j, k)
            wbatch = -1 if column else k
            if key in groups:
                gidx = groups[key]
                w_kv, w_qo = group_tasks[gidx]
            else:
                gidx = groups[key] = len(group_tasks)
                wdep = [group_done[gidx - 2]] if gidx >= 2 else []
                if policy.granularity == "fine":
                    w_kv = g.add(TaskKind.LOAD_WEIGHT, w_bytes["half"], wdep, unit, base + _H2D_CLASS["w_kv"],
                                 wbatch, "kv")
                    w_qo = g.add(TaskKind.LOAD_WEIGHT, w_bytes["half"], wdep, unit, base + _H2D_CLASS["w_qo"],
                                 wbatch, "qo")
                else:
                    w_kv = w_qo = g.add(TaskKind.LOAD_WEIGHT, w_bytes["full"], wdep, unit,
                                        base + _H2D_CLASS["w_kv"], wbatch)
                group_tasks.append((w_kv, w_qo))
                group_done.append(None)

        x_load = None
        if column and l > 0:
            deps = [two_back("x")]
            if l > wl.prompt_len:  # the newest rebuilt position was produced during this decode
                m = l - wl.prompt_len
                if j >= 2:
                    deps.append(store_x_of[(m, j - 1, k)])
                elif m >= 2:
                    deps.append(ffn_of[(m - 1, L, k)])
            x_load = g.add(TaskKind.LOAD_ACTIVATION_RECOMPUTE, float(activation_bytes(spec, wl, l)), deps, unit,
                           base + _H2D_CLASS["x_recompute"])
            loads["x"] += 1

        kv_load = None
        if l < s:
            deps = [two_back("kv")] + ([store_kv_of[(i - 1, j, k)]] if i >= 2 else [])
            kv_load = g.add(TaskKind.LOAD_CACHE, kv_remainder_bytes(spec, wl, s, l), deps, unit, base + _H2D_CLASS["kv"])
            loads["kv"] += 1

        tok_load = None
        if column:
            deps = [two_back("tok")]
            if j >= 2:
                deps.append(store_x_of[(i, j - 1, k)])
            elif i >= 2:
                deps.append(store_x_of[(i - 1, L, k)])
            tok_load = g.add(TaskKind.LOAD_ACTIVATION, x_tok, deps, unit, base + _H2D_CLASS["x_token"])
            loads["tok"] += 1

        rec = None
        if l > 0:
            rec = g.add(TaskKind.COMPUTE_RECOMPUTE, float(recompute_flops(spec, wl, l)), [x_load, w_kv, prev_gpu],
                        unit, base + _GPU_CLASS["recompute"])
            prev_gpu = rec
            if x_load is not None:
                consumers["x"].append(rec)

        mha = g.add(TaskKind.COMPUTE_MHA, float(flops[i].mha), [rec, kv_load, tok_load, w_kv, w_qo, prev_gpu], unit,
                    base + _GPU_CLASS["mha"])
        prev_gpu = mha
        if kv_load is not None:
            consumers["kv"].append(mha)
        if tok_load is not None:
            consumers["tok"].append(mha)
        if gidx is not None and (not column or k == wl.num_batches - 1):
            group_done[gidx] = mha

        ffn = g.add(TaskKind.COMPUTE_FFN, float(flops[i].ffn), [mha], unit, base + _GPU_CLASS["ffn"])
        prev_gpu = ffn_of[unit] = ffn
        store_kv_of[unit] = g.add(TaskKind.STORE_CACHE, kv_tok, [mha], unit, base + _D2H_CLASS["kv"])
        if column:
            store_x_of[unit] = g.add(TaskKind.STORE_ACTIVATION, x_tok, [ffn], unit, base + _D2H_CLASS["x"])

    return TaskGraph(tuple(g.tasks), wl.batch_size * wl.num_batches * wl.gen_len, peak)


# ---------------------------------------------------------------------------
# engine

def task_durations(graph: TaskGraph, profile: HardwareProfile) -> np.ndarray:
    """Seconds per task (float64 array, as the reference returns): FLOPs / effective rate on the gpu lane,
    latency + bytes / bandwidth on the copy lanes (engine.py:79-90)."""
    out = np.empty(len(graph), dtype=np.float64)
    for tk in graph.tasks:
        if tk.resource is Resource.GPU:
            out[tk.id] = compute_time(profile, tk.cost)
        else:
            out[tk.id] = transfer_time(profile, tk.cost, tk.resource.value)
    return out


def _list_schedule(resource, duration, priority, deps, n_resources: int = 3) -> tuple[list[float], list[float]]:
    """Non-preemptive list scheduling (_engine_py.py:18-90): whenever a lane is idle it starts the ready
    task with the smallest (priority, id); all lanes finishing at the same instant complete before the
    next dispatch.  deps[i] = task ids task i waits for.  Returns (start, end) per task."""
    n = len(resource)
    waiting = [len(d) for d in deps]
    children: list[list[int]] = [[] for _ in range(n)]
    for i, ds in enumerate(deps):
        for d in ds:
            children[d].append(i)
    ready: list[list[tuple[int, int]]] = [[] for _ in range(n_resources)]
    for i in range(n):
        if waiting[i] == 0:
            heapq.heappush(ready[resource[i]], (priority[i], i))
    busy = [-1] * n_resources
    busy_until = [0.0] * n_resources
    start, end = [0.0] * n, [0.0] * n
    done = 0

    def fill(now: float) -> None:
        for r in range(n_resources):
            if busy[r] < 0 and ready[r]:
                i = heapq.heappop(ready[r])[1]
                start[i], end[i] = now, now + duration[i]
                busy[r], busy_until[r] = i, end[i]

    fill(0.0)
    while True:
        active = [busy_until[r] for r in range(n_resources) if busy[r] >= 0]
        if not active:
            break
        now = min(active)
        for r in range(n_resources):
            if busy[r] >= 0 and busy_until[r] == now:
                i, busy[r] = busy[r], -1
                done += 1
                for c in children[i]:
                    waiting[c] -= 1
                    if waiting[c] == 0:
                        heapq.heappush(ready[resource[c]], (priority[c], c))
        fill(now)
    if done != n:
        raise DependencyCycleError(f"{n - done} of {n} tasks never became ready")
    return start, end


# engine selection (engine.py:45-76): the pure-Python engine (`_list_schedule`) and the compiled one,
# `kvpr_list_schedule` in libkvpr (csrc/sched_engine.cu, the counterpart of the reference's _engine.pyx;
# identical schedules).  As in the reference: "c" when the library loads, KVOVERLAP_ENGINE=py|c forces one
# side, forcing "c" without it is an error.
_ENGINE_ENV = "KVOVERLAP_ENGINE"


def _c_available() -> bool:
    try:
        from . import _lib

        _lib.load()
        return True
    except (OSError, RuntimeError):
        return False


def available_engines() -> tuple[str, ...]:
    return ("py", "c") if _c_available() else ("py",)


def active_engine() -> str:
    """Engine simulate() uses right now, honouring the environment override."""
    forced = os.environ.get(_ENGINE_ENV, "").strip().lower()
    if forced:
        if forced not in ("py", "c"):
            raise ValueError(f"{_ENGINE_ENV} must be 'py' or 'c', got {forced!r}")
        if forced == "c" and not _c_available():
            raise RuntimeError("KVOVERLAP_ENGINE=c but the compiled engine is not built")
        return forced
    return "c" if _c_available() else "py"


def _engine(engine: str | None) -> str:
    name = engine if engine is not None else active_engine()
    if name == "c" and not _c_available():
        raise RuntimeError("compiled engine requested but not built")
    if name not in ("py", "c"):
        raise ValueError(f"unknown engine {name!r}")
    return name


def _dep_csr(graph: TaskGraph) -> tuple[np.ndarray, np.ndarray]:
    """The graph's dependencies as CSR arrays (engine.py:92-100)."""
    indptr = np.zeros(len(graph) + 1, dtype=np.int64)
    indptr[1:] = np.cumsum([len(t.deps) for t in graph.tasks])
    indices = np.fromiter((d for t in graph.tasks for d in t.deps), dtype=np.int64, count=int(indptr[-1]))
    return indptr, indices


def _run_c(resource, duration, priority, indptr, indices, n_resources: int):
    import ctypes

    from . import _lib

    res = np.ascontiguousarray(resource, dtype=np.int64)
    dur = np.ascontiguousarray(duration, dtype=np.float64)
    pri = np.ascontiguousarray(priority, dtype=np.int64)
    ip = np.ascontiguousarray(indptr, dtype=np.int64)
    ix = np.ascontiguousarray(indices, dtype=np.int64)
    n = len(res)
    start, end = np.zeros(n, dtype=np.float64), np.zeros(n, dtype=np.float64)
    ptr = lambda a: a.ctypes.data_as(ctypes.c_void_p) if a.size else None  # noqa: E731
    rc = _lib.load().kvpr_list_schedule(n, ptr(res), ptr(dur), ptr(pri), ptr(ip), ptr(ix), int(n_resources),
                                        ptr(start), ptr(end))
    if rc == _lib.KVPR_ECYCLE:
        raise DependencyCycleError(_lib.last_error())
    _lib.check(rc, "kvpr_list_schedule")
    return start, end


def run_schedule(resource, duration, priority, dep_indptr, dep_indices, n_resources: int, engine: str | None = None):
    """The reference's engine entry point (engine.py:61-76, _engine_py.py:18-90): dependencies as CSR
    (task i waits for dep_indices[dep_indptr[i]:dep_indptr[i+1]]); returns (start, end) float64 arrays."""
    if _engine(engine) == "c":
        return _run_c(resource, duration, priority, dep_indptr, dep_indices, n_resources)
    n = len(resource)
    indptr = np.asarray(dep_indptr, dtype=np.int64).tolist()
    indices = np.asarray(dep_indices, dtype=np.int64).tolist()
    deps = [indices[indptr[i]:indptr[i + 1]] for i in range(n)]
    start, end = _list_schedule(np.asarray(resource, dtype=np.int64).tolist(),
                                np.asarray(duration, dtype=np.float64).tolist(),
                                np.asarray(priority, dtype=np.int64).tolist(), deps, n_resources)
    return np.asarray(start, dtype=np.float64), np.asarray(end, dtype=np.float64)


def _bins(spans, makespan: float, bins: int) -> tuple[tuple[float, float], ...]:
    """GPU-lane busy fraction per equal-width bin (engine.py:122-137)."""
    if makespan <= 0 or not math.isfinite(makespan) or bins <= 0:
        return ()
    width = makespan / bins
    busy = [0.0] * bins
    for s, e in spans:
        lo = min(bins - 1, int(s / width))
        hi = min(bins - 1, int(e / width)) if e > s else lo
        for b in range(lo, hi + 1):
            left = b * width
            busy[b] += max(0.0, min(e, left + width) - max(s, left))
    return tuple(((b + 0.5) * width, min(1.0, busy[b] / width)) for b in range(bins))


def simulate(graph: TaskGraph, profile: HardwareProfile, *, engine: str | None = None, bins: int = 100,
             check: bool = True, durations: list[float] | None = None) -> tuple[Timeline, SimReport]:
    """(Timeline, SimReport) of the graph under the profile (engine.py:140-204).  ``durations``
    overrides the profile's per-task durations (e.g. measured ones: replaying a measured run through
    the same DAG and scheduler)."""
    name = _engine(engine)
    tasks = graph.tasks
    dur = list(durations) if durations is not None else task_durations(graph, profile).tolist()
    res, pri = [RESOURCE_INDEX[t.resource] for t in tasks], [t.priority for t in tasks]
    if name == "c":
        s_arr, e_arr = _run_c(res, dur, pri, *_dep_csr(graph), len(RESOURCE_INDEX))
        start, end = s_arr.tolist(), e_arr.tolist()
    else:
        start, end = _list_schedule(res, dur, pri, [t.deps for t in tasks])
    if check:
        check_schedule(graph, start, end)
    n = len(tasks)
    makespan = max(end) if n else 0.0
    timeline = Timeline(tuple(TimelineEntry(t.id, t.kind.value, t.resource.value, start[t.id], end[t.id], t.name)
                              for t in tasks), makespan)
    finite = makespan > 0 and math.isfinite(makespan)
    by_kind: dict[str, float] = {}
    gpu_busy, gpu_spans = 0.0, []
    for t in tasks:
        by_kind[t.kind.value] = by_kind.get(t.kind.value, 0.0) + dur[t.id]
        if t.resource is Resource.GPU:
            gpu_busy += dur[t.id]
            gpu_spans.append((start[t.id], end[t.id]))
    report = SimReport(
        makespan=makespan,
        decode_throughput=graph.tokens_generated / makespan if finite else 0.0,
        gpu_utilization=min(1.0, gpu_busy / makespan) if finite else 0.0,
        breakdown={k: min(1.0, v / makespan) for k, v in sorted(by_kind.items())} if finite else {},
        utilization_timeline=_bins(gpu_spans, makespan, bins) if finite else (),
        peak_gpu_bytes=graph.peak_gpu_bytes,
    )
    return timeline, report


def check_schedule(graph: TaskGraph, start, end) -> None:
    """One task at a time per lane, and no task before its dependencies (engine.py:103-119)."""
    lanes: dict[Resource, list[int]] = {}
    for t in graph.tasks:
        lanes.setdefault(t.resource, []).append(t.id)
    for ids in lanes.values():
        ids.sort(key=lambda i: (start[i], i))
        for a, b in zip(ids, ids[1:]):
            if end[a] > start[b]:
                raise AssertionError(f"resource overlap: task {a} ends {end[a]!r} after task {b} starts {start[b]!r}")
    for t in graph.tasks:
        for d in t.deps:
            if start[t.id] < end[d]:
                raise AssertionError(f"dependency violated: task {t.id} starts before dep {d} ends")


# ---------------------------------------------------------------------------
# exporters and the policy comparison table (pipesim/trace.py:17-110)

TRACE_LANES = {"h2d": 0, "gpu": 1, "d2h": 2}
METRICS_COLUMNS = ("policy", "schedule", "granularity", "recompute", "makespan_s", "throughput_tok_s", "gpu_util",
                   "peak_gpu_bytes")


def export_trace(timeline: Timeline) -> list[dict]:
    """Chrome trace events, one complete ("X") event per task, lanes h2d 0 / gpu 1 / d2h 2 (trace.py:30-43)."""
    return [{"name": e.name, "cat": e.kind, "ph": "X", "ts": e.start * 1e6, "dur": (e.end - e.start) * 1e6,
             "pid": 0, "tid": TRACE_LANES[e.resource]} for e in timeline.entries]


def write_trace(timeline: Timeline, path: str) -> None:
    """Compact, key-sorted JSON plus a newline: the reference's bytes (trace.py:46-49)."""
    with open(path, "w") as fh:
        json.dump(export_trace(timeline), fh, sort_keys=True, separators=(",", ":"))
        fh.write("\n")


def metrics_row(label: str, policy: Policy, report: SimReport) -> dict:
    return {"policy": label, "schedule": policy.schedule, "granularity": policy.granularity,
            "recompute": "on" if policy.recompute else "off", "makespan_s": report.makespan,
            "throughput_tok_s": report.decode_throughput, "gpu_util": report.gpu_utilization,
            "peak_gpu_bytes": report.peak_gpu_bytes}


def cell(value) -> str:
    """Floats by repr (round-trip exact), everything else by str (trace.py:73-76)."""
    return repr(value) if isinstance(value, float) else str(value)


def write_metrics_csv(rows, fh) -> None:
    """Fixed-schema metrics table; extra row keys are ignored (trace.py:65-70)."""
    w = csv.writer(fh, lineterminator="\n")
    w.writerow(METRICS_COLUMNS)
    for row in rows:
        w.writerow([cell(row[c]) for c in METRICS_COLUMNS])


def plan_for_policy(spec: ModelSpec, wl: WorkloadSpec, profile: HardwareProfile, policy: Policy) -> SplitPlan:
    """The solver's plan when recomputing, the all-zero plan for the naive baseline (trace.py:79-85)."""
    if policy.recompute:
        return plan_generation(spec, wl, profile, policy.schedule)
    return constant_plan(wl, policy.schedule, 0)


def compare(spec: ModelSpec, wl: WorkloadSpec, profile: HardwareProfile, policies, gpu_mem_budget=None,
            engine: str | None = None) -> list[dict]:
    """Simulate each (label, Policy) on one config; rows carry speedup_vs_first (trace.py:88-110)."""
    if not policies:
        raise ValueError("need at least one policy")
    rows, base = [], None
    for label, policy in policies:
        plan = plan_for_policy(spec, wl, profile, policy)
        _, rep = simulate(build_task_graph(spec, wl, profile, plan, policy, gpu_mem_budget), profile, engine=engine)
        row = metrics_row(label, policy, rep)
        if base is None:
            base = rep.makespan
        row["speedup_vs_first"] = base / rep.makespan if rep.makespan > 0 else 0.0
        rows.append(row)
    return rows
