"""Decode throughput of KVPR's offloaded decode path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl kvpr|reference] [--model opt-6.7b]
                    [--batch 32] [--prompt 1024]

Metric (BASELINE.json): decode tokens/s + per-layer latency, OPT-6.7B b32
prompt 1024, KV offloaded to host.  One "step" = one decode token for every
sequence of the batch through all layers: per layer H2D X[:, :l] + KV[l:s'-1]
from page-locked host stores, K1 recompute of K,V[0:l), K2 attention, the
rest of the OPT layer, D2H of the new X row and K,V page.  l per step comes
from the bit-exact split solver (column mode) fed by the live profile of
this GPU (profiler.measure -> hwprofile.calibrate).

value     device-timed (CUDA events, compute stream) tokens/s over K steps,
          inputs = the host stores (the workload defines them to live in
          host DRAM; they are streamed over PCIe inside every step).
e2e       the same through the public per-step API: prompt/next-token ids
          H2D from pinned host memory and the generated ids D2H every step,
          host-synchronised per step.
roofline  the per-layer overlap roofline of the north star,
          T_roof(l) = max(H2D bytes / BW_h2d_measured, recompute FLOPs / F_peak):
          achieved = algorithmic H2D bytes per layer / measured layer time.
          Kernel rooflines (K1 tensor, K2 HBM) are measured in the same run.
Multi-GPU (torchrun): the global batch (--batch, default 32) is partitioned
over the ranks (BASELINE config 3: b/G sequences per GPU), each rank with its
own host stores, PCIe link, profile and plan; no data-path collective.  Total
work is fixed as N grows (scaling "strong"), so the pinned host stores of all
ranks together stay at one batch's size however many GPUs run; the decode is
PCIe-bound, so tok/s per GPU is nearly independent of the slice size.
--impl reference: the reference's CPU path (split_merge_kv + decode_attention,
fp64 NumPy, restated in oracle/numerics_ref.py) timed on this host's cores.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        d["source"] = "measured"
        return d
    d = dict(PEAKS_FALLBACK)
    d["source"] = "fallback"
    return d


COMM_DEV = "cpu"  # where the timing reductions live: the rank's GPU under NCCL, host under gloo


def allreduce(vals, op="max"):
    """Max (or sum) of a few floats over the ranks; identity at world size 1."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return list(vals)
    t = torch.tensor(list(vals), dtype=torch.float64, device=COMM_DEV)
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return [float(x) for x in t.tolist()]


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ---------------------------------------------------------------------------
# CPU reference arm

def cpu_reference_sample(hidden, heads, seq_len, split, budget_s=12.0, max_reps=40, seed=0):
    """Time the reference CPU path for ONE sequence-layer: split_merge_kv + decode_attention (fp64)."""
    import numpy as np

    from oracle import numerics_ref as nr

    rng = np.random.default_rng(seed)
    x = rng.standard_normal((seq_len, hidden))
    w_k = rng.standard_normal((hidden, hidden)) * 0.02
    w_v = rng.standard_normal((hidden, hidden)) * 0.02
    w_o = rng.standard_normal((hidden, hidden)) * 0.02
    q = rng.standard_normal(hidden)
    k_suf = rng.standard_normal((heads, seq_len - split, hidden // heads))
    v_suf = rng.standard_normal((heads, seq_len - split, hidden // heads))
    suffix = nr.KVState(k_suf, v_suf)
    ts = []
    t_begin = time.perf_counter()
    while len(ts) < max_reps and (not ts or (time.perf_counter() - t_begin) < budget_s):
        t0 = time.perf_counter()
        kv = nr.split_merge_kv(x, split, w_k, w_v, suffix)
        nr.decode_attention(q, kv, w_o)
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts)), len(ts)


def cpu_oracle_e2e(cfg, w, prompt, splits, prompt_len):
    """the fp32 CPU OPT decoder (oracle/opt_ref.py: host X/KV stores, split-merge
    rebuild at the same l per step) end to end on this host, same weights and prompt; decode steps
    timed after an untimed prefill."""
    import numpy as np

    from oracle import opt_ref

    shape = opt_ref.OPTShape(cfg.hidden, cfg.layers, cfg.heads, cfg.ffn, cfg.vocab, cfg.max_pos, cfg.eps)
    o = opt_ref.OPTOracle(shape, w.numpy_dict(), prompt.shape[0], storage=np.float16, compute=np.float32)
    lg = o.prefill(prompt.numpy(), capacity=prompt_len + len(splits) + 1)
    tok = opt_ref.greedy(lg)
    t0 = time.perf_counter()
    for l in splits:
        tok = opt_ref.greedy(o.decode_step(tok, min(l, o.len + 1)))
    dt = time.perf_counter() - t0
    return {"value": prompt.shape[0] * len(splits) / dt, "unit": "tok/s", "cores": blas_threads(), "kind": "port",
            "sample": f"{len(splits)} decode steps x b{prompt.shape[0]} of the fp32 NumPy OPT decoder "
                      f"(oracle/opt_ref.py, host stores + split-merge rebuild), after an untimed prefill"}


def blas_threads():
    try:
        from threadpoolctl import threadpool_info

        return max((i.get("num_threads") or 0) for i in threadpool_info()) or os.cpu_count()
    except Exception:
        return os.cpu_count()


def use_all_host_threads():
    """torchrun exports OMP_NUM_THREADS=1 to every rank; the CPU reference arm is rank 0 alone, so it
    lifts the BLAS pool back to every host core."""
    try:
        from threadpoolctl import threadpool_limits

        threadpool_limits(limits=os.cpu_count())
    except Exception:
        pass


def bench_config(args, ws: int, cfg) -> dict:
    """The workload this line measures: identical in both arms (the driver compares them), so nothing
    run-dependent (profile, plan, timings) lives here; those go under "run"."""
    b = args.batch // (1 if args.tp else ws)
    return {
        "workload": f"{args.model} b{args.batch} prompt{args.prompt} decode, KV+X offloaded to pinned host",
        "geometry": cfg.describe(), "batch": args.batch, "batch_per_gpu": b, "prompt_len": args.prompt,
        "decode_steps_timed": args.steps, "mode": "column",
        "parallelism": f"tp{ws} (head-sharded)" if args.tp else f"batch-partition x{ws}",
        "l2": "inputs larger than L2: every step streams GBs of X/KV from host and reads all layer weights",
    }


def run_reference(args):
    """The reference arm: kvoverlap's CPU path for this workload (split_merge_kv + decode_attention in
    fp64 NumPy, restated in oracle/numerics_ref.py, which tests/golden pins to the live reference) on
    every host core.  One full step (b sequences x L layers) takes minutes on a CPU, so each timed
    "step" is a bounded sample: one sequence-layer at that step's (s', l); ms_per_step is the measured
    sample time and value is extrapolated to b x L sequence-layers (extrapolated: true)."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    use_all_host_threads()
    from paper_2411_17089_b200.costmodel import WorkloadSpec
    from paper_2411_17089_b200.hwprofile import HardwareProfile
    from paper_2411_17089_b200.scheduler import plan_generation
    from paper_2411_17089_b200.weights import preset

    cfg = preset(args.model)
    b = args.batch // (1 if args.tp else ws)
    wl = WorkloadSpec(batch_size=b, prompt_len=args.prompt, gen_len=args.warmup + args.steps)
    # no GPU probe on this arm: the split comes from the reference solver on the B200-guess profile
    # (within ~2% of the live-profile l the kvpr arm uses; the CPU time is flat in l there)
    prof = HardwareProfile(gpu_flops=1391.2e12, h2d_bandwidth=55e9, d2h_bandwidth=55e9)
    plan = plan_generation(cfg.spec(), wl, prof, "column")
    sample_s, reps = [], 0
    t_wall0 = time.perf_counter()
    d0 = plan.decisions[0]
    cpu_reference_sample(cfg.hidden, cfg.heads, d0.seq_len, d0.recompute_len, budget_s=1.0, max_reps=2)  # BLAS pool
    for i in range(args.warmup + args.steps):
        d = plan.decisions[i]
        t, n = cpu_reference_sample(cfg.hidden, cfg.heads, d.seq_len, d.recompute_len, budget_s=2.0, max_reps=3,
                                    seed=i)
        if i >= args.warmup:
            sample_s.append(t)
            reps += n
    t_seq_layer = sum(sample_s) / len(sample_s)
    full_step_s = t_seq_layer * cfg.layers * args.batch  # every sequence of the job, all layers
    value = args.batch / full_step_s
    cores = blas_threads()
    sample = (f"per timed step: median of 3 runs of 1 sequence x 1 layer of split_merge_kv + decode_attention "
              f"(fp64 NumPy, {cores} BLAS threads) at that step's (s', l); value extrapolated x{args.batch} "
              f"sequences x{cfg.layers} layers")
    line = {
        "metric": "decode_tokens_per_s", "value": value, "unit": "tok/s", "impl": "reference",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_seq_layer * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(args, ws, cfg),
        "extrapolated": True,
        "extrapolation": {"sampled_sequence_layers_per_step": 1, "sequence_layers_per_full_step": args.batch * cfg.layers,
                          "ms_per_full_step": full_step_s * 1e3, "sample_runs": reps},
        "run": {"plan_profile": "b200-guess (1391.2e12 FLOP/s, 55e9 B/s), reference solver, column",
                "splits_timed": plan.splits[args.warmup:]},
        "cpu_baseline": {"value": value, "unit": "tok/s", "cores": cores, "kind": "port", "sample": sample,
                         "host_cpus": os.cpu_count()},
        "e2e": {"value": value, "unit": "tok/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": time.perf_counter() - t_wall0,
    }
    print(json.dumps(line))


# ---------------------------------------------------------------------------
# clocks sampler

class Clocks:
    def __init__(self):
        self.nvml = []
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("pci.bus_id,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-lms",
                                       "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    @staticmethod
    def _pci(gpu_index):
        """The CUDA device's PCI address (nvidia-smi / NVML enumerate in their own order)."""
        from paper_2411_17089_b200.multigpu import pci_address

        return pci_address(gpu_index)

    def sample_now(self, gpu_index=0):
        """One in-process NVML sample (for timed regions shorter than nvidia-smi's 200 ms period):
        call it while the GPU is busy with the timed work."""
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByPciBusId(self._pci(gpu_index).encode())
            sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
            names = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
                     "sw_power_cap": 0x4}
            self.nvml.append((float(sm), float(mx), sorted(n for n, bit in names.items() if r & bit)))
        except Exception as e:  # pragma: no cover - best effort
            self.nvml_error = str(e)

    def stop(self, gpu_index=0):
        if self.p is None and not self.nvml:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        if self.p is not None:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except Exception:
                self.p.kill()
        self.f.flush()
        rows = []
        pci = self._pci(gpu_index)
        for line in Path(self.f.name).read_text().splitlines():
            c = [x.strip() for x in line.split(",")]
            if len(c) >= 9 and c[0].lower().endswith(pci[-12:].lower()):
                rows.append(c)
        if not rows:
            if self.nvml:  # region shorter than the nvidia-smi period: the in-process NVML samples
                sm = sorted(x[0] for x in self.nvml)
                return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": self.nvml[0][1],
                        "reasons": sorted({n for x in self.nvml for n in x[2]}), "samples": len(sm),
                        "source": "nvml in-process (timed region shorter than the nvidia-smi period)"}
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = sorted(float(r[1]) for r in rows)
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for n, v in zip(names, r[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": float(rows[0][2]), "reasons": sorted(reasons),
                "samples": len(rows), "power_w_max": max(float(r[3]) for r in rows if r[3] not in ("", "[N/A]"))}


# ---------------------------------------------------------------------------
# B200 arm

def _events_time(rt, fn, dev) -> float:
    """Seconds of fn()'s GPU work on rt.cs, CUDA events on both sides, synchronised."""
    import torch

    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    a.record(rt.cs)
    fn()
    e.record(rt.cs)
    torch.cuda.synchronize(dev)
    return a.elapsed_time(e) / 1e3


def k1_launch_shapes(rt, plan_decisions, warmup, batch, hidden, sms):
    """(positions, tile) of every K1 launch the runtime issues for the timed steps (runtime.chunk_bounds,
    the executor's chunking) with kvpr_recompute_tile's choice for each."""
    from paper_2411_17089_b200 import _lib
    from paper_2411_17089_b200.runtime import chunk_bounds

    lib = _lib.load()
    out = []
    for d in plan_decisions[warmup:]:
        lp = min(d.recompute_len, d.seq_len - 1)
        if rt.x_resident:
            bounds = [(0, lp)] if lp else []
        else:
            bounds = chunk_bounds(lp, rt.chunks, rt.chunk_rows, rt.chunk_wave)
        for p0, p1 in bounds:
            out.append((p1 - p0, lib.kvpr_recompute_tile(batch, p1 - p0, hidden, sms)))
    return out


TILE_NAMES = {512: "tcgen05 cta_group::2, 256x256 CTA-pair tile, TMA, TMEM"}


def tile_name(bn: int) -> str:
    return TILE_NAMES.get(bn, f"tcgen05 1-CTA 128x{bn} tile, TMA, TMEM")


def k1_traffic(batch: int, hidden: int, positions: int, tile: int):
    """ncu dram read+write per launch for exactly this K1 launch shape, if one was captured
    (profiles/k1_traffic.json, written from `ncu --set full` captures), else None."""
    p = ROOT / "profiles" / "k1_traffic.json"
    if not p.exists():
        return None
    for rec in json.loads(p.read_text()).get("captures", []):
        if (rec["batch"], rec["hidden"], rec["positions"], rec["tile"]) == (batch, hidden, positions, tile):
            return rec
    return None


def run_config1(args, dev, peaks):
    """BASELINE config 1 in the same run: OPT-125M shape, b4, prompt 256, 16 decode tokens, live profile,
    reference solver (column).  Device-timed and end to end (host ids in/out every step)."""
    import torch

    from paper_2411_17089_b200 import _lib, profiler
    from paper_2411_17089_b200.costmodel import WorkloadSpec, activation_bytes, kv_remainder_bytes
    from paper_2411_17089_b200.runtime import KVPRRuntime
    from paper_2411_17089_b200.scheduler import overlap_roofline, plan_generation
    from paper_2411_17089_b200.weights import OPTWeights, preset

    cfg, b, S0, gen = preset("opt-125m"), 4, 256, 16
    calib, recs = profiler.measure(cfg.hidden, b, device=dev)
    prof, bw = calib.profile, profiler.peak_h2d(recs)
    wl = WorkloadSpec(batch_size=b, prompt_len=S0, gen_len=gen)
    plan = plan_generation(cfg.spec(), wl, prof, "column")
    w = OPTWeights.random(cfg, seed=0, device=dev)
    prompt = torch.randint(0, cfg.vocab, (b, S0), generator=torch.Generator().manual_seed(1))
    rt = KVPRRuntime(w, b, S0 + gen + 1, device=dev)
    first = rt.prefill(prompt)
    rt.decode(plan.splits[:4], tokens=first)  # warmup
    rt.reset(S0)
    lib = _lib.load()
    n0 = lib.kvpr_kernel_launches()
    t = _events_time(rt, lambda: rt.decode(plan.splits, tokens=first), dev)
    launches = lib.kvpr_kernel_launches() - n0
    f_peak = peaks["bf16_tflops_sustained"] * 1e12
    spec, L = cfg.spec(), cfg.layers
    troof = sum(overlap_roofline(spec, wl, d.seq_len - 1, min(d.recompute_len, d.seq_len - 1), bw, f_peak) * L
                for d in plan.decisions)
    h2d = sum((activation_bytes(spec, wl, min(d.recompute_len, d.seq_len - 1)) +
               kv_remainder_bytes(spec, wl, d.seq_len - 1, min(d.recompute_len, d.seq_len - 1))) * L
              for d in plan.decisions)
    # end to end: ids H2D from pinned host, one step per call, generated ids D2H, host-synchronised
    rt.reset(S0)
    tok_host = torch.empty(b, dtype=torch.int32, pin_memory=True)
    tok_host.copy_(first.cpu())
    torch.cuda.synchronize(dev)
    te0 = time.perf_counter()
    for l in plan.splits:
        out = rt.decode([l], tokens=tok_host.to(dev, non_blocking=True))
        tok_host.copy_(out[0], non_blocking=True)
        torch.cuda.current_stream(dev).synchronize()
    e2e_s = time.perf_counter() - te0
    rt.close()
    return {"value": b * gen / t, "unit": "tok/s", "ms_per_step": t / gen * 1e3, "steps": gen,
            "workload": "opt-125m shape (h768 x12, 12 heads), b4, prompt 256, 16 decode tokens, KV+X on pinned host",
            "splits": plan.splits, "overlap_roofline_frac": troof / t, "h2d_bytes_per_step": int(h2d / gen),
            "gpu_launches": launches, "launches_per_step": launches / gen,
            "e2e": {"value": b * gen / e2e_s, "unit": "tok/s", "steps": gen, "h2d_bytes_per_step": int(h2d / gen) + 4 * b,
                    "d2h_bytes_per_step": 3 * b * cfg.hidden * 2 * L + 4 * b},
            "profile": {"h2d_bandwidth": prof.h2d_bandwidth, "gpu_flops": prof.gpu_flops, "bw_peak": bw}}


def run_config5(args, dev, peaks, prof, bw, prompts=(512, 1024, 2048, 4096, 8192), layers=2, steps=3, grid=8):
    """BASELINE config 5: OPT-6.7B layer shapes, b32, per-layer decode latency at prompts 512..8192 for
    l = 0 (naive offload), the reference solver's l (column, live profile), l = s' and a forced-l grid
    (steps of max(64, s'/grid) over [0, s']); reports T_roof fractions and the measured argmin over all
    points (scheduler-chosen l vs measured optimum).  Per-layer latency is
    what is compared, so `layers` of the 32 identical layers bound the host stores (6.4 GB per layer at
    prompt 8192)."""
    import statistics

    import torch

    from paper_2411_17089_b200.costmodel import WorkloadSpec
    from paper_2411_17089_b200.runtime import DecodeTiming, KVPRRuntime
    from paper_2411_17089_b200.scheduler import layer_time, overlap_roofline, solve_split
    from paper_2411_17089_b200.weights import OPTConfig, OPTWeights, preset

    base, b = preset("opt-6.7b"), 32
    f_peak = peaks["bf16_tflops_sustained"] * 1e12
    out = []
    for P in prompts:
        cfg = OPTConfig(base.hidden, layers + 1, base.heads, base.ffn, base.vocab, max(base.max_pos, P + 16))
        w = OPTWeights.random(cfg, seed=0, device=dev)
        prompt = torch.randint(0, cfg.vocab, (b, P), generator=torch.Generator().manual_seed(1))
        rt = KVPRRuntime(w, b, P + steps + 1, device=dev)
        first = rt.prefill(prompt)
        spec, s1 = cfg.spec(), P + 1
        wl = WorkloadSpec(batch_size=b, prompt_len=P, gen_len=steps)
        l_sched = solve_split(spec, wl, prof, s1, "column").recompute_len
        pts = []
        step_l = max(64, -(-s1 // grid // 64) * 64)
        forced = [("grid", l) for l in range(step_l, s1, step_l) if l != l_sched]
        for name, l in [("naive", 0), ("solver", l_sched), ("full", s1)] + forced:
            rt.reset(P)
            tim = DecodeTiming()
            rt.decode([min(l, P + 1 + i) for i in range(steps)], tokens=first, timing=tim)
            per_layer = [x for row in tim.layer_ms for x in row[1:]]  # layer 0 carries the embed + pipeline fill
            med = statistics.median(per_layer)
            lp = min(l, s1 - 1)
            troof = overlap_roofline(spec, wl, s1 - 1, lp, bw, f_peak) * 1e3
            pts.append({"plan": name, "l": l, "layer_ms": med, "troof_ms": troof, "frac": troof / med,
                        "ref_pred_column_ms": layer_time(spec, wl, prof, s1, l, "column").total * 1e3})
        best = min(pts, key=lambda r: r["layer_ms"])
        sched = next(r for r in pts if r["plan"] == "solver")
        out.append({"prompt": P, "l_sched": l_sched, "l_grid_step": step_l, "points": pts,
                    "measured_argmin_l": best["l"], "sched_vs_measured_opt": best["layer_ms"] / sched["layer_ms"]})
        rt.close()
        del rt, w
        torch.cuda.empty_cache()
    return {"model": "opt-6.7b layer shapes, b32", "layers_timed_per_step": layers, "steps": steps,
            "note": "per-layer latency (median over steps of layers 2..L, CUDA events on the compute stream); "
                    "T_roof = max(H2D(X[:, :l] + KV[l:s'-1]) / measured pinned H2D peak, 4 b l h^2 / sustained "
                    "bf16 peak); sched_vs_measured_opt = measured optimum layer time / layer time at the "
                    "reference solver's l (1.0 = the solver's l is the measured optimum)",
            "prompts": out}


def run_kvpr(args):
    import torch
    import torch.distributed as dist

    from paper_2411_17089_b200 import _lib, kernels, profiler
    from paper_2411_17089_b200.costmodel import WorkloadSpec, activation_bytes, kv_remainder_bytes, recompute_flops
    from paper_2411_17089_b200.runtime import DecodeTiming, KVPRRuntime
    from paper_2411_17089_b200.scheduler import overlap_roofline, plan_generation
    from paper_2411_17089_b200.weights import OPTWeights, preset

    global COMM_DEV
    ws, rank, local = dist_env()
    # KVPR_BENCH_SHARE_GPU=1: test mode for the multi-rank path on a 1-GPU box (ranks share cuda:0,
    # reductions over gloo, since NCCL refuses two ranks on one device)
    share = os.environ.get("KVPR_BENCH_SHARE_GPU") == "1"
    gpu = local % torch.cuda.device_count() if share else local
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    from paper_2411_17089_b200.multigpu import bind_to_gpu_numa

    numa = bind_to_gpu_numa(gpu)  # before any pinned allocation: this rank's host stores on its GPU's socket
    if ws > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
            COMM_DEV = dev
        args.no_alt = True  # alt lines are single-GPU context; N ranks x their host stores would crowd host DRAM
    peaks = load_peaks()
    cfg = preset(args.model)
    cfg = cfg.with_positions(args.prompt + args.warmup + args.steps + 8)
    from paper_2411_17089_b200.multigpu import partition

    gb = args.batch  # global batch: TP runs all of it on every rank, batch partition a b/G slice per rank
    sl = partition(gb, 1 if args.tp else ws)[0 if args.tp else rank]
    b = sl.count
    total_steps = args.warmup + args.steps
    wl = WorkloadSpec(batch_size=b, prompt_len=args.prompt, gen_len=total_steps)
    spec, L = cfg.spec(), cfg.layers
    sms = torch.cuda.get_device_properties(dev).multi_processor_count

    # profiler -> scheduler (bit-exact solver on the live profile); under TP every rank
    # must run the same plan, so rank 0's profile is broadcast
    if args.fixed_profile:  # e.g. under ncu, where the probe timings are replay artefacts
        from paper_2411_17089_b200.hwprofile import HardwareProfile

        prof, bw_peak = HardwareProfile(gpu_flops=1391.2e12, h2d_bandwidth=55e9, d2h_bandwidth=55e9), 55e9
    else:
        calib, recs = profiler.measure(cfg.hidden, b if not args.tp else max(1, b // ws), device=dev)
        prof = calib.profile
        bw_peak = profiler.peak_h2d(recs)
    if args.tp and ws > 1:
        obj = [prof, bw_peak]
        dist.broadcast_object_list(obj, src=0)
        prof, bw_peak = obj
    plan = plan_generation(spec, wl, prof, "column")
    splits = plan.splits

    try:  # host stores are page-locked: warn early if the ranks of this node will not fit in DRAM
        import psutil

        need = L * (args.prompt + total_steps + 1) * b * cfg.hidden * 2 * 3
        local_ws = int(os.environ.get("LOCAL_WORLD_SIZE", "1"))
        avail = psutil.virtual_memory().available
        if need * local_ws > 0.9 * avail:
            print(f"warning: {local_ws} ranks x {need / 2**30:.1f} GiB of pinned host stores vs "
                  f"{avail / 2**30:.1f} GiB available", file=sys.stderr)
    except ImportError:
        pass
    w = OPTWeights.random(cfg, seed=0, device=dev)
    weights_bytes = w.nbytes()
    g = torch.Generator().manual_seed(1)
    prompt = torch.randint(0, cfg.vocab, (gb, args.prompt), generator=g)[sl.start:sl.start + b]  # this rank's rows
    if args.tp:
        from paper_2411_17089_b200.tp import TPRuntime

        rt = TPRuntime(w, b, args.prompt + total_steps + 1, device=dev)
        del w.layers[:]  # full-width layer weights are no longer needed once sharded
        torch.cuda.empty_cache()
        args.no_alt = True
    else:
        rt = KVPRRuntime(w, b, args.prompt + total_steps + 1, device=dev)
    t0 = time.perf_counter()
    first = rt.prefill(prompt)
    prefill_s = time.perf_counter() - t0

    # warmup steps (untimed)
    rt.decode(splits[: args.warmup], tokens=first)
    torch.cuda.synchronize(dev)
    if ws > 1:
        dist.barrier()
    clocks = Clocks() if rank == 0 else None
    lib = _lib.load()
    launches0 = lib.kvpr_kernel_launches()  # every kernel libkvpr launches in this process
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    # the timed region: K steps as a user runs them (no per-kernel instrumentation on the path)
    host_t0 = time.time()
    start.record(rt.cs)
    rt.decode(splits[args.warmup:])
    end.record(rt.cs)
    if clocks:
        clocks.sample_now(gpu)  # the decode is enqueued and running
    torch.cuda.synchronize(dev)
    host_t1 = time.time()
    launches = lib.kvpr_kernel_launches() - launches0
    launches = int(allreduce([launches], op="sum")[0])  # all ranks
    elapsed = start.elapsed_time(end) / 1e3
    clk = clocks.stop(gpu) if clocks else None
    rank_elapsed = elapsed
    elapsed = allreduce([elapsed])[0]
    value = gb * args.steps / elapsed  # every rank's slice, over the slowest rank's time
    windows = None
    if ws > 1:  # per-rank host windows of the timed region: the driver can check the ranks overlapped
        got = [None] * ws
        dist.all_gather_object(got, (rank, host_t0, host_t1, rank_elapsed, b))
        t_min = min(x[1] for x in got)
        windows = [{"rank": r, "start_s": a - t_min, "end_s": e - t_min, "device_s": d, "batch": bb}
                   for r, a, e, d, bb in sorted(got)]

    # instrumented replay of the same K steps (same splits, same start length): CUDA events around
    # every K1 / K2 launch and after every layer give the per-layer latency and the kernel rooflines
    tim = DecodeTiming()
    kstats = {}
    if hasattr(rt, "reset"):
        rt.reset(args.prompt + args.warmup)
        if hasattr(rt, "kernel_timing"):
            rt.kernel_timing = []
        rt.decode(splits[args.warmup:], timing=tim)
        torch.cuda.synchronize(dev)
        kstats = rt.kernel_stats() if hasattr(rt, "kernel_stats") else {}
        if hasattr(rt, "kernel_timing"):
            rt.kernel_timing = None

    # per-layer latency and overlap roofline over the timed steps.  The runtime ships X[:, :l'] and
    # KV[l':s'-1] with l' = min(l, s'-1) (the new position's k, v come from the q/k/v projection),
    # so T_roof counts exactly those bytes and 4 b l' h^2 FLOPs
    layer_ms = [x for row in tim.layer_ms for x in row[1:]]  # drop each step's first layer (embed + fill)
    steady_layer_s = (sorted(layer_ms)[len(layer_ms) // 2] / 1e3) if layer_ms else elapsed / (args.steps * L)
    f_peak = peaks["bf16_tflops_sustained"] * 1e12
    troof, h2d_alg, flops_alg = 0.0, 0.0, 0.0
    for d in plan.decisions[args.warmup:]:
        lp = min(d.recompute_len, d.seq_len - 1)
        troof += overlap_roofline(spec, wl, d.seq_len - 1, lp, bw_peak, f_peak) * L
        h2d_alg += (activation_bytes(spec, wl, lp) + kv_remainder_bytes(spec, wl, d.seq_len - 1, lp)) * L
        flops_alg += recompute_flops(spec, wl, lp) * L
    achieved_gbs = h2d_alg / elapsed / 1e9

    # alternate plan (extension, not the reference solver): the runtime's own overlap objective
    alt = None
    if not args.no_alt:
        from paper_2411_17089_b200.scheduler import plan_generation_overlap

        alt_splits = plan_generation_overlap(spec, wl, prof).splits[args.warmup:]
        rt.reset(args.prompt + args.warmup)
        alt_s = _events_time(rt, lambda: rt.decode(alt_splits, tokens=first), dev)
        alt = {"value": gb * args.steps / alt_s, "unit": "tok/s", "splits": alt_splits,
               "ms_per_step": alt_s / args.steps * 1e3,
               "note": "extension objective max(t_act + t_kv, t_rec) of the chunked pipeline "
                       "(scheduler.solve_split_overlap); l differs from the reference's column solver, "
                       "so this is NOT the headline"}

    # kernel rooflines, measured on the compute stream after the timed region
    mid = plan.decisions[args.warmup + args.steps // 2]
    lmid = min(mid.recompute_len, mid.seq_len - 1)
    kern = {}
    if rank == 0 and not args.tp:
        lw = w.layers[0]
        xd, kvd = rt.x_dev[0], rt.kv_dev[0]

        def ev_time(fn, reps=10):
            for _ in range(3):
                fn()
            a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(rt.cs)
            for _ in range(reps):
                fn()
            e.record(rt.cs)
            e.synchronize()
            return a.elapsed_time(e) / reps / 1e3

        if lmid > 0:
            t_k1 = ev_time(lambda: kernels.recompute_kv(xd, lw.w_kv, lw.b_kv, kvd, b, 0, lmid, stream=rt.cs))
            fl = recompute_flops(spec, wl, lmid)
            kern["k1_recompute_gemm_standalone"] = {"bound": "tensor", "achieved": fl / t_k1 / 1e12,
                                         "peak": peaks["bf16_tflops"], "unit": "TFLOP/s",
                                         "frac": fl / t_k1 / 1e12 / peaks["bf16_tflops"], "traffic": None,
                                         "us": t_k1 * 1e6, "M": b * lmid, "N": 2 * cfg.hidden, "K": cfg.hidden,
                                         "tile": tile_name(lib.kvpr_recompute_tile(b, lmid, cfg.hidden, sms))}
        s = mid.seq_len
        t_k2 = ev_time(lambda: kernels.decode_attention(rt.q, kvd, rt.attn, rt.ws, b, cfg.heads, cfg.head_dim, s,
                                                        stream=rt.cs))
        by = 2 * b * s * cfg.hidden * 2
        kern["k2_decode_attention_standalone"] = {"bound": "hbm", "achieved": by / t_k2 / 1e9, "peak": peaks["hbm_gbs"],
                                       "unit": "GB/s", "frac": by / t_k2 / 1e9 / peaks["hbm_gbs"], "traffic": None,
                                       "us": t_k2 * 1e6}
        # the decode projections stream their weights from HBM (L2-cold: 13 GB of weights cycle through
        # between two uses of a layer in the step); timed back to back over 4 different layers
        acc = _lib.EPI_F32 | _lib.EPI_ACCUM
        lws = [w.layers[j] for j in range(min(4, L))]
        for name, fn_of, nbytes in (
                ("out_proj", lambda q: kernels.linear_simple(rt.attn, q.wo, q.bo, rt.hres, flags=acc, stream=rt.cs,
                                                             ws=rt.ws), cfg.hidden * cfg.hidden * 2),
                ("fc1", lambda q: kernels.linear_simple(rt.y, q.w1, q.b1, rt.mid, flags=_lib.EPI_RELU, stream=rt.cs,
                                                        ws=rt.ws), cfg.ffn * cfg.hidden * 2),
                ("fc2", lambda q: kernels.linear_simple(rt.mid, q.w2, q.b2, rt.hres, flags=acc, stream=rt.cs,
                                                        ws=rt.ws), cfg.ffn * cfg.hidden * 2)):
            t = ev_time(lambda: [fn_of(q) for q in lws], reps=5) / len(lws)
            kern[f"decode_{name}_standalone"] = {"bound": "hbm", "achieved": nbytes / t / 1e9,
                                                 "peak": peaks["hbm_gbs"], "unit": "GB/s",
                                                 "frac": nbytes / t / 1e9 / peaks["hbm_gbs"], "us": t * 1e6,
                                                 "M": b, "weight_bytes": nbytes}
        # In the step, K2 is ONE launch per layer and always runs while the copy engine streams the
        # next layer's X / KV into HBM (that is the overlap).  Its ceiling there: single launches
        # (each timed alone, median; back-to-back launches overlap their ramp and tail under PDL)
        # with a host->device DMA in flight on the H2D stream (tools/k2_probe.py isolates the effect).
        def single_time(fn, reps=9):
            ts = []
            for _ in range(reps):
                a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(rt.cs)
                fn()
                e.record(rt.cs)
                e.synchronize()
                ts.append(a.elapsed_time(e) / 1e3)
            return sorted(ts)[len(ts) // 2]

        k2_call = lambda: kernels.decode_attention(rt.q, kvd, rt.attn, rt.ws, b, cfg.heads,  # noqa: E731
                                                   cfg.head_dim, s, stream=rt.cs)
        t_k2s = single_time(k2_call)
        kern["k2_decode_attention_single_launch"] = {"bound": "hbm", "achieved": by / t_k2s / 1e9,
                                                     "peak": peaks["hbm_gbs"], "unit": "GB/s",
                                                     "frac": by / t_k2s / 1e9 / peaks["hbm_gbs"],
                                                     "us": t_k2s * 1e6}
        if hasattr(rt, "stores") and rt.stores.x is not None and rt.nbuf > 1:
            src = rt.stores.x[1]
            n = min(src.numel() * src.element_size(), rt.x_dev[1].numel() * rt.x_dev[1].element_size())
            rt.hs.wait_stream(rt.cs)
            _lib.call("kvpr_copy_async", rt.x_dev[1].data_ptr(), src.data_ptr(), n, rt.hs.cuda_stream)
            t0_dma = time.perf_counter()
            t_k2c = single_time(k2_call)
            span = time.perf_counter() - t0_dma
            rt.hs.synchronize()
            if n / 55e9 > span:  # the DMA outlasted all the timed launches
                kern["k2_decode_attention_single_launch_dma"] = {
                    "bound": "hbm", "achieved": by / t_k2c / 1e9, "unit": "GB/s", "us": t_k2c * 1e6,
                    "dma_bytes": n, "note": "single launches with a concurrent pinned H2D on the copy engine "
                                            "(the in-step condition)"}

    # e2e through the public per-step API over ALL timed steps: this step's ids H2D from pinned host
    # memory, one decode step (its X/KV streamed from the host stores inside), the generated ids D2H
    rt.reset(args.prompt + args.warmup)
    tok_host = torch.empty(b, dtype=torch.int32, pin_memory=True)
    tok_host.copy_(first.cpu())
    torch.cuda.synchronize(dev)
    if ws > 1:
        dist.barrier()
    te0 = time.perf_counter()
    for i in range(args.steps):
        out = rt.decode([splits[args.warmup + i]], tokens=tok_host.to(dev, non_blocking=True))
        tok_host.copy_(out[0], non_blocking=True)
        torch.cuda.current_stream(dev).synchronize()
    e2e_s = time.perf_counter() - te0
    e2e_s = allreduce([e2e_s])[0]
    e2e_value = gb * args.steps / e2e_s
    h2d_step = h2d_alg / args.steps + b * 4
    d2h_step = (3 * b * cfg.hidden * 2) * L + b * 4
    if ws > 1 and not args.tp:  # whole-job bytes
        h2d_step, d2h_step = allreduce([h2d_step, d2h_step], op="sum")

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:  # the CPU baseline is an N=1 measurement
        t_seq_layer, n = cpu_reference_sample(cfg.hidden, cfg.heads, mid.seq_len, mid.recompute_len,
                                              budget_s=args.cpu_budget)
        cpu_tok_s = 1.0 / (t_seq_layer * L)
        cpu = {"value": cpu_tok_s, "unit": "tok/s", "cores": blas_threads(), "kind": "port",
               "sample": (f"{n} reps of one sequence-layer split_merge_kv+decode_attention (fp64 NumPy, "
                          f"oracle/numerics_ref.py) at s'={mid.seq_len}, l={mid.recompute_len}; "
                          f"tok/s = 1/(t x {L} layers)"),
               "host_cpus": os.cpu_count()}
        if cfg.hidden * cfg.layers <= 1024 * 24:  # config-1-sized: the whole CPU decoder fits the budget
            cpu["oracle_e2e"] = cpu_oracle_e2e(cfg, w, prompt, splits[args.warmup:args.warmup + 4], args.prompt)

    # K1 (dominant kernel) launch shapes of the timed steps, before the headline runtime goes away
    shapes = k1_launch_shapes(rt, plan.decisions, args.warmup, b, cfg.hidden, sms) if not args.tp else []

    # row schedule (the reference's other mode, graph.py:16-17): X resident in HBM, only KV[l:] on PCIe
    alt_row = None
    if not args.no_alt and not args.tp:
        rt.close()
        del rt
        torch.cuda.empty_cache()
        plan_r = plan_generation(spec, wl, prof, "row")
        rt = KVPRRuntime(w, b, args.prompt + total_steps + 1, device=dev, x_resident=True)
        fr = rt.prefill(prompt)
        rt.decode(plan_r.splits[: args.warmup], tokens=fr)
        row_s = _events_time(rt, lambda: rt.decode(plan_r.splits[args.warmup:]), dev)
        troof_r, tgpu_r = 0.0, 0.0
        hbm = peaks["hbm_gbs"] * 1e9
        for d in plan_r.decisions[args.warmup:]:
            lp = min(d.recompute_len, d.seq_len - 1)
            t_rec = recompute_flops(spec, wl, lp) / f_peak
            troof_r += max(kv_remainder_bytes(spec, wl, d.seq_len - 1, lp) / bw_peak, t_rec) * L
            # the rest of the layer streams its weights (~12 h^2 fp16) and the whole KV cache (K2) from HBM
            # on the same SMs K1 occupies, so a GPU-bound row step is at best K1 + that, serially
            rest = (12 * cfg.hidden * cfg.hidden * 2 + 2 * b * d.seq_len * cfg.hidden * 2) / hbm
            tgpu_r += (t_rec + rest) * L
        alt_row = {"value": gb * args.steps / row_s, "unit": "tok/s", "splits": plan_r.splits[args.warmup:],
                   "ms_per_step": row_s / args.steps * 1e3, "roofline_frac": troof_r / row_s,
                   "gpu_serial_roofline_frac": tgpu_r / row_s,
                   "note": "row schedule: layer inputs X resident in HBM (8.9 GB), only KV[l:s'-1] over PCIe; "
                           "reference solver in mode 'row' (t_act = 0); roofline max(KV bytes/BW, FLOPs/F_sust); "
                           "GPU-bound, so also gpu_serial_roofline_frac = (K1 FLOPs/F_sust + decode weights and "
                           "KV-cache HBM bytes/HBM peak) / measured"}

    # compressed KV offload (§8f: 4-bit groupwise KV, kv_bytes_per_element 0.5625), same model / batch
    alt_kv4 = None
    if not args.no_alt and not args.tp:
        rt.close()
        del rt
        torch.cuda.empty_cache()
        wl4 = WorkloadSpec(batch_size=b, prompt_len=args.prompt, gen_len=total_steps, kv_bytes_per_element=0.5625)
        plan4 = plan_generation(spec, wl4, prof, "column")
        rt = KVPRRuntime(w, b, args.prompt + total_steps + 1, device=dev, kv_bits=4)
        f4 = rt.prefill(prompt)
        rt.decode(plan4.splits[: args.warmup], tokens=f4)
        kv4_s = _events_time(rt, lambda: rt.decode(plan4.splits[args.warmup:]), dev)
        troof4 = sum(overlap_roofline(spec, wl4, d.seq_len - 1, min(d.recompute_len, d.seq_len - 1), bw_peak,
                                      f_peak) * L for d in plan4.decisions[args.warmup:])
        alt_kv4 = {"value": gb * args.steps / kv4_s, "unit": "tok/s", "splits": plan4.splits[args.warmup:],
                   "ms_per_step": kv4_s / args.steps * 1e3, "roofline_frac": troof4 / kv4_s,
                   "note": "KV cache stored and streamed as 4-bit groupwise pages (0.5625 B/elem, lossy); "
                           "reference solver with kv_bytes_per_element=0.5625; not the headline workload"}

    # BASELINE configs 1 and 5 in the same run (single GPU), after the headline runtime is released
    alt_c1 = alt_c5 = None
    if not args.no_alt and not args.tp:
        rt.close()
        del rt, w
        torch.cuda.empty_cache()
        rt = None
        if not args.no_config1:
            alt_c1 = run_config1(args, dev, peaks)
        if not args.no_config5:
            alt_c5 = run_config5(args, dev, peaks, prof, bw_peak)

    # dominant kernel (K1) roofline from the launches inside the timed region (events on its stream)
    k1_roof = None
    if "k1" in kstats:
        n, t, fl = kstats["k1"]
        from collections import Counter

        (pos_mode, tile_mode), n_mode = Counter(shapes).most_common(1)[0] if shapes else ((0, 0), 0)
        cap = k1_traffic(b, cfg.hidden, pos_mode, tile_mode)
        k1_roof = {"bound": "tensor", "kernel": f"K1 recompute GEMM ({tile_name(tile_mode)})",
                   "achieved": fl / t / 1e12, "peak": peaks["bf16_tflops_sustained"], "unit": "TFLOP/s",
                   "frac": fl / t / 1e12 / peaks["bf16_tflops_sustained"],
                   "traffic": cap["dram_bytes_per_launch"] if cap else None,
                   "launches": n, "flops_per_launch": fl, "us_per_launch": t * 1e6,
                   "launch_shapes": {"modal_positions": pos_mode, "modal_tile": tile_mode, "modal_count": n_mode,
                                     "total": len(shapes), "M": pos_mode * b, "N": 2 * cfg.hidden, "K": cfg.hidden},
                   "algorithmic_bytes_per_launch": cap["algorithmic_bytes_per_launch"] if cap else None,
                   "frac_vs_burst": fl / t / 1e12 / peaks["bf16_tflops"],
                   "traffic_note": (f"ncu dram read+write of one launch of the modal shape ({cap['source']})" if cap
                                    else "no ncu capture of this launch shape (profiles/k1_traffic.json)"),
                   "peak_note": "sustained bf16 (kernel timed inside a long step); "
                                f"burst {peaks['bf16_tflops']} TFLOP/s.  The step is PCIe-bound, so the "
                                "tensor cores idle ~2/3 of it and K1 can clock above a back-to-back "
                                "GEMM's sustained rate (frac > 1 is possible; frac_vs_burst bounds it)"}
    if "k2" in kstats:
        n, t, by = kstats["k2"]
        kern["k2_decode_attention_in_step"] = {"bound": "hbm", "achieved": by / t / 1e9, "peak": peaks["hbm_gbs"],
                                               "unit": "GB/s", "frac": by / t / 1e9 / peaks["hbm_gbs"],
                                               "launches": n, "us_per_launch": t * 1e6}
        if "k2_decode_attention_single_launch_dma" in kern:
            c = kern["k2_decode_attention_single_launch_dma"]["achieved"]
            kern["k2_decode_attention_in_step"].update(
                {"frac_vs_dma_ceiling": by / t / 1e9 / c,
                 "note": "frac_vs_dma_ceiling: vs single launches of the same K2 timed with a concurrent H2D "
                         "(the in-step condition)"})

    copy_stream = None
    if "h2d" in kstats:  # every H2D DMA of the timed-kernels run, bracketed by events on the copy stream
        n, t, by = kstats["h2d"]
        tl = sum(tim.step_ms) / 1e3
        copy_stream = {"dmas": n, "mb_per_dma": by / 1e6, "us_per_dma": t * 1e6, "gbs_in_copy": by / t / 1e9,
                       "gbs_vs_peak": by / t / bw_peak, "busy_frac": (n * t / tl) if tl > 0 else None,
                       "note": "H2D copy engine: bytes / time inside each DMA (events on the copy stream, in the "
                               "separate timed-kernels run); busy_frac = summed DMA time / that run's step time"}

    if rank == 0:
        line = {
            "metric": "decode_tokens_per_s", "value": value, "unit": "tok/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": elapsed / args.steps * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "fp16", "data": "synthetic",
            "config": bench_config(args, ws, cfg),
            "run": {"splits_timed": splits[args.warmup:], "plan_profile": "live (profiler.measure on this GPU)",
                    "per_layer_ms": steady_layer_s * 1e3, "prefill_s": prefill_s, "numa": numa,
                    "h2d_bytes_per_step": h2d_alg / args.steps, "weights_bytes": weights_bytes,
                    "backend": (dist.get_backend().upper() if ws > 1 else None)},
            "roofline": k1_roof,
            "overlap_roofline": {
                "bound": "pcie", "achieved": achieved_gbs, "peak": bw_peak / 1e9, "unit": "GB/s",
                "frac": troof / elapsed, "traffic": None,
                "achieved_vs_gen5_x16_nominal": achieved_gbs / 64.0, "copy_stream": copy_stream,
                "note": "north-star per-layer overlap roofline max(H2D(X[:, :l'] + KV[l':s'-1]) / measured pinned "
                        "H2D peak, 4 b l' h^2 / sustained bf16 peak), l' = min(l, s'-1): exactly the bytes the "
                        "runtime ships; frac = T_roof / T_measured over the timed steps",
            },
            "kernels": kern,
            "profile": {"gpu_flops": prof.gpu_flops, "h2d_bandwidth": prof.h2d_bandwidth,
                        "d2h_bandwidth": prof.d2h_bandwidth, "transfer_latency": prof.transfer_latency},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "tok/s", "h2d_bytes_per_step": int(h2d_step),
                    "d2h_bytes_per_step": int(d2h_step), "steps": args.steps},
            "rank_windows": windows,
            "alt_overlap_plan": alt,
            "alt_row_schedule": alt_row,
            "alt_kv4": alt_kv4,
            "alt_config1": alt_c1,
            "alt_config5": alt_c5,
            "gpu_launches": launches,
            "clocks": clk,
            "peaks_source": peaks["source"],
        }
        print(json.dumps(line))
    if rt is not None:
        rt.close()
    if ws > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="kvpr", choices=["kvpr", "reference"])
    ap.add_argument("--model", default="opt-6.7b")
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--prompt", type=int, default=1024)
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-alt", action="store_true", help="skip the extension-objective measurement")
    ap.add_argument("--no-config1", action="store_true", help="skip the in-run BASELINE config-1 line")
    ap.add_argument("--no-config5", action="store_true", help="skip the in-run BASELINE config-5 sweep")
    ap.add_argument("--fixed-profile", action="store_true",
                    help="plan with the B200-guess profile instead of the live probe (profiler runs)")
    ap.add_argument("--tp", action="store_true",
                    help="config 4: head-sharded tensor parallelism over the torchrun ranks (NCCL)")
    args = ap.parse_args()
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if args.gpus != ws:
        sys.exit(f"bench.py --gpus {args.gpus} needs that many ranks: launch it under torchrun "
                 f"--nproc-per-node {args.gpus} (WORLD_SIZE is {ws})")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_kvpr(args)


if __name__ == "__main__":
    main()
