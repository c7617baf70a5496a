"""Host-side runtime logic without a GPU: X chunking, plan plumbing, and the
batch-partitioned multi-process path over gloo (world_size 2)."""

from __future__ import annotations

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2411_17089_b200 import multigpu
from paper_2411_17089_b200.costmodel import WorkloadSpec, opt_preset
from paper_2411_17089_b200.hwprofile import HardwareProfile
from paper_2411_17089_b200.runtime import chunk_bounds, wave_positions
from paper_2411_17089_b200.scheduler import solve_split


@pytest.mark.parametrize("n,chunks", [(0, 4), (1, 4), (63, 4), (64, 4), (882, 4), (1000, 3), (257, 8)])
def test_chunk_bounds_partition(n, chunks):
    b = chunk_bounds(n, chunks)
    if n == 0:
        assert b == []
        return
    assert b[0][0] == 0 and b[-1][1] == n
    assert all(p1 > p0 for p0, p1 in b)
    assert all(b[i][1] == b[i + 1][0] for i in range(len(b) - 1))
    assert len(b) <= chunks
    sizes = [p1 - p0 for p0, p1 in b]
    assert max(sizes) - min(sizes) <= 1


def test_partition_slices():
    s = multigpu.partition(32, 8)
    assert [x.count for x in s] == [4] * 8 and s[-1].start == 28
    s = multigpu.partition(10, 4)
    assert [x.count for x in s] == [3, 3, 2, 2] and [x.start for x in s] == [0, 3, 6, 8]
    with pytest.raises(ValueError):
        multigpu.partition(3, 4)


def test_rank_plan_is_reference_solver_on_the_slice():
    spec = opt_preset("opt-13b")
    wl = WorkloadSpec(batch_size=32, prompt_len=1024, gen_len=4)
    prof = HardwareProfile(gpu_flops=1391.2e12, h2d_bandwidth=55e9, d2h_bandwidth=55e9, transfer_latency=1e-5)
    for world in (1, 2, 4, 8):
        for r in range(world):
            plan = multigpu.rank_plan(spec, wl, prof, world, r)
            b = multigpu.partition(32, world)[r].count
            wl_r = WorkloadSpec(batch_size=b, prompt_len=1024, gen_len=4)
            assert plan.decisions[0] == solve_split(spec, wl_r, prof, 1025, "column", step=1)
    # OPT-13B b4 (G=8 shard) with 10 us latency -> l = 858
    assert multigpu.rank_plan(spec, wl, prof, 8, 0).decisions[0].recompute_len == 858


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _tiny_decoder():
    import numpy as np

    from oracle import opt_ref
    from paper_2411_17089_b200.weights import OPTConfig, OPTWeights

    cfg = OPTConfig(hidden=64, layers=2, heads=4, ffn=256, vocab=97, max_pos=64)
    w = OPTWeights.random(cfg, seed=5, device="cpu", std=0.1, emb_std=0.1).numpy_dict()
    shape = opt_ref.OPTShape(cfg.hidden, cfg.layers, cfg.heads, cfg.ffn, cfg.vocab, cfg.max_pos, cfg.eps)
    return cfg, w, shape, np.random.default_rng(6)


def _worker(rank, world, port, global_batch, q):
    """One rank of the batch partition: partition -> its own plan (reference solver on its slice) -> its
    own decoder replica over its sequences -> gather_tokens.  The replica is the CPU OPT decoder with host
    stores and the split-merge rebuild (oracle/opt_ref.py, fp64): the GPU runtime needs a device
    (tests/test_multigpu_gpu.py runs the same flow with KVPRRuntime on the B200)."""
    import numpy as np

    from oracle import opt_ref

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg, w, shape, rng = _tiny_decoder()
        prompt = rng.integers(0, cfg.vocab, (global_batch, 12))
        sl = multigpu.partition(global_batch, world)[rank]
        wl = WorkloadSpec(batch_size=global_batch, prompt_len=12, gen_len=5)
        plan = multigpu.rank_plan(cfg.spec(), wl, PROF, world, rank)
        toks, logits, _ = opt_ref.generate(shape, w, prompt[sl.start:sl.start + sl.count], plan.splits,
                                           storage=np.float64, compute=np.float64)
        full = multigpu.gather_tokens(torch.from_numpy(toks), global_batch)
        t = multigpu.max_over_ranks(float(rank + 1))
        q.put((rank, full.tolist(), np.stack(logits).tolist(), t))
    finally:
        dist.destroy_process_group()


PROF = HardwareProfile(gpu_flops=1391.2e12, h2d_bandwidth=55e9, d2h_bandwidth=55e9, transfer_latency=1e-5)


@pytest.mark.parametrize("global_batch", [8, 7])
def test_partitioned_decode_over_gloo(global_batch):
    """world 2 over gloo: the gathered tokens of the per-rank decoders equal the unpartitioned decode, and
    each rank's logits its rows of it (sequences are independent units)."""
    import numpy as np

    from oracle import opt_ref

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, global_batch, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg, w, shape, rng = _tiny_decoder()
    prompt = rng.integers(0, cfg.vocab, (global_batch, 12))
    wl = WorkloadSpec(batch_size=global_batch, prompt_len=12, gen_len=5)
    splits = multigpu.rank_plan(cfg.spec(), wl, PROF, 1, 0).splits
    toks, logits, _ = opt_ref.generate(shape, w, prompt, splits, storage=np.float64, compute=np.float64)
    logits = np.stack(logits)
    for rank, full, lg, t in res:
        assert full == toks.tolist()
        assert t == float(world)
        sl = multigpu.partition(global_batch, world)[rank]
        assert np.abs(np.array(lg) - logits[:, sl.start:sl.start + sl.count]).max() <= 1e-9


@pytest.mark.parametrize("h,f", [(4096, 16384), (768, 3072), (64, 256)])
def test_streamed_weight_regions_tile_the_layer(h, f):
    """Fine-grained loads: the W_KV part and the rest cover every byte of a layer exactly once,
    and the W_KV part is exactly what K1 reads (rows [h, 3h) of wqkv and b_k|b_v)."""
    from paper_2411_17089_b200.streamed import weight_regions

    total = weight_regions(h, f, "all")[0][1]
    assert total == (3 * h * h + 3 * h + h * h + h + 4 * h + f * h + f + h * f + h) * 2
    covered = sorted(weight_regions(h, f, "kv") + weight_regions(h, f, "rest"))
    pos = 0
    for off, n in covered:
        assert off == pos and n > 0
        pos += n
    assert pos == total
    kv = weight_regions(h, f, "kv")
    assert kv[0] == (h * h * 2, 2 * h * h * 2) and kv[1] == (3 * h * h * 2 + 2 * h, 4 * h)
    assert all(off % 16 == 0 for off, _ in covered)  # DMA / TMA friendly alignment
    with pytest.raises(ValueError):
        weight_regions(h, f, "ffn")


def test_parse_cpulist():
    assert multigpu.parse_cpulist("0-3,8,10-11\n") == [0, 1, 2, 3, 8, 10, 11]
    assert multigpu.parse_cpulist("5") == [5]
    assert multigpu.parse_cpulist("") == []
    with pytest.raises(ValueError):
        multigpu.parse_cpulist("4-2")


def test_wave_positions_and_wave_chunks():
    # OPT-6.7B b32 on 148 SMs: 296 positions = 37 pair m-blocks x 32 n-blocks = 16 waves of 74 pairs
    assert wave_positions(32, 4096, 148) == 296
    assert wave_positions(32, 5120, 148) == 296  # 13B: 40 n-blocks, still 37 m-blocks
    assert wave_positions(4, 768, 148) == 0      # config 1: no whole-wave chunk under 1024 positions
    for n, chunks in ((888, 4), (1000, 4), (1500, 4), (296, 4), (300, 2), (5000, 4)):
        b = chunk_bounds(n, chunks, 64, wave=296)
        assert b[0][0] == 0 and b[-1][1] == n and len(b) <= chunks
        assert all(b[i][1] == b[i + 1][0] for i in range(len(b) - 1))
        assert all((p1 - p0) % 296 == 0 for p0, p1 in b[:-1])
    assert chunk_bounds(888, 4, 64, wave=296) == [(0, 296), (296, 592), (592, 888)]
    assert chunk_bounds(895, 4, 64, wave=296) == [(0, 296), (296, 592), (592, 895)]  # short tail merged
    assert chunk_bounds(1100, 4, 64, wave=296) == [(0, 296), (296, 592), (592, 888), (888, 1100)]
    assert chunk_bounds(200, 4, 64, wave=296) == chunk_bounds(200, 4, 64)  # shorter than a wave: even split
