"""Host logic of the head-sharded TP mode (config 4) without GPUs.

* TPLayout: block-cyclic X ownership partitions the positions, compact store
  indices are a bijection per rank, rounds assemble natural order.
* shard_layer: shards reconstruct the weights; row-parallel partials sum to
  the unsharded projection (bias carried once, by rank 0).
* world_size 2 over gloo: each rank runs the TP data flow of TPRuntime
  (compact X blocks -> per-round all-gather -> local-head K1 rebuild ->
  local attention -> rank-0-accumulate + all-reduce) in fp64 on the CPU and
  its logits equal the unsharded oracle (oracle/opt_ref.py) to 1e-6 (the oracle returns fp32 logits).
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2411_17089_b200.tp import TPLayout, shard_layer
from paper_2411_17089_b200.weights import OPTConfig, OPTWeights


@pytest.mark.parametrize("world,block,n", [(2, 4, 37), (8, 64, 1596), (4, 16, 64), (3, 5, 1)])
def test_layout_partitions_positions(world, block, n):
    owners = {}
    for r in range(world):
        lay = TPLayout(world, r, 48 * world, 4 * world, 16 * world, block)
        runs = lay.owned_runs(n)
        idx = []
        for p0, p1 in runs:
            for p in range(p0, p1):
                assert p not in owners
                owners[p] = r
                assert lay.owner(p) == r
                idx.append(lay.compact_index(p))
        assert idx == sorted(set(idx))  # compact indices are increasing and unique
        assert max(idx, default=-1) < lay.compact_capacity(n)
    assert sorted(owners) == list(range(n))
    lay = TPLayout(world, 0, 48 * world, 4 * world, 16 * world, block)
    rs = lay.rounds(n)
    assert rs[0][1] == 0 and rs[-1][2] == n
    assert all(rs[k][2] == rs[k + 1][1] for k in range(len(rs) - 1))
    with pytest.raises(ValueError):
        TPLayout(world, world, 48, 4 * world, 16 * world)


def test_shard_layer_reconstructs_and_sums():
    cfg = OPTConfig(hidden=64, layers=1, heads=4, ffn=128, vocab=50, max_pos=16)
    w = OPTWeights.random(cfg, seed=3, device="cpu")
    lw = w.layers[0]
    world = 2
    shards = [shard_layer(lw, TPLayout(world, r, 64, 4, 128)) for r in range(world)]
    h, hs = 64, 32
    for part in range(3):
        full = lw.wqkv[part * h:(part + 1) * h]
        rebuilt = torch.cat([s.wqkv[part * hs:(part + 1) * hs] for s in shards])
        assert torch.equal(full, rebuilt)
    x = torch.randn(5, h, dtype=torch.float64)
    a = torch.randn(5, h, dtype=torch.float64)
    want = a @ lw.wo.double().T + lw.bo.double()
    got = sum(a[:, r * hs:(r + 1) * hs] @ shards[r].wo.double().T + shards[r].bo.double() for r in range(world))
    assert torch.allclose(got, want, atol=1e-12)
    y = x @ lw.w1.double().T
    got1 = torch.cat([x @ s.w1.double().T for s in shards], dim=1)
    assert torch.allclose(got1, y, atol=1e-12)


# ---------------------------------------------------------------------------
# gloo: the TP data flow on CPU, fp64


def _ln(x, g, b, eps=1e-5):
    mu = x.mean(-1, keepdim=True)
    var = ((x - mu) ** 2).mean(-1, keepdim=True)
    return (x - mu) / torch.sqrt(var + eps) * g + b


def _tp_rank(rank, world, port, q, prompt, splits, block):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = OPTConfig(hidden=64, layers=2, heads=4, ffn=128, vocab=60, max_pos=64)
        w = OPTWeights.random(cfg, seed=7, device="cpu", std=0.1, emb_std=0.1)
        lay = TPLayout(world, rank, cfg.hidden, cfg.heads, cfg.ffn, block)
        L = [shard_layer(lw, lay) for lw in w.layers]
        D = lambda t: t.double()  # noqa: E731
        b, S0 = prompt.shape
        h, hs, H, d = cfg.hidden, lay.hs, lay.heads_local, lay.head_dim
        cap = S0 + len(splits) + 1
        Xst = [torch.zeros(lay.compact_capacity(cap), b, h, dtype=torch.float64) for _ in L]
        KVst = [torch.zeros(cap, 2, b, hs, dtype=torch.float64) for _ in L]

        def rowpar(a, wt, bias, hres):
            part = a @ D(wt).T + (D(bias) if rank == 0 else 0)
            t = (hres + part if rank == 0 else part).contiguous()  # gloo reduces the raw storage
            dist.all_reduce(t)
            return t

        def attend(qv, K, V):  # qv [b, hs]; K,V [s, b, hs]
            s = K.shape[0]
            lg = torch.einsum("sbhd,bhd->bhs", K.reshape(s, b, H, d), qv.reshape(b, H, d)) / d ** 0.5
            return torch.einsum("bhs,sbhd->bhd", torch.softmax(lg, -1), V.reshape(s, b, H, d)).reshape(b, hs)

        # prefill (pos-major rows)
        toks = torch.tensor(prompt.T)
        hcur = D(w.embed)[toks] + D(w.pos)[torch.arange(S0) + 2][:, None, :]
        for j, lw in enumerate(L):
            x = _ln(hcur, D(lw.ln1_g), D(lw.ln1_b))
            for p0, p1 in lay.owned_runs(S0):
                i0 = lay.compact_index(p0)
                Xst[j][i0:i0 + (p1 - p0)] = x[p0:p1]
            y = x @ D(lw.wqkv).T + D(lw.bqkv)
            qv, k, v = y[..., :hs], y[..., hs:2 * hs], y[..., 2 * hs:]
            KVst[j][:S0, 0], KVst[j][:S0, 1] = k, v
            lg = torch.einsum("tbhd,sbhd->bhts", qv.reshape(S0, b, H, d), k.reshape(S0, b, H, d)) / d ** 0.5
            lg = lg.masked_fill(torch.triu(torch.ones(S0, S0, dtype=torch.bool), 1), float("-inf"))
            a = torch.einsum("bhts,sbhd->tbhd", torch.softmax(lg, -1), v.reshape(S0, b, H, d)).reshape(S0, b, hs)
            hcur = rowpar(a, lw.wo, lw.bo, hcur)
            f = torch.relu(_ln(hcur, D(lw.ln2_g), D(lw.ln2_b)) @ D(lw.w1).T + D(lw.b1))
            hcur = rowpar(f, lw.w2, lw.b2, hcur)
        z = _ln(hcur[-1], D(w.lnf_g), D(w.lnf_b))
        logits = [z @ D(w.embed).T]
        tok = logits[-1].argmax(-1)
        length = S0
        for l in splits:
            s = length + 1
            lp = min(l, s - 1)
            hcur = D(w.embed)[tok] + D(w.pos)[s - 1 + 2]
            for j, lw in enumerate(L):
                # X[0:lp] assembled round by round from every rank's compact blocks
                R = lay.round_len
                Xg = torch.zeros(((lp + R - 1) // R) * R, b, h, dtype=torch.float64)
                for t, r0, r1 in lay.rounds(lp):
                    q0, q1 = lay.my_block(t, lp)
                    mine = torch.zeros(block, b, h, dtype=torch.float64)
                    if q1 > q0:
                        i0 = lay.compact_index(q0)
                        mine[: q1 - q0] = Xst[j][i0:i0 + (q1 - q0)]
                    parts = [torch.zeros_like(mine) for _ in range(world)]
                    dist.all_gather(parts, mine)
                    Xg[t * R:(t + 1) * R] = torch.cat(parts)
                xn = _ln(hcur, D(lw.ln1_g), D(lw.ln1_b))
                y = xn @ D(lw.wqkv).T + D(lw.bqkv)
                qv, kn, vn = y[..., :hs], y[..., hs:2 * hs], y[..., 2 * hs:]
                K = torch.empty(s, b, hs, dtype=torch.float64)
                V = torch.empty(s, b, hs, dtype=torch.float64)
                if lp:
                    kv = Xg[:lp] @ D(lw.wqkv[hs:]).T + D(lw.bqkv[hs:])
                    K[:lp], V[:lp] = kv[..., :hs], kv[..., hs:]
                K[lp:s - 1], V[lp:s - 1] = KVst[j][lp:s - 1, 0], KVst[j][lp:s - 1, 1]
                K[s - 1], V[s - 1] = kn, vn
                if lay.owner(s - 1) == rank:
                    Xst[j][lay.compact_index(s - 1)] = xn
                KVst[j][s - 1, 0], KVst[j][s - 1, 1] = kn, vn
                hcur = rowpar(attend(qv, K, V), lw.wo, lw.bo, hcur)
                f = torch.relu(_ln(hcur, D(lw.ln2_g), D(lw.ln2_b)) @ D(lw.w1).T + D(lw.b1))
                hcur = rowpar(f, lw.w2, lw.b2, hcur)
            z = _ln(hcur, D(w.lnf_g), D(w.lnf_b))
            logits.append(z @ D(w.embed).T)
            tok = logits[-1].argmax(-1)
            length = s
        q.put((rank, [x.numpy() for x in logits]))
    finally:
        dist.destroy_process_group()


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_tp2_gloo_matches_unsharded_oracle(criterion):
    from oracle import opt_ref

    world, block = 2, 4
    rng = np.random.default_rng(5)
    prompt = rng.integers(0, 60, (3, 21))
    splits = [0, 11, 22, 5, 24]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_tp_rank, args=(r, world, port, q, prompt, splits, block)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = OPTConfig(hidden=64, layers=2, heads=4, ffn=128, vocab=60, max_pos=64)
    w = OPTWeights.random(cfg, seed=7, device="cpu", std=0.1, emb_std=0.1)
    shape = opt_ref.OPTShape(64, 2, 4, 128, 60, 64)
    _, ref, _ = opt_ref.generate(shape, w.numpy_dict(), prompt, splits, storage=np.float64, compute=np.float64)
    err = max(float(np.abs(res[r][i] - ref[i]).max()) for r in range(world) for i in range(len(ref)))
    ok = err <= 1e-6  # oracle logits are returned as fp32
    criterion("P2", f"TP=2 head-sharded data flow (gloo, fp64) == unsharded oracle (max |dlogit| {err:.1e})", ok)
    assert ok, err
