"""The native C executor (csrc/executor.cu) against the Python issue loop: same tokens and logits
bit for bit (column and row schedules, ragged splits), and lower host cost per layer."""

from __future__ import annotations

import time

import pytest
import torch

from paper_2411_17089_b200.runtime import KVPRRuntime
from paper_2411_17089_b200.weights import OPTConfig, OPTWeights

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("x_resident,wave,k1s", [(False, 0, False), (True, 0, False), (False, 24, False),
                                                  (False, 24, True), (True, 0, True)])
def test_native_equals_python_loop_bitwise(x_resident, wave, k1s):
    """k1s: the executor issues K1 a unit ahead on its own stream (only the schedule changes)."""
    cfg = OPTConfig(hidden=512, layers=4, heads=8, ffn=2048, vocab=2048, max_pos=512)
    b, S0 = 3, 150
    splits = [75, 0, 152, 1, 154, 100, 3]
    w = OPTWeights.random(cfg, seed=31, device="cuda", std=0.1, emb_std=0.1)
    prompt = torch.randint(0, cfg.vocab, (b, S0), generator=torch.Generator().manual_seed(32))
    outs = []
    for native in (False, True):
        rt = KVPRRuntime(w, b, S0 + len(splits) + 1, x_resident=x_resident, chunk_rows=64, chunk_wave=wave,
                         k1_stream=k1s)
        first = rt.prefill(prompt)
        toks = rt.decode(splits, tokens=first, keep_logits=True, native=native)
        torch.cuda.synchronize()
        n = S0 + len(splits)  # positions written (the last capacity slot is never touched)
        outs.append((toks.cpu(), rt.last_logits.cpu(), rt.stores.kv[:, :n].clone(), rt.stores.x[:, :n].clone()))
        rt.close()
    for a, c in zip(*outs):
        assert torch.equal(a, c)


@pytest.mark.parametrize("layers", [1, 3])
def test_issue_schedule_variants_bitwise(layers):
    """Only the schedule may change with the issue knobs: 2 or 3 device buffers, 1 or 4 X chunks
    (chunk_rows), K1 on its own stream or not, native or Python issue, X streamed or resident -- all
    give the same tokens, logits and host stores bit for bit.  layers = 1 covers the single-layer
    ordering (unit u+1's loads wait on unit u's own D2H of the new position)."""
    cfg = OPTConfig(hidden=256, layers=layers, heads=4, ffn=1024, vocab=1024, max_pos=256)
    b, S0 = 2, 90
    splits = [45, 91, 0, 93, 10, 95, 60, 1]
    w = OPTWeights.random(cfg, seed=41, device="cuda", std=0.1, emb_std=0.1)
    prompt = torch.randint(0, cfg.vocab, (b, S0), generator=torch.Generator().manual_seed(42))
    variants = [dict(nbuf=2, chunk_rows=1000, k1_stream=False, native=True),
                dict(nbuf=3, chunk_rows=1000, k1_stream=False, native=True),
                dict(nbuf=2, chunk_rows=12, k1_stream=False, native=True),
                dict(nbuf=3, chunk_rows=12, k1_stream=True, native=True),
                dict(nbuf=2, chunk_rows=12, k1_stream=True, native=False),
                dict(nbuf=3, chunk_rows=12, k1_stream=False, native=False),
                dict(nbuf=2, chunk_rows=12, k1_stream=True, native=True, x_resident=True)]
    outs = []
    for v in variants:
        v = dict(v)
        native = v.pop("native")
        rt = KVPRRuntime(w, b, S0 + len(splits) + 1, chunk_wave=0, **v)
        first = rt.prefill(prompt)
        toks = rt.decode(splits, tokens=first, keep_logits=True, native=native)
        torch.cuda.synchronize()
        n = S0 + len(splits)
        outs.append((toks.cpu(), rt.last_logits.cpu(), rt.stores.kv[:, :n].clone()))
        rt.close()
    for k, o in enumerate(outs[1:], start=1):
        for a, c in zip(outs[0], o):
            assert torch.equal(a, c), variants[k]


@pytest.mark.parametrize("x_resident", [False, True])
def test_grouped_dmas_bitwise(x_resident):
    """H2D copies of G consecutive layers as one strided DMA (kvpr_decoder_desc.dma_group): only the copy
    schedule changes -- tokens, logits and host stores equal the one-DMA-per-layer run bit for bit, for
    G = 2, 3, 4 (12 layers, fused small-batch tail), splits from 0 to s', X streamed or resident."""
    cfg = OPTConfig(hidden=256, layers=12, heads=4, ffn=1024, vocab=1024, max_pos=256)
    b, S0 = 4, 70
    splits = [35, 71, 0, 73, 10, 75, 74, 1, 40]
    w = OPTWeights.random(cfg, seed=43, device="cuda", std=0.1, emb_std=0.1)
    prompt = torch.randint(0, cfg.vocab, (b, S0), generator=torch.Generator().manual_seed(44))
    outs = []
    for g in (1, 2, 3, 4):
        rt = KVPRRuntime(w, b, S0 + len(splits) + 1, x_resident=x_resident, dma_group=g)
        assert rt.dma_group == g and rt.nbuf >= 2 * g
        first = rt.prefill(prompt)
        toks = rt.decode(splits, tokens=first, keep_logits=True)
        torch.cuda.synchronize()
        n = S0 + len(splits)
        outs.append((toks.cpu(), rt.last_logits.cpu(), rt.stores.kv[:, :n].clone(), rt.stores.x[:, :n].clone()))
        rt.close()
    for k, o in enumerate(outs[1:], start=2):
        for a, c in zip(outs[0], o):
            assert torch.equal(a, c), k


def test_decode_split_over_calls_bitwise():
    """Nine steps as one decode() call, as 5 + 4 calls, and as nine single-step calls (the e2e path)
    give the same tokens, logits and host stores: the executor's event rings, grouped KV copies and
    staging buffers carry no state across calls that changes the result (12 layers, fused tail,
    KV tails in groups of 2)."""
    cfg = OPTConfig(hidden=256, layers=12, heads=4, ffn=1024, vocab=1024, max_pos=256)
    b, S0 = 4, 70
    splits = [35, 71, 0, 73, 10, 75, 74, 1, 40]
    w = OPTWeights.random(cfg, seed=45, device="cuda", std=0.1, emb_std=0.1)
    prompt = torch.randint(0, cfg.vocab, (b, S0), generator=torch.Generator().manual_seed(46))
    outs = []
    for parts in ([9], [5, 4], [1] * 9):
        rt = KVPRRuntime(w, b, S0 + len(splits) + 1)
        assert rt.fused_tail and rt.dma_group == 2
        tok = rt.prefill(prompt)
        toks, logits, i = [], [], 0
        for n in parts:
            t = rt.decode(splits[i:i + n], tokens=tok, keep_logits=True)
            toks.append(t)
            logits.append(rt.last_logits[-1].clone())  # [steps, batch, vocab] of this call: its last step
            tok = t[-1]
            i += n
        torch.cuda.synchronize()
        n = S0 + len(splits)
        outs.append((torch.cat(toks).cpu(), logits[-1].cpu(), rt.stores.kv[:, :n].clone(), rt.stores.x[:, :n].clone()))
        rt.close()
    for k, o in enumerate(outs[1:], start=1):
        for a, c in zip(outs[0], o):
            assert torch.equal(a, c), k


def test_native_loop_cuts_host_time():
    """Config-1 geometry is host bound under the Python loop; the executor issues a step far faster."""
    cfg = OPTConfig(hidden=768, layers=12, heads=12, ffn=3072)
    b, S0, steps = 4, 256, 8
    w = OPTWeights.random(cfg, seed=0, device="cuda")
    prompt = torch.randint(0, cfg.vocab, (b, S0), generator=torch.Generator().manual_seed(1))
    rt = KVPRRuntime(w, b, S0 + 2 * steps + 2)
    first = rt.prefill(prompt)
    rt.decode([200] * 2, tokens=first, native=True)
    t = {}
    for native in (False, True):
        rt.reset(S0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rt.decode([200] * steps, tokens=first, native=native)
        torch.cuda.synchronize()
        t[native] = time.perf_counter() - t0
    rt.close()
    assert t[True] < t[False], t


def test_native_timeline_matches_python_convention():
    """decode(timing=...) runs through the executor and fills DecodeTiming with the Python loop's
    shape (steps x layers), positive times whose per-step sums track the step times."""
    from paper_2411_17089_b200.runtime import DecodeTiming

    cfg = OPTConfig(hidden=512, layers=3, heads=8, ffn=2048, vocab=2048, max_pos=512)
    b, S0, splits = 2, 100, [50, 0, 102, 7]
    w = OPTWeights.random(cfg, seed=5, device="cuda", std=0.1, emb_std=0.1)
    prompt = torch.randint(0, cfg.vocab, (b, S0), generator=torch.Generator().manual_seed(6))
    rt = KVPRRuntime(w, b, S0 + len(splits) + 1)
    first = rt.prefill(prompt)
    tims, toks = [], []
    for native in (False, True):
        rt.reset(S0)
        tim = DecodeTiming()
        toks.append(rt.decode(splits, tokens=first, timing=tim, native=native).cpu())
        tims.append(tim)
    rt.close()
    assert torch.equal(toks[0], toks[1])
    nat = tims[1]
    assert len(nat.step_ms) == len(splits) and [len(r) for r in nat.layer_ms] == [cfg.layers] * len(splits)
    assert all(x > 0 for r in nat.layer_ms for x in r)
    for row, st in zip(nat.layer_ms, nat.step_ms):
        assert sum(row) <= st + 1e-3  # the head closes each step after its last layer
