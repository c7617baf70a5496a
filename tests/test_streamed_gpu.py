"""Streamed-weights, multi-batch column schedule (§8f rank 1) on the B200: every batch decodes
bit-identically to the weights-resident runtime on the same prompt and plan, with fine and
coarse weight granularity."""

from __future__ import annotations

import pytest
import torch

from paper_2411_17089_b200.runtime import KVPRRuntime
from paper_2411_17089_b200.streamed import StreamedRuntime
from paper_2411_17089_b200.weights import OPTConfig, OPTWeights

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("granularity,K", [("fine", 3), ("coarse", 2), ("fine", 1)])
def test_streamed_equals_resident_bitwise(granularity, K):
    cfg = OPTConfig(hidden=512, layers=3, heads=8, ffn=2048, vocab=2048, max_pos=512)
    b, S0 = 4, 120
    splits = [60, 0, 122, 7, 124]
    w = OPTWeights.random(cfg, seed=21, device="cuda", std=0.1, emb_std=0.1)
    prompts = [torch.randint(0, cfg.vocab, (b, S0), generator=torch.Generator().manual_seed(100 + k))
               for k in range(K)]
    rt = StreamedRuntime(w, b, K, S0 + len(splits) + 1, granularity=granularity)
    first = rt.prefill(prompts)
    toks = rt.decode(splits, tokens=first, keep_logits=True)
    torch.cuda.synchronize()
    got_l = rt.last_logits.cpu()
    assert rt.h2d_bytes > 0
    rt.close()
    for k in range(K):
        # the streamed runtime runs the multi-kernel layer chain: compare with the same chain (at b4 the
        # resident runtime would otherwise take the fused layer tail, equal only to fp32 rounding)
        ref = KVPRRuntime(w, b, S0 + len(splits) + 1, fused_tail=False)
        f = ref.prefill(prompts[k])
        t = ref.decode(splits, tokens=f, keep_logits=True)
        torch.cuda.synchronize()
        assert torch.equal(first[k].cpu(), f.cpu()), k
        assert torch.equal(toks[:, k].cpu(), t.cpu()), k
        assert torch.equal(got_l[:, k], ref.last_logits.cpu()), k
        ref.close()


def test_fine_weight_loads_never_lose_measured(criterion):
    """Criterion 05b of the reference (test_acceptance.py:223-262: fine-grained weight loads never lose
    to coarse) on MEASURED runs of the streamed-weights runtime: OPT-6.7B layer shapes, 2 layers x 2 GPU
    batches of 32, prompt 1024, at the reference solver's column l and at the weight-gated l = s'
    (the rebuild needs only W_K|W_V, which fine granularity ships first).  Each makespan is the best of
    two runs (CUDA events); fine <= coarse x 1.01 (timing noise)."""
    from paper_2411_17089_b200.costmodel import WorkloadSpec
    from paper_2411_17089_b200.hwprofile import HardwareProfile
    from paper_2411_17089_b200.scheduler import plan_generation
    from paper_2411_17089_b200.weights import preset

    base = preset("opt-6.7b")
    cfg = OPTConfig(base.hidden, 2, base.heads, base.ffn, base.vocab, 2048)
    b, K, S0, steps = 32, 2, 1024, 3
    prof = HardwareProfile(gpu_flops=1391.2e12, h2d_bandwidth=55e9, d2h_bandwidth=55e9)
    wl = WorkloadSpec(batch_size=b, prompt_len=S0, gen_len=steps, num_batches=K)
    plans = {"solver": plan_generation(cfg.spec(), wl, prof, "column").splits,
             "weight_gated": [S0 + i + 1 for i in range(steps)]}
    w = OPTWeights.random(cfg, seed=0, device="cuda")
    prompts = [torch.randint(0, cfg.vocab, (b, S0), generator=torch.Generator().manual_seed(k)) for k in range(K)]
    out = {}
    for gran in ("fine", "coarse"):
        rt = StreamedRuntime(w, b, K, S0 + steps + 1, granularity=gran)
        first = rt.prefill(prompts)
        for name, splits in plans.items():
            best = float("inf")
            for _ in range(2):
                rt.len = S0
                torch.cuda.synchronize()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record(rt.cs)
                rt.decode(splits, tokens=first)
                e.record(rt.cs)
                torch.cuda.synchronize()
                best = min(best, s.elapsed_time(e) / 1e3)
            out[(gran, name)] = best
        rt.close()
    ok = all(out[("fine", n)] <= 1.01 * out[("coarse", n)] for n in plans)
    criterion("S05b", "measured streamed-weights makespan, fine vs coarse weight loads: " + ", ".join(
        f"{n} {out[('fine', n)] * 1e3:.2f} vs {out[('coarse', n)] * 1e3:.2f} ms" for n in plans) +
        " (fine <= coarse x 1.01)", ok)
    assert ok, out
