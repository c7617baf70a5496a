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
        ref = KVPRRuntime(w, b, S0 + len(splits) + 1)
        f = ref.prefill(prompts[k])
        t = ref.decode(splits, tokens=f, keep_logits=True)
        torch.cuda.synchronize()
        assert torch.equal(first[k].cpu(), f.cpu()), k
        assert torch.equal(toks[:, k].cpu(), t.cpu()), k
        assert torch.equal(got_l[:, k], ref.last_logits.cpu()), k
        ref.close()
