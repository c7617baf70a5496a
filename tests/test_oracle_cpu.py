"""Pin the CPU oracle before trusting it (no GPU).

* oracle/numerics_ref.py vs fixtures produced by the LIVE reference
  kvoverlap.numerics (tests/golden/numerics_golden.npz): split_merge_kv,
  decode_attention, append_token_kv — equal to the last bit (same fp64 ops).
* split-merge exactness over all splits (criterion 07 of
  pkg/tests/test_acceptance.py:288-328, 1e-12), restated.
* oracle/opt_ref.py: output independent of the split at fp64 (1e-12), and
  its OPT layer semantics equal transformers' OPTForCausalLM on the same
  weights (greedy logits, fp32, rel 1e-4) — the reference has no decoder, so
  this is the secondary pin for logits.
"""

from __future__ import annotations

import json

import numpy as np
import pytest
import torch

from oracle import numerics_ref as nr
from oracle import opt_ref

from .conftest import GOLDEN


def _golden():
    z = np.load(GOLDEN / "numerics_golden.npz")
    return z, json.loads(str(z["meta"]))


def test_numerics_oracle_matches_live_reference(criterion):
    z, meta = _golden()
    for m in meta:
        i, heads, split = m["i"], m["heads"], m["split"]
        g = lambda k: z[f"c{i}_{k}"]  # noqa: E731
        full = nr.build_kv(g("x"), g("w_k"), g("w_v"), heads)
        suffix = nr.KVState(full.keys[:, split:], full.values[:, split:])
        merged = nr.split_merge_kv(g("x"), split, g("w_k"), g("w_v"), suffix)
        assert np.array_equal(merged.keys, g("keys")) and np.array_equal(merged.values, g("values"))
        att = nr.decode_attention(g("q"), merged, g("w_o"))
        assert np.max(np.abs(att - g("att"))) <= 1e-12
        grown = nr.append_token_kv(full, g("x_new"), g("w_k"), g("w_v"))
        assert np.array_equal(grown.keys, g("grown_keys")) and np.array_equal(grown.values, g("grown_values"))
    criterion("O1", f"numerics oracle == live kvoverlap.numerics on {len(meta)} golden cases", True)


def test_split_merge_exact_all_splits(criterion):
    rng = np.random.default_rng(7)
    checks = 0
    worst = 0.0
    while checks < 1000:
        heads = int(rng.choice([1, 2, 4]))
        d = int(rng.integers(1, 5))
        h = heads * d
        seq = int(rng.integers(1, 33))
        x = rng.standard_normal((seq, h))
        w_k, w_v, w_o = (rng.standard_normal((h, h)) for _ in range(3))
        q = rng.standard_normal(h)
        full = nr.build_kv(x, w_k, w_v, heads)
        ref = nr.decode_attention(q, full, w_o)
        for split in range(seq + 1):
            merged = nr.split_merge_kv(x, split, w_k, w_v, nr.KVState(full.keys[:, split:], full.values[:, split:]))
            e = max(np.max(np.abs(merged.keys - full.keys)), np.max(np.abs(merged.values - full.values)),
                    np.max(np.abs(nr.decode_attention(q, merged, w_o) - ref)))
            worst = max(worst, float(e))
            checks += 1
    ok = worst <= 1e-12
    criterion("O2", f"split rebuild exact within 1e-12 over {checks} randomized checks (oracle)", ok)
    assert ok


def test_numerics_oracle_validation():
    x = np.zeros((3, 4))
    w = np.zeros((4, 4))
    full = nr.build_kv(x, w, w, 2)
    with pytest.raises(ValueError, match="suffix"):
        nr.split_merge_kv(x, 1, w, w, full)
    with pytest.raises(ValueError, match="split"):
        nr.split_merge_kv(x, 5, w, w, full)
    with pytest.raises(ValueError, match="empty"):
        nr.decode_attention(np.zeros(4), nr.KVState(full.keys[:, :0], full.values[:, :0]), w)
    assert nr.split_merge_kv(x, 0, w, w, full) is full


def _tiny(seed=0, h=64, heads=4, layers=2, ffn=256, vocab=97, max_pos=64):
    from paper_2411_17089_b200.weights import OPTConfig, OPTWeights

    cfg = OPTConfig(hidden=h, layers=layers, heads=heads, ffn=ffn, vocab=vocab, max_pos=max_pos)
    w = OPTWeights.random(cfg, seed=seed, device="cpu", std=0.1, emb_std=0.1)
    shape = opt_ref.OPTShape(h, layers, heads, ffn, vocab, max_pos, cfg.eps)
    return cfg, w, shape


def test_opt_oracle_split_invariant_fp64(criterion):
    cfg, w, shape = _tiny(1)
    prompt = np.random.default_rng(0).integers(0, cfg.vocab, (3, 20))
    plans = [[0] * 6, [21, 22, 23, 24, 25, 26], [5, 9, 13, 2, 24, 26], [1] * 6]
    outs = [opt_ref.generate(shape, w.numpy_dict(), prompt, p, storage=np.float64, compute=np.float64)
            for p in plans]
    worst = max(float(np.max(np.abs(a - b))) for o in outs[1:] for a, b in zip(o[1], outs[0][1]))
    same = all(np.array_equal(o[0], outs[0][0]) for o in outs)
    ok = worst <= 1e-12 and same
    criterion("O3", f"OPT oracle decode independent of split at fp64 (max dlogit {worst:.1e})", ok)
    assert ok


def test_opt_oracle_matches_hf_opt(criterion):
    transformers = pytest.importorskip("transformers")
    cfg, w, shape = _tiny(2)
    hf_cfg = transformers.OPTConfig(
        vocab_size=cfg.vocab, hidden_size=cfg.hidden, num_hidden_layers=cfg.layers, ffn_dim=cfg.ffn,
        num_attention_heads=cfg.heads, max_position_embeddings=cfg.max_pos, do_layer_norm_before=True,
        word_embed_proj_dim=cfg.hidden, enable_bias=True, layer_norm_elementwise_affine=True, dropout=0.0,
        attention_dropout=0.0, activation_function="relu", pad_token_id=None,
    )
    model = transformers.OPTForCausalLM(hf_cfg).eval().float()
    h = cfg.hidden
    sd = {"model.decoder.embed_tokens.weight": w.embed, "model.decoder.embed_positions.weight": w.pos,
          "model.decoder.final_layer_norm.weight": w.lnf_g, "model.decoder.final_layer_norm.bias": w.lnf_b,
          "lm_head.weight": w.embed}
    for j, lw in enumerate(w.layers):
        p = f"model.decoder.layers.{j}."
        for nm, sl in (("q", slice(0, h)), ("k", slice(h, 2 * h)), ("v", slice(2 * h, 3 * h))):
            sd[p + f"self_attn.{nm}_proj.weight"] = lw.wqkv[sl]
            sd[p + f"self_attn.{nm}_proj.bias"] = lw.bqkv[sl]
        sd.update({p + "self_attn.out_proj.weight": lw.wo, p + "self_attn.out_proj.bias": lw.bo,
                   p + "self_attn_layer_norm.weight": lw.ln1_g, p + "self_attn_layer_norm.bias": lw.ln1_b,
                   p + "final_layer_norm.weight": lw.ln2_g, p + "final_layer_norm.bias": lw.ln2_b,
                   p + "fc1.weight": lw.w1, p + "fc1.bias": lw.b1, p + "fc2.weight": lw.w2, p + "fc2.bias": lw.b2})
    missing, unexpected = model.load_state_dict({k: v.float() for k, v in sd.items()}, strict=False)
    assert not [m for m in missing if "lm_head" not in m], missing
    prompt = np.random.default_rng(1).integers(0, cfg.vocab, (2, 12))
    steps = 5
    toks, logits, _ = opt_ref.generate(shape, w.numpy_dict(), prompt, [4] * steps, storage=np.float32,
                                       compute=np.float32)
    ids = torch.tensor(prompt)
    hf_logits = []
    with torch.no_grad():
        for i in range(steps + 1):
            out = model(input_ids=ids).logits[:, -1].numpy()
            hf_logits.append(out)
            ids = torch.cat([ids, torch.tensor(toks[i])[:, None]], dim=1)
    rel = max(float(np.abs(a - b).max() / np.abs(b).max()) for a, b in zip(logits, hf_logits))
    ok = rel <= 1e-4 and all(np.array_equal(np.argmax(b, -1), toks[i]) for i, b in enumerate(hf_logits))
    criterion("O4", f"OPT oracle == transformers OPTForCausalLM (fp32, rel {rel:.1e})", ok)
    assert ok, rel


def test_fp16_helpers_bit_identical_to_numpy():
    """oracle/csrc/fp16conv.c's casts are NumPy's IEEE casts, bit for bit (ties to even, subnormals,
    overflow to inf, NaN)."""
    if not opt_ref._fp16lib():
        pytest.skip("oracle/libfp16conv.so not built (python -m oracle.build)")
    rng = np.random.default_rng(0)
    f = np.concatenate([rng.standard_normal(100003).astype(np.float32) * 10.0 ** rng.integers(-9, 6, 100003),
                        np.array([0.0, -0.0, 65504.0, 65520.0, 1e6, -1e6, np.inf, -np.inf, 5.96e-8, 2.98e-8,
                                  1.0 + 2.0 ** -11, 1.0 + 3 * 2.0 ** -11], dtype=np.float32)]).astype(np.float32)
    assert np.array_equal(opt_ref.narrow(f).view(np.uint16), f.astype(np.float16).view(np.uint16))
    assert np.array_equal(opt_ref.round16(f), f.astype(np.float16).astype(np.float32))
    h = np.arange(65536, dtype=np.uint16).view(np.float16)
    w = opt_ref.widen(h)
    ref = h.astype(np.float32)
    same = (w.view(np.uint32) == ref.view(np.uint32)) | (np.isnan(w) & np.isnan(ref))
    assert same.all()


@pytest.mark.parametrize("splits", [[0, 0, 0], [21, 5, 23]])
def test_oracle_c_attention_equals_numpy_path(splits, monkeypatch):
    """The fp16-storage oracle's C attention (double accumulation straight from the fp16 store rows)
    and its NumPy einsum path agree to fp32 rounding, including a rebuilt prefix."""
    if not opt_ref._fp16lib():
        pytest.skip("oracle/libfp16conv.so not built (python -m oracle.build)")
    cfg, w, shape = _tiny(3)
    prompt = np.random.default_rng(4).integers(0, cfg.vocab, (3, 20))
    fast = opt_ref.generate(shape, w.numpy_dict(), prompt, splits)
    monkeypatch.setattr(opt_ref, "_FP16", False)
    slow = opt_ref.generate(shape, w.numpy_dict(), prompt, splits)
    rel = max(float(np.abs(a - b).max() / np.abs(b).max()) for a, b in zip(fast[1], slow[1]))
    assert rel <= 2e-5, rel
    assert np.array_equal(fast[0], slow[0])
