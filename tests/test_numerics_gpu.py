"""The reference's numeric contract (pkg/tests/test_numerics.py) run against the
GPU drop-in paper_2411_17089_b200.numerics, checked against the fp64 oracle
restatement (oracle/numerics_ref.py, itself pinned to the live reference).

Tolerance: fp16 storage / fp32 accumulation vs fp64 —
|gpu - oracle| <= 2e-2 * max|oracle| (the north-star relative bound).
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import numerics_ref as nr
from paper_2411_17089_b200 import numerics as gn

pytestmark = pytest.mark.gpu
RTOL = 2e-2


def _case(seed, heads=4, d=64, seq=70):
    rng = np.random.default_rng(seed)
    h = heads * d
    s = 1.0 / np.sqrt(h)
    return (rng.standard_normal((seq, h)), rng.standard_normal((h, h)) * s, rng.standard_normal((h, h)) * s,
            rng.standard_normal((h, h)) * s, rng.standard_normal(h))


def _rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))


@pytest.mark.parametrize("heads,d,seq", [(4, 64, 70), (2, 128, 33), (1, 64, 1)])
def test_split_merge_matches_full_cache(heads, d, seq):
    x, w_k, w_v, w_o, q = _case(3, heads, d, seq)
    full = nr.build_kv(x, w_k, w_v, heads)
    ref = nr.decode_attention(q, full, w_o)
    for split in sorted({0, 1, seq // 3, seq // 2, seq - 1, seq}):
        if split > seq:
            continue
        suffix = gn.KVState(full.keys[:, split:], full.values[:, split:])
        merged = gn.split_merge_kv(x, split, w_k, w_v, suffix)
        assert merged.keys.shape == full.keys.shape
        assert _rel(merged.keys, full.keys) <= RTOL and _rel(merged.values, full.values) <= RTOL
        out = gn.decode_attention(q, merged, w_o)
        assert _rel(out, ref) <= RTOL, (split, _rel(out, ref))


def test_split_zero_passes_suffix_through():
    x, w_k, w_v, _, _ = _case(4)
    full = gn.KVState(*[a for a in (nr.build_kv(x, w_k, w_v, 4).keys, nr.build_kv(x, w_k, w_v, 4).values)])
    assert gn.split_merge_kv(x, 0, w_k, w_v, full) is full


def test_validation_matches_reference():
    x, w_k, w_v, w_o, q = _case(6)
    full = gn.KVState(nr.build_kv(x, w_k, w_v, 4).keys, nr.build_kv(x, w_k, w_v, 4).values)
    with pytest.raises(ValueError, match="suffix"):
        gn.split_merge_kv(x, 2, w_k, w_v, full)
    with pytest.raises(ValueError, match="split"):
        gn.split_merge_kv(x, 71, w_k, w_v, full)
    empty = gn.KVState(full.keys[:, :0], full.values[:, :0])
    with pytest.raises(ValueError, match="empty"):
        gn.decode_attention(q, empty, w_o)
    with pytest.raises(ValueError, match="length"):
        gn.decode_attention(q[:-1], full, w_o)
    bad = w_k.copy()
    bad[0, 0] = np.inf
    with pytest.raises(ValueError, match="finite"):
        gn.split_merge_kv(x, 3, bad, w_v, gn.KVState(full.keys[:, 3:], full.values[:, 3:]))


@pytest.mark.parametrize("heads,d,seq", [(4, 64, 70), (2, 128, 33)])
def test_build_append_project_match_oracle(heads, d, seq):
    """build_kv / append_token_kv / project_qkv / stable_softmax on the GPU vs the fp64 oracle; the
    appended token equals what split_merge_kv rebuilds for that position, bit for bit (both K1)."""
    x, w_k, w_v, w_o, q = _case(9, heads, d, seq)
    full = gn.build_kv(x, w_k, w_v, heads)
    ref = nr.build_kv(x, w_k, w_v, heads)
    assert _rel(full.keys, ref.keys) <= RTOL and _rel(full.values, ref.values) <= RTOL
    grown = gn.append_token_kv(gn.build_kv(x[:-1], w_k, w_v, heads), x[-1], w_k, w_v)
    assert np.array_equal(grown.keys, full.keys) and np.array_equal(grown.values, full.values)
    rebuilt = gn.split_merge_kv(x, seq, w_k, w_v, gn.KVState(full.keys[:, :0], full.values[:, :0]))
    assert np.array_equal(rebuilt.keys, full.keys)
    w_q = w_o  # any h x h matrix
    qh, kh, vh = gn.project_qkv(x, w_q, w_k, w_v, heads)
    assert _rel(qh, nr.per_head(x @ w_q, heads)) <= RTOL
    assert _rel(kh, ref.keys) <= RTOL and _rel(vh, ref.values) <= RTOL
    z = np.random.default_rng(1).standard_normal(37) * 5
    assert np.max(np.abs(gn.stable_softmax(z) - nr.stable_softmax(z))) <= 1e-12
    with pytest.raises(ValueError, match="width"):
        gn.append_token_kv(full, x[-1, :-1], w_k[:-1, :-1], w_v[:-1, :-1])


def test_reference_validate_generator_through_gpu_dropin(criterion):
    """The reference's own randomized harness (cli.py:343-377: heads in {1,2,4}, head_dim in [1,4],
    s' in [1,32], up to 4 sequences, every split l in [0, s']) pointed at the GPU drop-in: head dims
    below 64 are zero-padded inside numerics.decode_attention.  The reference demands 1e-12 of its
    fp64 path; here every split agrees with the fp64 oracle within the north-star 2e-2 (fp16 storage),
    and the GPU output is the same for every split (K1 rebuild == the transferred cache)."""
    rng = np.random.default_rng(0)
    worst, cases, bad_split = 0.0, 0, []
    for case in range(6):
        heads = int(rng.choice([1, 2, 4]))
        d = int(rng.integers(1, 5))
        h = heads * d
        seq = int(rng.integers(1, 33))
        for _ in range(int(rng.integers(1, 5))):
            x, w_k, w_v, w_o = (rng.standard_normal(s) for s in ((seq, h), (h, h), (h, h), (h, h)))
            q = rng.standard_normal(h)
            full = nr.build_kv(x, w_k, w_v, heads)
            ref = nr.decode_attention(q, full, w_o)
            gfull = gn.build_kv(x, w_k, w_v, heads)
            outs = []
            for split in range(seq + 1):
                merged = gn.split_merge_kv(x, split, w_k, w_v, gn.KVState(gfull.keys[:, split:],
                                                                          gfull.values[:, split:]))
                outs.append(gn.decode_attention(q, merged, w_o))
                worst = max(worst, _rel(outs[-1], ref))
                cases += 1
            if not all(np.array_equal(o, outs[0]) for o in outs):
                bad_split.append((case, h, seq))
    ok = worst <= RTOL and not bad_split
    criterion("N1", f"reference validate generator (head_dim 1..4, padded) through the GPU drop-in: {cases} "
                    f"(case, split) pairs within {worst:.2e} <= 2e-2 of the fp64 oracle, split-invariant", ok)
    assert worst <= RTOL, worst
    assert not bad_split, bad_split


@pytest.mark.parametrize("d", [128, 64, 48, 3])
def test_decode_attention_batch_ragged(d):
    """Per-sequence caches of different lengths (the reference's KVState is per sequence) in one ragged
    K2 launch: each row equals the single-sequence call bit for bit, and the fp64 oracle within 2e-2."""
    rng = np.random.default_rng(d)
    heads = 2
    h = heads * d
    lens = [1, 37, 130, 64, 5]
    w_o = rng.standard_normal((h, h)) / np.sqrt(h)
    kvs, qs, refs = [], [], []
    for s in lens:
        k, v = rng.standard_normal((heads, s, d)), rng.standard_normal((heads, s, d))
        kvs.append(gn.KVState(k, v))
        qs.append(rng.standard_normal(h))
        refs.append(nr.decode_attention(qs[-1], nr.KVState(k, v), w_o))
    out = gn.decode_attention_batch(np.stack(qs), kvs, w_o)
    for i in range(len(lens)):
        single = gn.decode_attention(qs[i], kvs[i], w_o)
        assert np.array_equal(out[i], single), i
        assert _rel(out[i], refs[i]) <= RTOL, (i, _rel(out[i], refs[i]))
    with pytest.raises(ValueError, match="empty"):
        gn.decode_attention_batch(np.stack(qs[:2]), [kvs[0], gn.KVState(kvs[1].keys[:, :0], kvs[1].values[:, :0])],
                                  w_o)
    with pytest.raises(ValueError, match="head_dim"):
        gn.decode_attention(np.zeros(2 * 130), gn.KVState(np.zeros((2, 3, 130)), np.zeros((2, 3, 130))),
                            np.eye(260))
