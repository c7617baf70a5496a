"""CPU oracle for KVPR's per-layer decode path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` leg may import this package, and only as the checker or
the reported CPU baseline.  The product path (paper_2411_17089_b200) never
imports it; it fails loudly when libkvpr.so is missing.

Contents (each function cites the reference file:line it restates):
  numerics_ref  fp64 NumPy restatement of kvoverlap.numerics
                (split_merge_kv, decode_attention, build_kv, append_token_kv).
                Pinned against fixtures produced by the live reference:
                tests/golden/numerics_golden.npz (tests/golden/make_golden.py).
  scheduler_ref exhaustive-scan restatement of Eq. 10 (scheduler.py:76-92,
                176-188).  Pinned against tests/golden/scheduler_golden.json.
  opt_ref       NumPy OPT decoder with host-offloaded X / KV stores and the
                split-merge rebuild at the planned l each step (numerics.py:
                107-191 for the split/merge attention; OPT layer semantics from
                transformers' modeling_opt since the reference has no decoder
                — SURVEY.md §8c: logits/greedy parity is *unpinned by the
                reference*; its split/merge core is pinned through
                numerics_ref, and its layer semantics are cross-checked against
                HF OPTForCausalLM in tests/test_oracle_cpu.py).
"""
