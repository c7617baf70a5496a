#!/usr/bin/env bash
# X-chunking A/B on the small per-GPU batch shards (the batch-partitioned multi-GPU mode's per-rank
# workload): one bench line per (model, batch, knob), tag in <out>.tags
out=${1:-gpurun_out/chunk_ab.jsonl}
mkdir -p "$(dirname "$out")"
r() { tag=$1; model=$2; b=$3; shift 3; env "$@" timeout 600 python bench.py --model $model --batch $b --prompt 1024 --no-alt --no-cpu-baseline >> "$out" 2>>"${out%.jsonl}.err" && echo "$tag $model b$b $*" >> "${out%.jsonl}.tags"; }
for b in 4 8 16; do
  r new opt-6.7b $b X=1
  r old4mb opt-6.7b $b KVPR_CHUNK_MB=4
done
r new opt-13b 4 X=1
r old4mb opt-13b 4 KVPR_CHUNK_MB=4
