#!/usr/bin/env bash
# Per-config measurements (BASELINE.json configs 1 and 3) with bench.py on one GPU.
# Config 3 at G GPUs = batch 32/G per GPU on its own PCIe link: the per-GPU shard is measured here;
# the same for config 2 (the driver's N-GPU bench partitions its batch of 32 the same way).
set -u
out=${1:-gpurun_out/r02_configs.jsonl}
: > "$out"
run() { timeout 600 python bench.py --steps 8 --warmup 3 --no-alt --cpu-budget 4 "$@" >> "$out" 2>> "${out%.jsonl}.err"; }
run --model opt-125m --batch 4 --prompt 256
run --model opt-13b --batch 32 --prompt 1024
run --model opt-13b --batch 16 --prompt 1024
run --model opt-13b --batch 8 --prompt 1024
run --model opt-13b --batch 4 --prompt 1024
run --model opt-6.7b --batch 16 --prompt 1024
run --model opt-6.7b --batch 8 --prompt 1024
run --model opt-6.7b --batch 4 --prompt 1024
