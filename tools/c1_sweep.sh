#!/usr/bin/env bash
# Config-1 decode variants through the native executor (tools/issue_probe.py), one JSON line each:
# where does a small-model layer's time go?  column plan (default), deeper buffering, X resident
# with every position recomputed (no PCIe on the path: the pure GPU chain), all-KV streamed (no K1).
# Usage (on the box): bash tools/c1_sweep.sh <tag>  -> gpurun_out/<tag>_c1_sweep.jsonl
set -u
tag=${1:-c1}
out=gpurun_out/${tag}_c1_sweep.jsonl
mkdir -p gpurun_out
: > "$out"
run() { timeout 300 python tools/issue_probe.py --steps 8 "$@" >> "$out" 2>> gpurun_out/${tag}_c1_sweep.err; }
run
run --nbuf 3
run --nbuf 4
run --x-resident
run --x-resident --split -1
run --split 0
run --split -1
KVPR_PDL=0 run
cat "$out"
