#!/usr/bin/env bash
# Profiles for profiles/: ncu launch list of the bench command + full captures of the hot kernels.
# Usage (on the box): bash tools/profile_round.sh <tag>   -> gpurun_out/<tag>_*
set -u
tag=${1:-r01}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/${tag}_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-alt --no-cpu-baseline --fixed-profile > gpurun_out/${tag}_launches_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_tcgen05_2sm -s 1 -c 1 -o gpurun_out/${tag}_k1_chunk \
    python tools/ncu_target.py k1chunk > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:decode_attn_kernel -s 1 -c 1 -o gpurun_out/${tag}_k2 \
    python tools/ncu_target.py k2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_swapab -s 2 -c 5 -o gpurun_out/${tag}_dec_gemm \
    python tools/ncu_target.py dec > /dev/null 2>&1
ls -la gpurun_out/${tag}_*
