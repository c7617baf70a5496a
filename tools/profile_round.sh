#!/usr/bin/env bash
# One box pass for profiles/: the default bench (plain run, no profiler), the ncu launch list of the
# same command (short), config 1's launch list, and full captures of the hot kernels.
# Usage (on the box): bash tools/profile_round.sh <tag>   -> gpurun_out/<tag>_*
set -u
tag=${1:-r02}
mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/${tag}_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-alt --no-cpu-baseline --fixed-profile > gpurun_out/${tag}_launches_bench.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/${tag}_c1_launches.csv \
    python bench.py --model opt-125m --batch 4 --prompt 256 --steps 4 --warmup 1 --no-alt --no-cpu-baseline \
    --fixed-profile > gpurun_out/${tag}_c1_launches_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_tcgen05_2sm -s 1 -c 1 -o gpurun_out/${tag}_k1_chunk \
    python tools/ncu_target.py k1chunk > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:decode_attn_kernel -s 1 -c 1 -o gpurun_out/${tag}_k2 \
    python tools/ncu_target.py k2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_swapab -s 2 -c 6 -o gpurun_out/${tag}_dec_gemm \
    python tools/ncu_target.py dec > /dev/null 2>&1
ls -la gpurun_out/${tag}_*
