#!/usr/bin/env bash
# compute-sanitizer passes over the kernel tests (memcheck all, racecheck on the round-2 kernels).
# Usage (on the box): bash tools/sanitize_round.sh > gpurun_out/<tag>_sanitizer.txt 2>&1
set -u
CS=/usr/local/cuda/bin/compute-sanitizer
echo "## memcheck: tests/test_kernels_gpu.py + tests/test_numerics_gpu.py"
timeout 1200 $CS --tool memcheck --print-limit 20 python -m pytest tests/test_kernels_gpu.py tests/test_numerics_gpu.py -q 2>&1 | tail -6
echo "## racecheck: stream-K decode GEMM, tiled weights, ragged K2"
timeout 1200 $CS --tool racecheck --print-limit 20 python -m pytest tests/test_kernels_gpu.py -q -k "stream_k or tiled" 2>&1 | tail -8
timeout 900 $CS --tool racecheck --print-limit 20 python -m pytest tests/test_numerics_gpu.py -q -k "ragged" 2>&1 | tail -6
echo "## synccheck: stream-K decode GEMM"
timeout 900 $CS --tool synccheck --print-limit 20 python -m pytest tests/test_kernels_gpu.py -q -k "stream_k" 2>&1 | tail -6
echo "## memcheck: executor + runtime (decode pipeline, full-size tests excluded)"
timeout 1500 $CS --tool memcheck --print-limit 20 python -m pytest tests/test_executor_gpu.py tests/test_runtime_gpu.py -q -k "not full_size and not host_time" 2>&1 | tail -6
echo "## racecheck + memcheck: tensor-core prefill attention, fused layer tail"
timeout 900 $CS --tool racecheck --print-limit 20 python -m pytest tests/test_kernels_gpu.py -q -k "prefill" 2>&1 | tail -4
timeout 900 $CS --tool memcheck --print-limit 20 python -m pytest tests/test_kernels_gpu.py -q -k "prefill" 2>&1 | tail -4
timeout 1500 $CS --tool racecheck --print-limit 20 python -m pytest tests/test_layer_tail_gpu.py -q -k "matches_fp32 or bitwise_repeatable or multikernel" 2>&1 | tail -4
echo "## memcheck: grouped KV-tail DMAs (executor)"
timeout 1500 $CS --tool memcheck --print-limit 20 python -m pytest tests/test_executor_gpu.py -q -k "grouped" 2>&1 | tail -4
