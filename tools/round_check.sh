#!/usr/bin/env bash
# One GPU-box pass: full GPU test suite, smoke, the headline bench, config-1 bench, reference arm.
# Usage (on the box): bash tools/round_check.sh <tag>   -> gpurun_out/<tag>_*.{log,json}
set -u
tag=${1:-check}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rA > gpurun_out/${tag}_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_smoke.log
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
timeout 600 python bench.py --model opt-125m --batch 4 --prompt 256 --no-alt --cpu-budget 4 > gpurun_out/${tag}_bench_config1.json 2> gpurun_out/${tag}_bench_config1.err
timeout 600 python bench.py --impl reference > gpurun_out/${tag}_bench_reference.json 2> gpurun_out/${tag}_bench_reference.err
