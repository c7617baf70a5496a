#!/usr/bin/env bash
# The reference's own simulator-engine benchmark (benchmarks/bench_engine.py, read from /root/reference;
# build container only) run against this package through tests/refshim: pure-Python engine vs
# kvpr_list_schedule (csrc/sched_engine.cu), bit-identical check included.
set -eu
ROOT=$(cd "$(dirname "$0")/.." && pwd)
PYTHONPATH="$ROOT/tests/refshim:$ROOT" python /root/reference/pkg/benchmarks/bench_engine.py "$@"
