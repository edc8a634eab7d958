#!/bin/bash
# one gpurun iteration: targeted GPU tests, then developer timings (tools/loop_bench.py)
set -u
mkdir -p gpurun_out
T=${TESTS:-}
if [ -n "$T" ]; then
  timeout 900 python -m pytest $T -x -q -p no:cacheprovider > gpurun_out/iter_tests.log 2>&1
  echo "tests rc=$?" >> gpurun_out/iter_tests.log
  tail -5 gpurun_out/iter_tests.log
fi
if [ -n "${SPECS:-}" ]; then
  timeout 900 python tools/loop_bench.py $SPECS > gpurun_out/iter_timing.jsonl 2> gpurun_out/iter_timing.err
  echo "timing rc=$?"; cat gpurun_out/iter_timing.jsonl; tail -5 gpurun_out/iter_timing.err
fi
