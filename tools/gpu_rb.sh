#!/bin/bash
# register-resident tables / pair group: parity then A/B timings of the P3 / P4 modal cell kernels
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/rb_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/rb_tests.log
tail -5 gpurun_out/rb_tests.log
: > gpurun_out/rb_timing.jsonl
for v in 0 1 2 3 4 5 6; do
  echo "{\"p3_variant\": $v}" >> gpurun_out/rb_timing.jsonl
  TMF_CELL_VARIANT=$v timeout 600 python tools/loop_bench.py cg:3:48:r:auto:auto cg:3:48:u:auto:auto >> gpurun_out/rb_timing.jsonl 2>> gpurun_out/rb_timing.err
done
for v in 0 1 2 3 4; do
  echo "{\"p4_variant\": $v}" >> gpurun_out/rb_timing.jsonl
  TMF_CELL_VARIANT=$v timeout 600 python tools/loop_bench.py cg:4:48:r:auto:auto cg:4:48:u:auto:auto >> gpurun_out/rb_timing.jsonl 2>> gpurun_out/rb_timing.err
done
# parity of the variants on the goldens
for v in 1 2 3 4 5 6; do
  TMF_CELL_VARIANT=$v timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "cg" > gpurun_out/rb_tests_v$v.log 2>&1
  echo "variant $v tests rc=$?"; tail -1 gpurun_out/rb_tests_v$v.log
done
cat gpurun_out/rb_timing.jsonl; tail -5 gpurun_out/rb_timing.err
