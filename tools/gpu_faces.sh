#!/bin/bash
# split-mode modal face kernel: parity, then A/B timings against the flat layout and CTA variants
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "face_engines or defaults" > gpurun_out/faces_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/faces_tests.log
tail -15 gpurun_out/faces_tests.log
: > gpurun_out/faces_timing.jsonl
for spec in dg:3:48:r:auto:auto:modal_flat dg:3:48:r:auto:auto:modal helmk:2:64:r:auto:auto:modal_flat helmk:2:64:r:auto:auto:modal dg:4:32:r:auto:auto:modal_flat dg:4:32:r:auto:auto:modal dg:2:64:r:auto:auto:modal_flat dg:2:64:r:auto:auto:modal; do
  timeout 600 python tools/loop_bench.py $spec >> gpurun_out/faces_timing.jsonl 2>> gpurun_out/faces_timing.err
done
for v in 1 2 3 4 5; do
  for spec in dg:3:48:r:auto:auto:modal helmk:2:64:r:auto:auto:modal; do
    echo "{\"variant\": $v}" >> gpurun_out/faces_timing.jsonl
    TMF_FACE_VARIANT=$v timeout 600 python tools/loop_bench.py $spec >> gpurun_out/faces_timing.jsonl 2>> gpurun_out/faces_timing.err
  done
done
for v in 1 2; do
  echo "{\"variant\": $v}" >> gpurun_out/faces_timing.jsonl
  TMF_FACE_VARIANT=$v timeout 600 python tools/loop_bench.py dg:4:32:r:auto:auto:modal >> gpurun_out/faces_timing.jsonl 2>> gpurun_out/faces_timing.err
done
cat gpurun_out/faces_timing.jsonl; tail -5 gpurun_out/faces_timing.err
