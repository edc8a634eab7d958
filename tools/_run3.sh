set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale_parity.py -x -q -p no:cacheprovider 2>&1 | tail -3
: > gpurun_out/run_timing.jsonl
for r in 0 2 8 16; do
  echo "{\"face_run\": $r}" >> gpurun_out/run_timing.jsonl
  TMF_FACE_RUN=$r timeout 900 python tools/loop_bench.py dg:3:64:r:auto:auto dg:4:40:r:auto:auto dg:2:64:r:auto:auto helmk:2:64:r:auto:auto dg:3:64:u:auto:auto >> gpurun_out/run_timing.jsonl 2>> gpurun_out/run_timing.err
done
cut -c1-190 gpurun_out/run_timing.jsonl; tail -3 gpurun_out/run_timing.err
