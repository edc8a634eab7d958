set -u
mkdir -p gpurun_out
: > gpurun_out/runs_timing.jsonl
for v in 0 6 7 8 9; do
  echo "{\"face_variant\": $v}" >> gpurun_out/runs_timing.jsonl
  TMF_FACE_VARIANT=$v timeout 600 python tools/loop_bench.py dg:3:64:r:auto:auto dg:3:48:u:auto:auto >> gpurun_out/runs_timing.jsonl 2>> gpurun_out/runs_timing.err
done
TMF_FACE_VARIANT=8 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "dg" 2>&1 | tail -2
cat gpurun_out/runs_timing.jsonl | cut -c1-200; tail -3 gpurun_out/runs_timing.err
