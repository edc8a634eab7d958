set -u
mkdir -p gpurun_out
TMF_FACE_VARIANT=10 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "dg or helm" 2>&1 | tail -2
: > gpurun_out/sg_timing.jsonl
for v in 0 10 11 12 0 10; do
  echo "{\"face_variant\": $v}" >> gpurun_out/sg_timing.jsonl
  TMF_FACE_VARIANT=$v timeout 900 python tools/loop_bench.py dg:3:64:r:auto:auto helmk:2:96:r:auto:auto >> gpurun_out/sg_timing.jsonl 2>> gpurun_out/sg_timing.err
done
cut -c1-120 gpurun_out/sg_timing.jsonl; tail -3 gpurun_out/sg_timing.err
