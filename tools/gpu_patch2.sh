set -x
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -x -q -k "patch" > gpurun_out/patch_parity.log 2>&1; echo "parity rc=$?"
for spec in cgr:1:48:0:dmma:off cgr:1:48:0:dmma:on cgr:2:48:0:dmma:off cgr:2:48:0:dmma:on cgr:3:48:0:dmma:off cgr:3:48:0:dmma:on cg:1:48:0:dmma:on; do
  timeout 300 python tools/quick_bench.py $spec >> gpurun_out/patch_qb2.jsonl 2>> gpurun_out/patch_qb2.err
done
echo done
