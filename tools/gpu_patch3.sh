set -x
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -x -q -k "patch" > gpurun_out/patch_parity.log 2>&1; echo "parity rc=$?"
python tools/loop_bench.py cgr:1:48:0:dmma:on cgr:1:48:1:dmma:on cgr:1:48:2:dmma:on cgr:1:48:5:dmma:on cgr:1:48:0:dmma:off cgr:2:48:0:dmma:on cgr:2:48:0:dmma:off cgr:3:48:0:dmma:on cgr:3:48:0:dmma:off > gpurun_out/loop3.jsonl 2> gpurun_out/loop3.err
echo done
