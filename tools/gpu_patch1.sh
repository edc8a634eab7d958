set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -x -q -k "patch or engines" > gpurun_out/patch_parity.log 2>&1; echo "parity rc=$?"
for spec in cgr:1:48:0:dmma cgr:1:48:0:dfma:off cgr:1:48:0:dfma:on cgr:1:48:3:dfma:on cgr:1:48:5:dfma:on cgr:1:48:7:dfma:on cgr:1:48:2:dfma:on \
            cgr:2:48:0:dmma cgr:2:48:0:dfma:on cgr:2:48:3:dfma:on cgr:2:48:2:dfma:on cgr:2:48:6:dfma:on cgr:2:48:7:dfma:on \
            cgr:3:48:0:dmma cgr:3:48:3:dfma:on cgr:3:48:4:dfma:on cg:1:48:0:dfma:on; do
  timeout 300 python tools/quick_bench.py $spec >> gpurun_out/patch_qb.jsonl 2>> gpurun_out/patch_qb.err
done
echo done
