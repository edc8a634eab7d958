set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/dfma_parity.log 2>&1; echo "parity rc=$?"
for spec in cg:1:48:0:dmma cg:1:48:0:dfma cg:1:48:1:dfma cg:1:48:3:dfma cg:1:48:4:dfma cg:1:48:5:dfma cg:1:48:7:dfma cg:1:48:8:dfma \
            cg:2:48:0:dmma cg:2:48:1:dfma cg:2:48:2:dfma cg:2:48:3:dfma cg:2:48:4:dfma cg:2:48:5:dfma cg:2:48:6:dfma cg:2:48:7:dfma cg:2:48:8:dfma \
            cgr:2:48:0:dmma cgr:2:48:4:dfma cg:3:48:0:dmma cg:3:48:3:dfma cg:3:48:4:dfma cg:3:48:6:dfma \
            helmr:2:48:0:dmma helmr:2:48:0:dfma helmr:2:48:3:dfma helmr:2:48:4:dfma dgr:2:48:0:dmma dgr:2:48:4:dfma; do
  timeout 300 python tools/quick_bench.py $spec >> gpurun_out/dfma_qb.jsonl 2>> gpurun_out/dfma_qb.err
done
echo done
