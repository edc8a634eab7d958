# tensor cell engine: parity + timing sweep against the quadrature-point engine
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tensor" > gpurun_out/t1_pytest.log 2>&1; echo "pytest rc=$?"
for p in 1 2 3 4; do
  timeout 300 python tools/quick_bench.py cgr:$p:48:0:dmma cgr:$p:48:0:tensor cgr:$p:48:1:tensor cgr:$p:48:2:tensor cgr:$p:48:3:tensor cgr:$p:48:4:tensor cgr:$p:48:5:tensor cgr:$p:48:6:tensor cgr:$p:48:7:tensor >> gpurun_out/t1_qb.jsonl 2>> gpurun_out/t1_qb.err
done
timeout 300 python tools/quick_bench.py dg:3:64:0:dmma dg:3:64:0:tensor dg:3:64:2:tensor dg:3:64:5:tensor helm:2:96:0:dmma helm:2:96:0:tensor helm:2:96:2:tensor >> gpurun_out/t1_qb.jsonl 2>> gpurun_out/t1_qb.err
echo done
