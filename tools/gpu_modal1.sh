timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_solvers.py -m gpu -x -q > gpurun_out/m1_pytest.log 2>&1; echo "pytest rc=$?"
for p in 2 3 4; do
  timeout 300 python tools/quick_bench.py cgv:$p:48:0:tensor cgv:$p:48:0:modal cgv:$p:48:8:modal cgv:$p:48:10:modal cgv:$p:48:11:modal cgv:$p:48:2:modal cgv:$p:48:14:modal cgv:$p:48:15:modal >> gpurun_out/m1_qb.jsonl 2>> gpurun_out/m1_qb.err
done
timeout 300 python tools/quick_bench.py dg:3:64:0:tensor dg:3:64:0:modal dg:2:64:0:modal dg:2:64:0:tensor >> gpurun_out/m1_qb.jsonl 2>> gpurun_out/m1_qb.err
echo done
