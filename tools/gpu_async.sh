timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "modal" > gpurun_out/as_pytest.log 2>&1; echo "pytest rc=$?"
for p in 2 3 4; do
  timeout 600 python tools/quick_bench.py cgv:$p:48:0 cgv:$p:48:6 cgv:$p:48:5 cgv:$p:48:7 cg:$p:48:0 cg:$p:48:5 cg:$p:48:7 >> gpurun_out/as_qb.jsonl 2>> gpurun_out/as_qb.err
done
timeout 600 python tools/quick_bench.py dg:3:64:0 dg:3:64:5 dg:3:64:7 >> gpurun_out/as_qb.jsonl 2>> gpurun_out/as_qb.err
echo done
