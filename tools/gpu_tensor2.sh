# low-degree tensor variants (data prefetch, occupancy) and vertex renumbering
for p in 1 2; do
  timeout 300 python tools/quick_bench.py cgr:$p:48:0:tensor cgv:$p:48:0:tensor cgv:$p:48:8:tensor cgv:$p:48:9:tensor cgv:$p:48:10:tensor cgv:$p:48:11:tensor cgv:$p:48:12:tensor cgv:$p:48:13:tensor cgv:$p:48:14:tensor cg:$p:48:0:tensor cg:$p:48:8:tensor cg:$p:48:9:tensor >> gpurun_out/t2_qb.jsonl 2>> gpurun_out/t2_qb.err
done
for p in 3 4; do
  timeout 300 python tools/quick_bench.py cgr:$p:48:0:tensor cgv:$p:48:0:tensor >> gpurun_out/t2_qb.jsonl 2>> gpurun_out/t2_qb.err
done
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tensor" > gpurun_out/t2_pytest.log 2>&1; echo "pytest rc=$?"
echo done
