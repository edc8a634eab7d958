timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tensor_variants" > gpurun_out/p1_pytest.log 2>&1; echo "pytest rc=$?"
timeout 600 python tools/quick_bench.py cgr:1:48:0 cgr:1:48:15 cgr:1:48:13 cgr:1:48:7 cg:1:48:0 cg:1:48:15 cg:1:48:13 cg:1:48:7 cgr:1:96:0 cgr:1:96:15 cgr:1:96:13 cgr:1:96:7 > gpurun_out/p1_qb.jsonl 2> gpurun_out/p1_qb.err
echo done
