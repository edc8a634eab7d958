timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/c_pytest.log 2>&1; echo "pytest rc=$?"
timeout 900 python bench.py > gpurun_out/c_bench.json 2> gpurun_out/c_bench.err; echo "bench rc=$?"
timeout 1500 python tools/bench_configs.py c1 c3 c4 c5 csr > gpurun_out/c_configs.jsonl 2> gpurun_out/c_configs.err; echo "configs rc=$?"
echo done
