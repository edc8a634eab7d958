timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/d_pytest.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/d_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python tools/bench_configs.py c3 c4 c5 > gpurun_out/d_configs.jsonl 2> gpurun_out/d_configs.err; echo "configs rc=$?"
timeout 900 python bench.py > gpurun_out/d_bench.json 2> gpurun_out/d_bench.err; echo "bench rc=$?"
echo done
