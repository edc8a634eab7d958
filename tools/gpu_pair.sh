timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_solvers.py -m gpu -x -q > gpurun_out/pr_pytest.log 2>&1; echo "pytest rc=$?"
timeout 600 python tools/quick_bench.py cgv:3:48:0 cg:3:48:0 cgv:3:48:14 cgv:3:48:11 cgv:3:48:10 dg:3:64:0 > gpurun_out/pr_qb.jsonl 2> gpurun_out/pr_qb.err
echo done
