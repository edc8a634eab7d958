# p-multigrid: GPU tests + C5-problem solve comparison
set -x
timeout 900 python -m pytest tests/test_gpu_multigrid.py tests/test_gpu_solvers.py -x -q > gpurun_out/mg_pytest.log 2>&1; echo "pytest rc=$?"
timeout 900 python tools/bench_configs.py mg --n5 64 > gpurun_out/mg_64.jsonl 2> gpurun_out/mg_64.err; echo "mg64 rc=$?"
timeout 1500 python tools/bench_configs.py mg --n5 128 > gpurun_out/mg_128.jsonl 2> gpurun_out/mg_128.err; echo "mg128 rc=$?"
