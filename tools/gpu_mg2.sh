# p/cp-multigrid GPU tests + DG C3-problem solve comparison
set -x
timeout 900 python -m pytest tests/test_gpu_multigrid.py tests/test_gpu_solvers.py -x -q > gpurun_out/mg2_pytest.log 2>&1; echo "pytest rc=$?"
timeout 900 python tools/bench_configs.py mgdg --n3 32 > gpurun_out/mgdg_32.jsonl 2> gpurun_out/mgdg_32.err; echo "mgdg32 rc=$?"
timeout 1500 python tools/bench_configs.py mgdg --n3 64 > gpurun_out/mgdg_64.jsonl 2> gpurun_out/mgdg_64.err; echo "mgdg64 rc=$?"
timeout 1500 python tools/bench_configs.py mg --n5 128 > gpurun_out/mg_128b.jsonl 2> gpurun_out/mg_128b.err; echo "mg128 rc=$?"
