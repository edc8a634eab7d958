set -x
timeout 600 python -m pytest tests/test_gpu_multigrid.py tests/test_gpu_solvers.py -x -q > gpurun_out/c4mg_pytest.log 2>&1; echo "pytest rc=$?"
timeout 900 python tools/bench_configs.py mgc4 --n4 64 --tau-scale 4 > gpurun_out/c4mg_64_t4.jsonl 2> gpurun_out/c4mg_64_t4.err; echo "rc=$?"
timeout 1500 python tools/bench_configs.py mgc4 --n4 128 --tau-scale 4 > gpurun_out/c4mg_128_t4.jsonl 2> gpurun_out/c4mg_128_t4.err; echo "rc=$?"
