set -x
timeout 900 python -m pytest tests/test_gpu_multigrid.py -x -q > gpurun_out/mg5_pytest.log 2>&1; echo "pytest rc=$?"
timeout 900 python tools/bench_configs.py mg --n5 128 --precision mixed --coarse-matrix > gpurun_out/mg_128_mixed_csr.jsonl 2> gpurun_out/mg_128_mixed_csr.err; echo "rc=$?"
timeout 900 python tools/bench_configs.py mg --n5 128 --coarse-matrix > gpurun_out/mg_128_f64_csr.jsonl 2> gpurun_out/mg_128_f64_csr.err; echo "rc=$?"
