set -x
timeout 600 python -m pytest tests/test_gpu_multigrid.py -x -q > gpurun_out/mg9_pytest.log 2>&1; echo "pytest rc=$?"
H=64-32-16-8
timeout 1500 python tools/mg_sweep.py 128 321:3:20:mixed:csr:$H 321:2:20:mixed:csr:$H 321:3:50:mixed:csr:$H 321:3:10:mixed:csr:$H > gpurun_out/mg9_sweep.jsonl 2> gpurun_out/mg9_sweep.err; echo "rc=$?"
