set -x
timeout 900 python -m pytest tests/test_gpu_multigrid.py -x -q > gpurun_out/mg6_pytest.log 2>&1; echo "pytest rc=$?"
for args in "--precision mixed --h-coarse 64,32,16,8 --coarse-iterations 50" "--precision mixed --coarse-matrix --h-coarse 64,32,16,8 --coarse-iterations 50" "--h-coarse 64,32,16,8 --coarse-iterations 50"; do
  timeout 900 python tools/bench_configs.py mg --n5 128 $args >> gpurun_out/mg6_128.jsonl 2>> gpurun_out/mg6_128.err; echo "rc=$?"
done
