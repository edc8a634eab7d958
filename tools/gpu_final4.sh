set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g4_pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g4_smoke.log 2>&1; echo "smoke rc=$?"
