timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/f7_pytest.log 2>&1; echo "pytest rc=$?"
