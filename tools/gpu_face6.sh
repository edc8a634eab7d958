timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "face" > gpurun_out/f6_pytest.log 2>&1; echo "pytest rc=$?"
timeout 600 python tools/quick_bench.py helm:2:96:0 helm:2:96:208 helm:2:96:224 helm:2:96:240 dg:3:64:0 dg:3:64:208 dg:3:64:224 dg:3:64:240 dg:2:64:0 dg:2:64:208 dg:2:64:224 dg:4:48:0 dg:4:48:224 dg:4:48:240 > gpurun_out/f6_qb.jsonl 2> gpurun_out/f6_qb.err
echo done
