timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "face" > gpurun_out/f3_pytest.log 2>&1; echo "pytest rc=$?"
V=""
for v in 0 16 32 48 64 80 96; do V="$V dg:3:64:$v:auto:auto:tensor"; done
timeout 600 python tools/quick_bench.py dg:3:64:0:auto:auto:quadrature $V > gpurun_out/f3_qb.jsonl 2> gpurun_out/f3_qb.err
V=""
for v in 0 16 32 48 64 80 96; do V="$V helm:2:96:$v:auto:auto:tensor"; done
timeout 600 python tools/quick_bench.py helm:2:96:0:auto:auto:quadrature $V dg:2:64:0:auto:auto:quadrature dg:2:64:0:auto:auto:tensor dg:4:48:0:auto:auto:quadrature dg:4:48:0:auto:auto:tensor dg:1:96:0:auto:auto:quadrature dg:1:96:0:auto:auto:tensor >> gpurun_out/f3_qb.jsonl 2>> gpurun_out/f3_qb.err
echo done
