timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "face" > gpurun_out/f4_pytest.log 2>&1; echo "pytest rc=$?"
V=""
for v in 0 80 16 32 2048 2128 3072 3152 3920 4000; do V="$V helm:2:96:$v"; done
timeout 900 python tools/quick_bench.py $V > gpurun_out/f4_qb.jsonl 2> gpurun_out/f4_qb.err
V=""
for v in 0 32 96 2048 2080 3072 3104 3840; do V="$V dg:3:64:$v"; done
timeout 900 python tools/quick_bench.py $V >> gpurun_out/f4_qb.jsonl 2>> gpurun_out/f4_qb.err
echo done
