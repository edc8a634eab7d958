set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "face_variants" > gpurun_out/face_parity.log 2>&1; echo "parity rc=$?"
python tools/quick_bench.py helmr:2:96 helmr:2:96:176 helmr:2:96:192 helmr:2:96:208 helmr:2:96:224 dgr:3:64 dgr:3:64:176 dgr:3:64:192 dgr:3:64:208 dgr:3:64:224 > gpurun_out/face1.jsonl 2> gpurun_out/face1.err
echo done
