timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "variants" > gpurun_out/wa_pytest.log 2>&1; echo "pytest rc=$?"
timeout 600 python tools/quick_bench.py cgv:1:48:0 cgv:1:48:12 cg:1:48:0 cg:1:48:12 cgv:2:48:0 cgv:2:48:12 cg:2:48:0 cg:2:48:12 cgv:3:48:0 cgv:3:48:12 cg:3:48:0 cg:3:48:12 cgv:4:48:0 cgv:4:48:12 cg:4:48:0 cg:4:48:12 cgv:2:48:12:tensor cgv:2:48:0:tensor cgv:1:96:0 cgv:1:96:12 > gpurun_out/wa_qb.jsonl 2> gpurun_out/wa_qb.err
echo done
