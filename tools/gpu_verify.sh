# fresh-box verification: GPU tests, smoke, default bench, reference arm
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/v_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/v_pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/v_bench.json 2> gpurun_out/v_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/v_bench_ref.json 2> gpurun_out/v_bench_ref.err; echo "ref rc=$?"
echo done
