# final validation + DG smoothing-degree sweep
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g2_pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g2_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/g2_bench.json 2> gpurun_out/g2_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/g2_bench_ref.json 2> gpurun_out/g2_bench_ref.err; echo "ref rc=$?"
for d in 2 3 4 6; do
  timeout 600 python tools/bench_configs.py mgdg --n3 32 --h-coarse 16,8,4 --dg-smoothing-degree $d >> gpurun_out/g2_mgdg_sweep.jsonl 2>> gpurun_out/g2_mgdg_sweep.err
done
echo done
