# end-of-session validation: full GPU suite, smoke, bench (default contract run), reference arm, MG best
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g3_pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g3_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/g3_bench.json 2> gpurun_out/g3_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/g3_bench_ref.json 2> gpurun_out/g3_bench_ref.err; echo "ref rc=$?"
timeout 900 python tools/bench_configs.py mg --n5 128 --best > gpurun_out/g3_mg_best.jsonl 2> gpurun_out/g3_mg_best.err; echo "mg rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/g3_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/g3_ncu.log 2>&1; echo "ncu rc=$?"
echo done
