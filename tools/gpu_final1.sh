# round-end style refresh: GPU tests, smoke, bench, configs, ncu of the C3 face kernel
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/f_pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err; echo "bench rc=$?"
timeout 1800 python tools/bench_configs.py c1 c3 c4 c5 > gpurun_out/f_configs.jsonl 2> gpurun_out/f_configs.err; echo "configs rc=$?"
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:face_apply -s 2 -c 1 -o /tmp/fd3 python tools/quick_bench.py dgv:3:64 > gpurun_out/f_ncu_fd3.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/fd3.ncu-rep --page raw --csv > gpurun_out/f_ncu_fd3_raw.csv 2>/dev/null
echo done
