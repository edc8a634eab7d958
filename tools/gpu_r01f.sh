timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/f_pytest.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --dist --steps 3 --warmup 3 --no-cpu --no-quadrature > gpurun_out/f_bench_dist.json 2> gpurun_out/f_bench_dist.err; echo "bench dist rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu --no-quadrature > gpurun_out/f_ncu_bench.log 2>&1; echo "ncu list rc=$?"
K='regex:cell_apply'
timeout 900 ncu -f --set full --clock-control none --import-source on -k "$K" -s 3 -c 1 -o /tmp/f_cg4 python tools/quick_bench.py cg:4:48 > gpurun_out/ncu_f_cg4.log 2>&1
ncu -i /tmp/f_cg4.ncu-rep --page raw --csv > gpurun_out/ncu_f_cg4_raw.csv 2>/dev/null
ncu -i /tmp/f_cg4.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_f_cg4_sass.csv 2>/dev/null
echo done
