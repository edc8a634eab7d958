# end-of-session verification: GPU tests, smoke, bench line, launch list, ncu of the top kernel
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/g5_pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g5_smoke.log 2>&1; echo "smoke rc=$?"
timeout 400 python bench.py > gpurun_out/g5_bench.log 2>&1; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/g5_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu --no-quadrature > gpurun_out/g5_ncu_launch.log 2>&1; echo "ncu-list rc=$?"
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:cell_apply -s 3 -c 1 -o /tmp/g5_p4 \
  python tools/quick_bench.py cg:4:48 > gpurun_out/g5_ncu_p4.log 2>&1; echo "ncu-full rc=$?"
ncu -i /tmp/g5_p4.ncu-rep --page raw --csv > gpurun_out/g5_ncu_p4_raw.csv 2>/dev/null
