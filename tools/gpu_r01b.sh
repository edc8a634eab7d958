# tensor engine as default: GPU tests, bench, launch list, ncu of the tensor cell kernels
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/b_pytest.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/b_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/b_bench.json 2> gpurun_out/b_bench.err; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/b_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu --no-quadrature > gpurun_out/b_ncu_bench.log 2>&1; echo "ncu list rc=$?"
K='regex:cell_tensor'
cap() {  # name spec
  timeout 600 ncu -f --set full --clock-control none --import-source on -k "$K" -s 3 -c 1 -o /tmp/$1 python tools/quick_bench.py $2 > gpurun_out/ncu_$1.log 2>&1
  ncu -i /tmp/$1.ncu-rep --page raw --csv > gpurun_out/ncu_$1_raw.csv 2>/dev/null
  ncu -i /tmp/$1.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_$1_sass.csv 2>/dev/null
  rm -f /tmp/$1.ncu-rep
}
cap t_cg4 cg:4:48
cap t_cg1r cgr:1:48
cap t_cg2r cgr:2:48
echo done
