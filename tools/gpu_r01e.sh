timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/e_pytest.log 2>&1; echo "pytest rc=$?"
timeout 900 python bench.py > gpurun_out/e_bench.json 2> gpurun_out/e_bench.err; echo "bench rc=$?"
timeout 1500 python tools/bench_configs.py c1 c3 c4 c5 > gpurun_out/e_configs.jsonl 2> gpurun_out/e_configs.err; echo "configs rc=$?"
K='regex:cell_apply'
cap() {
  timeout 900 ncu -f --set full --clock-control none --import-source on -k "$K" -s 3 -c 1 -o /tmp/$1 python tools/quick_bench.py $2 > gpurun_out/ncu_$1.log 2>&1
  ncu -i /tmp/$1.ncu-rep --page raw --csv > gpurun_out/ncu_$1_raw.csv 2>/dev/null
  ncu -i /tmp/$1.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_$1_sass.csv 2>/dev/null
  rm -f /tmp/$1.ncu-rep
}
cap m_cg4 cg:4:48
cap m_cg3v cgv:3:48
echo done
