set -x
timeout 600 python tools/ncu_f32.py 96 > gpurun_out/ncu_mg_plain.log 2>&1 || exit 1
for K in cell_f32_kernel restrict_kernel prolongate_kernel chebyshev_kernel; do
  timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -o /tmp/$K python tools/ncu_f32.py 96 > gpurun_out/ncu_mg_$K.log 2>&1
  ncu -i /tmp/$K.ncu-rep --page raw --csv > gpurun_out/ncu_mg_${K}_raw.csv 2>/dev/null
done
timeout 1200 python tools/mg_sweep.py 128 321:2:30:mixed:csr 321:2:60:mixed:csr 321:2:100:mixed:csr 321:3:60:mixed:csr 31:2:60:mixed:csr > gpurun_out/mg_sweep2.jsonl 2> gpurun_out/mg_sweep2.err
echo done
