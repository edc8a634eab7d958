K='regex:face_tensor'
cap() {  # name spec
  timeout 900 ncu -f --set full --clock-control none --import-source on -k "$K" -s 2 -c 1 -o /tmp/$1 python tools/quick_bench.py $2 > gpurun_out/ncu_$1.log 2>&1
  ncu -i /tmp/$1.ncu-rep --page raw --csv > gpurun_out/ncu_$1_raw.csv 2>/dev/null
  ncu -i /tmp/$1.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_$1_sass.csv 2>/dev/null
  rm -f /tmp/$1.ncu-rep
}
python tools/quick_bench.py helm:2:64 > /dev/null 2>&1 || exit 1
cap ft_h2 helm:2:64
cap ft_d3 dg:3:48
echo done
