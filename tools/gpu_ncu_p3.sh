set -x
K='regex:cell_apply'
python tools/quick_bench.py cgr:3:48 > /dev/null 2>&1 || exit 1
cap() {  # name spec [source]
  ncu -f --set full --clock-control none $3 -k "$K" -s 3 -c 1 -o /tmp/$1 python tools/quick_bench.py $2 > gpurun_out/ncu_$1.log 2>&1
  ncu -i /tmp/$1.ncu-rep --page raw --csv > gpurun_out/ncu_$1_raw.csv 2>/dev/null
  ncu -i /tmp/$1.ncu-rep --page details --csv > gpurun_out/ncu_$1_details.csv 2>/dev/null
  [ -n "$3" ] && ncu -i /tmp/$1.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_$1_sass.csv 2>/dev/null
  rm -f /tmp/$1.ncu-rep
}
cap cg3r_grp cgr:3:48 --import-source=on
cap cg2r_dmma cgr:2:48 --import-source=on
echo done
