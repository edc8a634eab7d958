cap() {  # name regex spec
  timeout 900 ncu -f --set full --clock-control none --import-source on -k "$2" -s $4 -c 1 -o /tmp/$1 python tools/quick_bench.py $3 > gpurun_out/ncu_$1.log 2>&1
  ncu -i /tmp/$1.ncu-rep --page raw --csv > gpurun_out/ncu_$1_raw.csv 2>/dev/null
  ncu -i /tmp/$1.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_$1_sass.csv 2>/dev/null
  rm -f /tmp/$1.ncu-rep
}

cap g_fh2 regex:face_apply helm:2:64 2
cap g_fd3 regex:face_apply dg:3:48 2
echo done
