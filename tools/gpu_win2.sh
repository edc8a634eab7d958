set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "dg or DG or sipg or helm or face or golden or parity" > gpurun_out/w2_pytest.log 2>&1; echo "pytest rc=$?"
timeout 900 python tools/quick_bench.py dgv:3:64:0:auto:auto:auto:window dgv:3:64:0:auto:auto:auto:plain dg:3:64:0:auto:auto:auto:window dg:3:64:0:auto:auto:auto:plain dgv:2:96:0:auto:auto:auto:window dgv:2:96:0:auto:auto:auto:plain > gpurun_out/w2_times.jsonl 2> gpurun_out/w2_times.err; echo "rc=$?"
timeout 900 ncu -f --set full --clock-control none -k regex:face_apply -s 2 -c 1 -o /tmp/fw python tools/quick_bench.py dgv:3:64:0:auto:auto:auto:window > gpurun_out/w2_ncu.log 2>&1
ncu -i /tmp/fw.ncu-rep --page raw --csv > gpurun_out/w2_ncu_raw.csv 2>/dev/null
echo done
