nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/mb_smi.txt 2>&1
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/mb_clocks.csv &
SMI=$!
timeout 120 ./tools/microbench/fp64_peak > gpurun_out/mb_fp64.json 2>&1
echo "exit $?" >> gpurun_out/mb_fp64.json
kill $SMI
lscpu | head -20 > gpurun_out/mb_lscpu.txt; nproc >> gpurun_out/mb_lscpu.txt
