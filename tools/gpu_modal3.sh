for p in 2 3 4; do
  V=""
  for v in 0 1 3 4 6 7 8 9 10 11 12; do V="$V cgv:$p:48:$v:modal"; done
  timeout 600 python tools/quick_bench.py $V >> gpurun_out/m3_qb.jsonl 2>> gpurun_out/m3_qb.err
done
timeout 600 python tools/quick_bench.py dg:3:64:0:modal dg:3:64:8:modal dg:3:64:10:modal dg:3:64:11:modal dg:3:64:9:modal cgv:2:48:0:dmma cgv:3:48:0:dmma >> gpurun_out/m3_qb.jsonl 2>> gpurun_out/m3_qb.err
echo done
