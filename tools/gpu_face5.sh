timeout 600 python tools/quick_bench.py helm:2:96:0 helm:2:96:112 helm:2:96:128 helm:2:96:32 helm:2:96:16 dg:3:64:0 dg:3:64:112 dg:3:64:32 > gpurun_out/f5_qb.jsonl 2> gpurun_out/f5_qb.err
echo done
