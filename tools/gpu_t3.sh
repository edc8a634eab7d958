timeout 600 python tools/quick_bench.py cgr:1:48:0:tensor cgr:1:96:0:tensor cgr:1:96:1:tensor cgr:1:96:4:tensor cgr:1:96:6:tensor cgr:2:96:0:tensor cgr:2:96:6:tensor > gpurun_out/t3_qb.jsonl 2> gpurun_out/t3_qb.err
echo done
