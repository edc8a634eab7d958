timeout 600 python tools/quick_bench.py cgr:1:48:7 cgr:1:48:13 cgr:1:96:7 cgr:1:96:13 cg:1:96:7 cg:1:96:13 > gpurun_out/p1b_qb.jsonl 2> gpurun_out/p1b_qb.err
echo done
