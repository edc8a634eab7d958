timeout 600 python tools/quick_bench.py cg:4:48:0 cg:4:48:6 cgv:4:48:0 cgv:4:48:6 cgr:4:48:0 cgr:4:48:6 cg:4:64:0 cg:4:64:6 cgv:4:64:0 cgv:4:64:6 > gpurun_out/as2_qb.jsonl 2> gpurun_out/as2_qb.err
echo done
