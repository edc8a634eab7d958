set -x
timeout 900 python tools/quick_bench.py cgv:3:48:0 cgv:3:48:9 cgv:2:48:0 cgv:2:48:9 cgv:4:48:0 cgv:4:48:9 dgv:3:64:0 dgv:3:64:9 cgv:3:128:0 cgv:3:128:9 > gpurun_out/occ.jsonl 2> gpurun_out/occ.err; echo "rc=$?"
