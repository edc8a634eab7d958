set -u
mkdir -p gpurun_out
timeout 900 python tools/exp_memset.py cg:1:48:r:auto:off cg:2:48:r:auto:auto cg:3:48:r:auto:auto cg:4:48:r:auto:auto > gpurun_out/exp_memset.jsonl 2> gpurun_out/exp_memset.err
cat gpurun_out/exp_memset.jsonl; tail -3 gpurun_out/exp_memset.err
timeout 900 python tools/loop_bench.py dg:3:64:r:auto:auto > gpurun_out/pair_dg3.jsonl 2>gpurun_out/pair_dg3.err; cat gpurun_out/pair_dg3.jsonl
