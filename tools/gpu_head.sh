#!/bin/bash
# HEAD verification on one B200: smoke, the whole GPU suite, both bench arms, the BASELINE configs
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/head_smoke.log 2>&1; echo "smoke rc=$?" | tee -a gpurun_out/head_smoke.log
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/head_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/head_tests.log; tail -4 gpurun_out/head_tests.log
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/head_bench_ref.json 2> gpurun_out/head_bench_ref.err; echo "ref rc=$?"
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/head_bench.json 2> gpurun_out/head_bench.err; echo "bench rc=$?"
cat gpurun_out/head_bench.json | cut -c1-3000
timeout 1500 python tools/bench_configs.py c1 c3 c4 c5 > gpurun_out/head_configs.jsonl 2> gpurun_out/head_configs.err; echo "configs rc=$?"
cat gpurun_out/head_configs.jsonl
