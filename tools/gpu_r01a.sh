set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
python bench.py > gpurun_out/bench_r01a.json 2> gpurun_out/bench_r01a.err; echo "bench rc=$?"
python tools/quick_bench.py cg:4:48 > gpurun_out/qb_cg4.log 2>&1 && \
ncu -f --set full --clock-control none --import-source on -k regex:cell_apply_kernel -s 2 -c 1 -o gpurun_out/prof_cg4 python tools/quick_bench.py cg:4:48 > gpurun_out/ncu_cg4.log 2>&1
echo "ncu rc=$?"
