set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
python tools/loop_bench.py cg:3:48 cgr:3:48 cgr:3:48:14 cgr:3:48:10 cgr:3:48:12 > gpurun_out/p3grp.jsonl 2>gpurun_out/p3grp.err
python tools/quick_bench.py dgr:3:64 dgr:3:64:10 dgr:3:64:14 cgr:1:48 > gpurun_out/p3grp_qb.jsonl 2>>gpurun_out/p3grp.err
echo done
