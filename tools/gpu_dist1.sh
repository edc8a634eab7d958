set -x
timeout 900 python bench.py --dist --steps 3 --warmup 3 --no-cpu > gpurun_out/d1_bench_dist.json 2> gpurun_out/d1_bench_dist.err; echo "rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29671 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu > gpurun_out/d1_bench_torchrun.json 2> gpurun_out/d1_bench_torchrun.err; echo "rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29672 tools/bench_scaling.py c5 > gpurun_out/d1_scale_c5.jsonl 2> gpurun_out/d1_scale_c5.err; echo "rc=$?"
