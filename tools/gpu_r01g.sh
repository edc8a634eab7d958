timeout 1800 python tools/bench_configs.py c1 c3 c4 c5 csr > gpurun_out/g_configs.jsonl 2> gpurun_out/g_configs.err; echo "configs rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29655 tools/bench_scaling.py c4 > gpurun_out/g_scale_c4.jsonl 2> gpurun_out/g_scale_c4.err; echo "scale c4 rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29656 tools/bench_scaling.py c5 > gpurun_out/g_scale_c5.jsonl 2> gpurun_out/g_scale_c5.err; echo "scale c5 rc=$?"
echo done
