for o in desc asc; do TMF_E2E_ORDER=$o timeout 600 python bench.py --no-cpu > gpurun_out/bench_o$o.json 2>>gpurun_out/bench_e2e.err; done
echo done
