set -x
H=64-32-16-8
timeout 1500 python tools/mg_sweep.py 128 321:2:50:mixed:csr:$H 321:3:50:mixed:csr:$H 321:2:20:mixed:csr:$H 321:4:50:mixed:csr:$H 31:3:50:mixed:csr:$H 321:3:50:f64::$H > gpurun_out/mg8_sweep.jsonl 2> gpurun_out/mg8_sweep.err; echo "rc=$?"
