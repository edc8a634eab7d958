set -x
for t in 1 2 4; do
timeout 900 python tools/bench_configs.py mgdg --n3 64 --tau-scale $t > gpurun_out/mgdg_64_tau$t.jsonl 2> gpurun_out/mgdg_64_tau$t.err; echo "rc=$?"
done
