set -x
timeout 900 python tools/bench_configs.py mgdg --n3 64 --tau-scale 4 --h-coarse 32,16,8 > gpurun_out/mg7_dg64.jsonl 2> gpurun_out/mg7_dg64.err; echo "rc=$?"
timeout 900 python tools/bench_configs.py mgdg --n3 32 --h-coarse 16,8,4 > gpurun_out/mg7_dg32.jsonl 2> gpurun_out/mg7_dg32.err; echo "rc=$?"
