set -x
timeout 600 python tools/check_face_variants.py > gpurun_out/mb_check.jsonl 2> gpurun_out/mb_check.err; echo "rc=$?"
timeout 1200 python tools/quick_bench.py hhv:2:96:0 hhv:2:96:176 hhv:2:96:192 dgv:3:64:0 dgv:3:64:176 dgv:3:64:192 dgv:2:96:0 dgv:2:96:176 dgv:2:96:192 > gpurun_out/mb_times.jsonl 2> gpurun_out/mb_times.err; echo "rc=$?"
