#!/bin/bash
# End-of-session check on one B200: smoke, the GPU suite, both bench arms, BASELINE configs,
# ncu launch list of the bench, ncu --set full of the C2 cell kernels and of the face kernels.
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?" | tee -a gpurun_out/final_smoke.log
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/final_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/final_tests.log; tail -4 gpurun_out/final_tests.log
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err; echo "ref rc=$?"
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "bench rc=$?"
cut -c1-400 gpurun_out/final_bench.json
timeout 1500 python tools/bench_configs.py c1 c3 c4 c5 > gpurun_out/final_configs.jsonl 2> gpurun_out/final_configs.err; echo "configs rc=$?"
cat gpurun_out/final_configs.jsonl
# launch list of the bench command (kernel shares of the step)
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/final_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-quadrature --c4-n 0 > gpurun_out/final_launches.log 2>&1; echo "launch list rc=$?"
bash tools/capture_roofline.sh; echo "roofline capture rc=$?"
for spec in dg:3:64:r:auto:auto helmk:2:64:r:auto:auto; do
  tag=$(echo $spec | cut -d: -f1-2 | tr : _)
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:face_a -s 4 -c 1 \
      -o gpurun_out/ncu_face_${tag} -f python tools/prof_apply.py $spec 3 > gpurun_out/ncu_face_${tag}.log 2>&1
  tail -1 gpurun_out/ncu_face_${tag}.log
done
