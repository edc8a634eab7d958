#!/bin/bash
# ncu --set full of the interior face kernels at HEAD: C3 (DG P3 64^3) and kappa-Helmholtz P2 64^3
set -u
mkdir -p gpurun_out
for spec in dg:3:64:r:auto:auto helmk:2:64:r:auto:auto; do
  tag=$(echo $spec | cut -d: -f1-2 | tr : _)
  python tools/prof_apply.py $spec 3 > gpurun_out/ncu_face_${tag}_plain.log 2>&1 || { echo "plain run failed"; tail -3 gpurun_out/ncu_face_${tag}_plain.log; continue; }
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:face_a -s 4 -c 1 \
      -o gpurun_out/ncu_face_${tag} -f python tools/prof_apply.py $spec 3 > gpurun_out/ncu_face_${tag}.log 2>&1
  tail -2 gpurun_out/ncu_face_${tag}.log
done
ls -la gpurun_out/*.ncu-rep
