#!/bin/bash
# ncu --set full of the 8 C2 cell-kernel launches (second round of tools/roofline_kernels.py)
# -> gpurun_out/prof_c2.ncu-rep; then (here) tools/summarize_roofline.py writes
# profiles/r02/ncu_dominant.json, which bench.py reads for roofline.traffic.
set -eu
mkdir -p gpurun_out
python tools/roofline_kernels.py > gpurun_out/roofline_order.txt 2> gpurun_out/roofline_plain.err
ncu --set full --clock-control none --import-source on -k regex:cell_ -s 8 -c 8 \
    -o gpurun_out/prof_c2 python tools/roofline_kernels.py > gpurun_out/roofline_ncu.log 2>&1
tail -2 gpurun_out/roofline_ncu.log
