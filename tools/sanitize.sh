#!/bin/bash
# compute-sanitizer memcheck and racecheck over the smallest golden of every kernel
# family (SURVEY §5 race-detection row): cell engines (modal / reference tensor /
# quadrature points incl. the cp.async ring at P4), face engines, the emulated peer
# (p2p) ranks, the multigrid transfers / V-cycle, the native PCG.  Logs -> gpurun_out/.
set -u
OUT=${OUT:-gpurun_out/sanitize}
mkdir -p "$OUT"
SEL_PARITY='test_gpu_matches_reference_golden and (cg_p1_n3_gm_dir2 or cg_p2_n8_gm or cg_p3_n3_gm_dir2 or cg_p4_n3_gm_dir or dg_p3_n3_gm_dir or helmk_p2_n3_gm_dir or helm3_p2_n2_gm_none)'
SEL_ENGINES='(test_gpu_cell_engines_match_golden or test_gpu_face_engines_match_golden) and (cg_p1_n3_gm_dir2 or cg_p4_n3_gm_dir or dg_p2_n3_gm_dir or helmk_p2_n3_gm_dir)'
TESTS=(
  "tests/test_gpu_parity.py -k \"$SEL_PARITY\""
  "tests/test_gpu_parity.py -k \"$SEL_ENGINES\""
  "tests/test_gpu_p2p.py -k emulated"
  "tests/test_gpu_multigrid.py -k \"test_transfers_match_oracle and 2-1 or test_vcycle_matches_oracle\""
  "tests/test_gpu_solvers.py -k \"test_native_pcg_matches_oracle or test_diagonal_matches_oracle\""
)
for tool in ${TOOLS:-memcheck racecheck}; do
  i=0
  for t in "${TESTS[@]}"; do
    i=$((i+1))
    log="$OUT/${tool}_$i.log"
    echo "== $tool $t" | tee "$log"
    eval timeout ${SAN_TIMEOUT:-900} /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 20 \
      ${SAN_EXTRA:-} python -m pytest -x -q -p no:cacheprovider $t >> "$log" 2>&1
    echo "rc=$?" | tee -a "$log"
    grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" "$log" | tail -3
  done
done
