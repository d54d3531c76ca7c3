#!/usr/bin/env bash
# compute-sanitizer on the GPU box: memcheck / synccheck /
# initcheck on the product library, racecheck on the sanitizer variant
# (lib/racecheck: -DSTEREO_RACECHECK, the x-pass ring refills ordered by CTA
# barriers; identical results, tests/test_gpu_parity.py::test_racecheck_variant_bit_exact).
# Usage: tools/sanitize.sh OUT.txt
set -uo pipefail
OUT="${1:-gpurun_out/sanitizers.txt}"
CS=compute-sanitizer
RC_LIB="$(pwd)/paper_2212_00488_b200/lib/racecheck/libstereo_b200.so"
{
  echo "# compute-sanitizer, $(date -u +%FT%TZ), $(nvidia-smi --query-gpu=name --format=csv,noheader | head -1)"
  for tool in memcheck synccheck initcheck; do
    echo "=== $tool (product library; c1, c2, 131x77 K=2, 2880x64 K=2 wide rows)"
    $CS --tool $tool python tools/sanitize_run.py c1 c2 odd wide 2>&1 | grep -E "ok|ERROR SUMMARY|Error" | head -20
  done
  echo "=== racecheck (sanitizer variant lib/racecheck; c1, c2, 131x77 K=2, 2880x64 K=2)"
  STEREO_B200_LIB="$RC_LIB" $CS --tool racecheck --racecheck-report all python tools/sanitize_run.py c1 c2 odd wide 2>&1 \
    | grep -E "ok|RACECHECK SUMMARY|ERROR SUMMARY|hazard|Race" | head -30
  echo "=== racecheck (product library, c1: the mbarrier-ordered refill, for reference)"
  $CS --tool racecheck python tools/sanitize_run.py c1 2>&1 | grep -E "ok|RACECHECK SUMMARY|ERROR SUMMARY|hazards\]" | head -8
  echo "=== memcheck c3 and band handles"
  $CS --tool memcheck python tools/sanitize_run.py c3 band 2>&1 | grep -E "ok|ERROR SUMMARY" | head
} > "$OUT" 2>&1
cat "$OUT"
