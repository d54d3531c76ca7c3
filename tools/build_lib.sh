#!/usr/bin/env bash
# Build libstereo_b200.so for sm_100a (in-tree; travels to the GPU box).
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC="$ROOT/paper_2212_00488_b200/csrc"
OUT="$ROOT/paper_2212_00488_b200/lib"
mkdir -p "$OUT"
NVCC="${NVCC:-nvcc}"
"$NVCC" -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo \
  -Xcompiler -fPIC,-ffp-contract=off,-fno-fast-math -Xptxas -v \
  --shared -o "$OUT/libstereo_b200.so.tmp" \
  "$SRC/stereo_kernels.cu" "$SRC/stereo_abi.cu" -lcudart "$@" 2> "$OUT/ptxas.log" || { cat "$OUT/ptxas.log"; exit 1; }
mv "$OUT/libstereo_b200.so.tmp" "$OUT/libstereo_b200.so"
grep -E "error|warning" "$OUT/ptxas.log" | grep -v "Potential Performance Loss" || true
