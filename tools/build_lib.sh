#!/usr/bin/env bash
# Build libstereo_b200.so for sm_100a (in-tree; travels to the GPU box) and the
# oracle's liboracle.so: the same steps as __graft_entry__.build().
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
cd "$ROOT" && python -c "import __graft_entry__ as g; g.build(force=${FORCE:-False})"
grep -E "error|warning" "$ROOT/paper_2212_00488_b200/lib/ptxas.log" | grep -v "Potential Performance Loss" || true
