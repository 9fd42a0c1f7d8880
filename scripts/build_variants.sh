#!/bin/bash
# Build library variants (points-per-thread, persistent CTA size) into
# paper_1302_0120_b200/lib/variants/<name>/ for scripts/variants.sh.
cd "$(dirname "$0")/.."
for v in "$@"; do
  IFS=: read -r name lgr nt <<< "$v"
  mkdir -p paper_1302_0120_b200/lib/variants/$name
  PM_LGR=$lgr PM_SOLVE_NT=$nt python -m paper_1302_0120_b200.build --out paper_1302_0120_b200/lib/variants/$name/libphasemask_b200.so || exit 1
done
