#!/bin/bash
# Persistent-kernel phase timing and per-size solve timing for every built
# library variant (scripts/build_variants.sh). Usage: variants.sh [phase cases] [perf cases]
cd "$(dirname "$0")/.."
for d in paper_1302_0120_b200/lib/variants/*/; do
  echo "== $d"
  PM_LIB=$d/libphasemask_b200.so timeout 120 python scripts/phase_times.py ${1:-0,3} 2>&1 | grep -v "^   it[0-9]"
  PM_LIB=$d/libphasemask_b200.so timeout 300 python scripts/sweep_perf.py ${2:-2} 2>&1
done
