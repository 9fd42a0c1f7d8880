#!/bin/bash
# Persistent-kernel phase timing for every built library variant.
cd "$(dirname "$0")/.."
for d in paper_1302_0120_b200/lib/variants/*/; do
  echo "== $d"
  PM_LIB=$d/libphasemask_b200.so timeout 120 python scripts/phase_times.py ${1:-0,3} 2>&1 | grep -v "^ *it"
done
