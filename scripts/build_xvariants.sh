#!/bin/bash
# Build library variants that differ by experiment macros into
# paper_1302_0120_b200/lib/variants/<name>/: build_xvariants.sh name:"-DA=1 -DB=2" ...
cd "$(dirname "$0")/.."
for v in "$@"; do
  name=${v%%:*}; defs=${v#*:}
  mkdir -p paper_1302_0120_b200/lib/variants/$name
  PM_XDEFS="$defs" python -m paper_1302_0120_b200.build --out paper_1302_0120_b200/lib/variants/$name/libphasemask_b200.so || exit 1
done
