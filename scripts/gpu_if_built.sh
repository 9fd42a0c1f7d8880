#!/bin/bash
# Build the library (and optional variants: "name:XONLY:XDEFS" ...); stop on any failure.
# Usage: scripts/gpu_if_built.sh [variant ...]
cd "$(dirname "$0")/.."
python -m paper_1302_0120_b200.build > /tmp/build_main.log 2>&1 || { echo "BUILD FAILED (main)"; grep -m5 error /tmp/build_main.log; exit 1; }
for v in "$@"; do
  name=${v%%:*}; rest=${v#*:}; only=${rest%%:*}; defs=${rest#*:}
  PM_XONLY=$only PM_XDEFS="$defs" python -m paper_1302_0120_b200.build --out paper_1302_0120_b200/lib/variants/$name/libphasemask_b200.so > /tmp/build_$name.log 2>&1 || { echo "BUILD FAILED ($name)"; grep -m5 error /tmp/build_$name.log; exit 1; }
done
echo "built"
