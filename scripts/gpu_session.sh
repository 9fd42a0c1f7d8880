#!/bin/bash
# One gpurun call's worth of evidence: GPU tests, smoke, per-size timings,
# the bench line, the ncu launch list and one full ncu capture of the
# persistent solve kernel. Usage (from the repo root, under gpurun):
#   bash scripts/gpu_session.sh [tag] [what...]   what: tests smoke perf bench launches benchfull ref configs paper full
set -u
TAG=${1:-r01}
shift || true
WHAT=${*:-tests smoke perf bench launches full}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > "$OUT/nvsmi.txt" 2>&1
lscpu | grep -E "Model name|^CPU\(s\)|Thread|Socket" > "$OUT/lscpu.txt" 2>&1
for w in $WHAT; do
  case $w in
    tests)
      timeout 1500 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1; echo "pytest gpu rc=$?" ;;
    smoke)
      timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?" ;;
    perf)
      timeout 600 python scripts/sweep_perf.py > "$OUT/perf.log" 2>&1; echo "perf rc=$?" ;;
    bench)
      timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"; echo "bench rc=$?"; tail -c 3000 "$OUT/bench.json" ;;
    launches)
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file "$OUT/launches.csv" python bench.py --steps 3 --warmup 3 --no-cpu-baseline > "$OUT/launches.log" 2>&1
      echo "launches rc=$?" ;;
    benchfull)
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:solve_kernel -s 5 -c 1 \
        -o "$OUT/bench_solve" -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline > "$OUT/benchfull.log" 2>&1
      echo "benchfull rc=$?" ;;
    ref)
      timeout 900 python bench.py --impl reference > "$OUT/bench_reference.json" 2> "$OUT/bench_reference.err"
      echo "ref rc=$?"; tail -c 1500 "$OUT/bench_reference.json" ;;
    configs)
      for c in 1 2 4 5; do
        timeout 900 python bench.py --config $c > "$OUT/bench_config$c.json" 2> "$OUT/bench_config$c.err"
        echo "config $c rc=$?"; tail -c 400 "$OUT/bench_config$c.json"
      done ;;
    paper)
      timeout 300 python scripts/paper_config.py > "$OUT/paper.log" 2>&1; echo "paper rc=$?"; cat "$OUT/paper.log" ;;
    full)
      timeout 1200 ncu --set full --clock-control none --import-source on -k regex:solve_kernel -s 2 -c 1 \
        -o "$OUT/solve_full" -f python scripts/prof_solve.py 1024 single 100 > "$OUT/full.log" 2>&1
      echo "full rc=$?" ;;
  esac
done
