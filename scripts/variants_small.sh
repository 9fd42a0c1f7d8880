for d in paper_1302_0120_b200/lib/variants/*/ default; do
  echo "== $d"
  if [ "$d" = default ]; then timeout 300 python scripts/sweep_perf.py ${CASES:-2,11,8,10,3,4} 2>&1 | grep -v "^lib"; else
  PM_LIB=$d/libphasemask_b200.so timeout 300 python scripts/sweep_perf.py ${CASES:-2,11,8,10,3,4} 2>&1 | grep -v "^lib"; fi
done
