for d in paper_1302_0120_b200/lib/variants/*/; do echo "== $d"; PM_LIB=$d/libphasemask_b200.so timeout 300 python -c "
import sys; sys.argv=['x']; sys.path.insert(0,'scripts')
exec(open('scripts/sweep_perf.py').read().split('print(\"lib\"')[0])
run(4096,'single',1,'gs',20); run(2048,'single',1,'gs',50)
"; done
