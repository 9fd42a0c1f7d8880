"""Minimal workload for ncu: a few 1024^2 fp32 GS solves through the C ABI."""
import sys
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_1302_0120_b200 as pm
from paper_1302_0120_b200.patterns import make_problem

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
tag = sys.argv[2] if len(sys.argv) > 2 else "single"
K = int(sys.argv[3]) if len(sys.argv) > 3 else 10
prec = pm.Precision.from_tag(tag)
p, m = make_problem(n, 50, 7)
spec = pm.GridSpec(n, n)
c = pm.SlmConstraint(pm.RealGrid(spec, p), prec)
mm = pm.FourierConstraint(pm.RealGrid(spec, m), prec)
for _ in range(3):
    r = pm.solve(c, mm, pm.SolveConfig(max_iters=K, precision=prec, record_every=K))
print("iters", r.iters_run, "dev ms", r.timing.fft_ms)
