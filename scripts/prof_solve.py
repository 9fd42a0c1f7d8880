"""Minimal workload for ncu: a few solves through the C ABI.

    python scripts/prof_solve.py [n] [single|double] [K] [batch] [gs|raar]
"""
import sys
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_1302_0120_b200 as pm
from paper_1302_0120_b200.batch import solve_stack
from paper_1302_0120_b200.patterns import make_problem

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
tag = sys.argv[2] if len(sys.argv) > 2 else "single"
K = int(sys.argv[3]) if len(sys.argv) > 3 else 10
B = int(sys.argv[4]) if len(sys.argv) > 4 else 1
algo = sys.argv[5] if len(sys.argv) > 5 else "gs"
prec = pm.Precision.from_tag(tag)
p, m = make_problem(n, 50 if n >= 128 else 4, 7)
cfg = pm.SolveConfig(max_iters=K, precision=prec, record_every=K, algorithm=algo)
if B == 1:
    spec = pm.GridSpec(n, n)
    c = pm.SlmConstraint(pm.RealGrid(spec, p), prec)
    mm = pm.FourierConstraint(pm.RealGrid(spec, m), prec)
    for _ in range(3):
        r = pm.solve(c, mm, cfg)
    print("iters", r.iters_run, "dev ms", r.timing.fft_ms)
else:
    ms = np.ascontiguousarray(np.broadcast_to(m, (B, n, n)), prec.float_dtype)
    for _ in range(3):
        r = solve_stack(p.astype(prec.float_dtype), ms, cfg)
    print("batch", B, "dev ms", r.device_ms)
