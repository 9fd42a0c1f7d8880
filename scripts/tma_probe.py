import sys; sys.path.insert(0,'/root/repo')
import numpy as np, paper_1302_0120_b200 as pm
from paper_1302_0120_b200.patterns import make_problem
for n, tag in [(int(a.split(':')[0]), a.split(':')[1]) for a in sys.argv[1:]]:
    prec = pm.Precision.from_tag(tag); p, m = make_problem(n, 8, 7); spec = pm.GridSpec(n, n)
    try:
        r = pm.solve(pm.SlmConstraint(pm.RealGrid(spec, p), prec), pm.FourierConstraint(pm.RealGrid(spec, m), prec), pm.SolveConfig(max_iters=5, precision=prec))
        print("ok", n, tag, r.final.gap, flush=True)
    except Exception as e:
        print("ERR", n, tag, e, flush=True); break
