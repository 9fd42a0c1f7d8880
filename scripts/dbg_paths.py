import os, sys
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_1302_0120_b200 as pm
from oracle import phasemask_oracle as orc
from paper_1302_0120_b200.patterns import make_problem
for n, tag in ((256, "single"), (256, "double")):
    p, m = make_problem(n, 8, 7)
    prec = pm.Precision.from_tag(tag)
    spec = pm.GridSpec(n, n)
    plan = pm.transform.get_plan(spec, prec)
    for K in (1, 2, 5):
        o = orc.solve(p, m, K, tag)
        for path in (0, 2):
            plan.set_path(path)
            try:
                r = pm.solve(pm.SlmConstraint(pm.RealGrid(spec, p), prec), pm.FourierConstraint(pm.RealGrid(spec, m), prec),
                             pm.SolveConfig(max_iters=K, precision=prec))
                print(os.environ.get("TAGX",""), n, tag, K, path, "u* err %.3e v* err %.3e" % (orc.relative_l2(r.u_star.data, o["u_star"]), orc.relative_l2(r.v_star.data, o["v_star"])),
                      "gap", r.history[0].gap, o["records"][0][1], flush=True)
            except Exception as e:
                print(n, tag, K, path, "EXC", e, flush=True)
        plan.set_path(0)
