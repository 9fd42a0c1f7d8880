"""Minimal workload for ncu: the stand-alone row and column sweeps of a
1024^2 fp32 GS plan at batch B (default 8), a few launches each."""
import sys
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_1302_0120_b200 as pm
from paper_1302_0120_b200 import _lib
from paper_1302_0120_b200.patterns import make_problem

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 8
prec = pm.SINGLE
p, m = make_problem(n, 50, 7)
plan = pm.transform.get_plan(pm.GridSpec(n, n), prec)
plan.set_path(2)
M = np.ascontiguousarray(np.broadcast_to(m, (batch, n, n)), np.float32)
P = p.astype(np.float32)
prm = _lib.pm_params(); prm.algorithm = 0; prm.beta = 0.9; prm.max_iters = 2; prm.record_every = 1
prm.early_stop_tol = -1.0; prm.t_lit = 0.1; prm.t_dark = 3e-4; prm.p_per_mask = 0; prm.init_complex = 0
tp = np.full(batch, prec.zero_tol(p.max())); tm = np.full(batch, prec.zero_tol(m.max())); en = np.full(batch, float((m**2).sum()))
res = _lib.pm_result()
_lib.check(plan.lib.pm_solve(plan.handle, _lib.ptr(P), _lib.ptr(M), None, batch, prm, _lib.ptr(tp), _lib.ptr(tm), _lib.ptr(en), res))
print("row us", plan.time_sweep(0, batch, 3) * 1e3, "col us", plan.time_sweep(1, batch, 3) * 1e3)
