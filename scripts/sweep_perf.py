"""Per-variant timing: 1024^2 fp32 solve (K=100) device ms, per-sweep times, batch throughput."""
import os, sys, time
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_1302_0120_b200 as pm
from paper_1302_0120_b200 import _lib
from paper_1302_0120_b200.patterns import make_problem

def run(n, tag, K=100, batch=1):
    prec = pm.Precision.from_tag(tag)
    p, m = make_problem(n, 50 if n >= 128 else 4, 7)
    plan = pm.transform.get_plan(pm.GridSpec(n, n), prec)
    fdt = prec.float_dtype
    P = np.ascontiguousarray(p, fdt); M = np.ascontiguousarray(np.broadcast_to(m, (batch,) + m.shape), fdt)
    prm = _lib.pm_params(); prm.algorithm = 0; prm.beta = 0.9; prm.max_iters = K; prm.record_every = K
    prm.early_stop_tol = -1.0; prm.t_lit = 0.1; prm.t_dark = 3e-4; prm.p_per_mask = 0; prm.init_complex = 0
    tp = np.full(batch, prec.zero_tol(p.max())); tm = np.full(batch, prec.zero_tol(m.max())); en = np.full(batch, float((m**2).sum()))
    ph = np.empty((batch, n, n)); ms = np.zeros(1, np.float32)
    res = _lib.pm_result(); res.phases = _lib.ptr(ph); res.device_ms = _lib.ptr(ms)
    best = 1e9
    for i in range(4):
        _lib.check(plan.lib.pm_solve(plan.handle, _lib.ptr(P), _lib.ptr(M), None, batch, prm, _lib.ptr(tp), _lib.ptr(tm), _lib.ptr(en), res))
        if i: best = min(best, float(ms[0]))
    r0 = plan.time_sweep(0, batch, 50); r1 = plan.time_sweep(1, batch, 50)
    csz = 8 if tag == 'single' else 16; rsz = csz // 2
    by = n * n * batch * (2 * csz + rsz)
    print(f"  {tag} n={n} batch={batch}: solve {best:.3f} ms ({best/batch:.3f} ms/mask, {best*1e3/K/batch:.2f} us/iter/mask)  row {r0*1e3:.2f} us ({by/r0/1e6:.0f} GB/s)  col {r1*1e3:.2f} us ({by/r1/1e6:.0f} GB/s)")

print("lib", os.environ.get("PM_LIB", "default"))
cases = [(1024, 'single', 1), (1024, 'single', 8), (512, 'single', 1), (2048, 'single', 1), (4096, 'single', 1), (1024, 'double', 1), (256, 'double', 1), (512, 'double', 1), (256, 'single', 1), (16, 'single', 1)]
if len(sys.argv) > 1: cases = cases[:int(sys.argv[1])]
for n, tag, b in cases:
    try:
        run(n, tag, batch=b)
    except Exception as e:
        print("  ERR", n, tag, b, e)
