"""Per-configuration device timing of the solve (BASELINE.json configs and
neighbours): ms per mask, us per iteration per mask, and the stand-alone
row / column sweep times of the same plan.

    python scripts/sweep_perf.py [n_cases | i,j,...]
"""
import os, sys
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_1302_0120_b200 as pm
from paper_1302_0120_b200 import _lib
from paper_1302_0120_b200.patterns import make_problem


def run(n, tag, batch=1, algo="gs", K=100, sweeps=True):
    prec = pm.Precision.from_tag(tag)
    p, m = make_problem(n, 50 if n >= 128 else 4, 7)
    plan = pm.transform.get_plan(pm.GridSpec(n, n), prec)
    fdt = prec.float_dtype
    P = np.ascontiguousarray(p, fdt); M = np.ascontiguousarray(np.broadcast_to(m, (batch,) + m.shape), fdt)
    prm = _lib.pm_params(); prm.algorithm = 0 if algo == "gs" else 1; prm.beta = 0.9; prm.max_iters = K
    prm.record_every = K; prm.early_stop_tol = -1.0; prm.t_lit = 0.1; prm.t_dark = 3e-4; prm.p_per_mask = 0
    prm.init_complex = 0
    tp = np.full(batch, prec.zero_tol(p.max())); tm = np.full(batch, prec.zero_tol(m.max())); en = np.full(batch, float((m**2).sum()))
    ph = np.empty((batch, n, n)); ms = np.zeros(1, np.float32)
    res = _lib.pm_result(); res.phases = _lib.ptr(ph); res.device_ms = _lib.ptr(ms)
    best = 1e9
    for i in range(4):
        _lib.check(plan.lib.pm_solve(plan.handle, _lib.ptr(P), _lib.ptr(M), None, batch, prm, _lib.ptr(tp), _lib.ptr(tm), _lib.ptr(en), res))
        if i: best = min(best, float(ms[0]))
    csz = 8 if tag == 'single' else 16; rsz = csz // 2
    per_it = (4 * csz + 2 * rsz + (4 * csz if algo == "raar" else 0)) * n * n   # algorithmic bytes / iteration
    line = (f"  {algo} {tag} n={n} batch={batch} K={K}: solve {best:.3f} ms ({best/batch:.3f} ms/mask, "
            f"{best*1e3/K/batch:.2f} us/iter/mask, {per_it*K*batch/best/1e6:.0f} GB/s algorithmic)")
    if sweeps and algo == "gs":
        r0 = plan.time_sweep(0, batch, 50); r1 = plan.time_sweep(1, batch, 50)
        by = n * n * batch * (2 * csz + rsz)
        line += f"  row {r0*1e3:.2f} us ({by/r0/1e6:.0f} GB/s)  col {r1*1e3:.2f} us ({by/r1/1e6:.0f} GB/s)"
    print(line, flush=True)


print("lib", os.environ.get("PM_LIB", "default"))
cases = [(1024, 'single', 1, 'gs', 100), (1024, 'single', 8, 'gs', 100), (256, 'double', 1, 'gs', 100),
         (512, 'single', 1, 'raar', 200), (512, 'double', 1, 'raar', 200), (1024, 'single', 32, 'gs', 100),
         (2048, 'single', 1, 'gs', 100), (4096, 'single', 1, 'gs', 100), (512, 'single', 1, 'gs', 100),
         (1024, 'double', 1, 'gs', 100), (512, 'double', 1, 'gs', 100), (256, 'single', 1, 'gs', 100),
         (16, 'single', 1, 'gs', 100)]
if len(sys.argv) > 1:   # n_cases, or a comma list of case indices
    a = sys.argv[1]
    cases = [cases[int(i)] for i in a.split(",") if i] if "," in a else cases[:int(a)]
for n, tag, b, algo, K in cases:
    try:
        run(n, tag, b, algo, K)
    except Exception as e:
        print("  ERR", n, tag, b, algo, e)
