"""How the L2 state before a step changes the headline solve's device time
(1024^2 fp32 GS x100): no flush, a 256 MiB write (dirty lines left in L2), a
256 MiB read (clean lines), and a write followed by a read.

    python scripts/flush_effect.py
"""
import sys
sys.path.insert(0, '/root/repo')
import numpy as np
import torch
import paper_1302_0120_b200 as pm
from paper_1302_0120_b200 import _lib
from paper_1302_0120_b200.patterns import make_problem
from paper_1302_0120_b200.solver import _params

n = 1024
K = int(sys.argv[1]) if len(sys.argv) > 1 else 100
prec = pm.SINGLE
p, m = make_problem(n, 50, 7)
plan = pm.transform.get_plan(pm.GridSpec(n, n), prec, 0)
stream = torch.cuda.Stream()
plan.set_stream(stream.cuda_stream)
d_p = torch.from_numpy(p.astype(np.float32)).cuda()
d_m = torch.from_numpy(m.astype(np.float32)).cuda()
d_phase = torch.empty((n, n), dtype=torch.float64, device="cuda")
buf = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
tol_p = np.array([prec.zero_tol(p.max())]); tol_m = np.array([prec.zero_tol(m.max())])
energy = np.array([float((m ** 2).sum())])
prm = _params(pm.SolveConfig(max_iters=K, precision=prec, record_every=K, device=0), False, False)
gaps = np.full(K, np.nan); iters = np.zeros(1, np.int32); dms = np.zeros(1, np.float32)


def solve():
    res = _lib.pm_result()
    res.phases = _lib.C.c_void_p(d_phase.data_ptr()); res.gap = _lib.ptr(gaps); res.iters_run = _lib.ptr(iters)
    res.device_ms = _lib.ptr(dms)
    _lib.check(plan.lib.pm_solve_device(plan.handle, _lib.C.c_void_p(d_p.data_ptr()), _lib.C.c_void_p(d_m.data_ptr()),
                                        None, 1, prm, _lib.ptr(tol_p), _lib.ptr(tol_m), _lib.ptr(energy), res), "solve")


plan2 = pm.transform.get_plan(pm.GridSpec(n, n), prec, 0, slot=1)
plan2.set_stream(stream.cuda_stream)
prm1 = _params(pm.SolveConfig(max_iters=1, precision=prec, record_every=1, device=0), False, False)
d_p2 = d_p.clone(); d_m2 = d_m.clone()


def solve_other():      # the same kernel on another plan's buffers: warms the code, not this plan's data
    res = _lib.pm_result()
    _lib.check(plan2.lib.pm_solve_device(plan2.handle, _lib.C.c_void_p(d_p2.data_ptr()), _lib.C.c_void_p(d_m2.data_ptr()),
                                         None, 1, prm1, _lib.ptr(tol_p), _lib.ptr(tol_m), _lib.ptr(energy), res), "solve2")


modes = {
    "read+code": lambda: (buf.sum(), solve_other()),
    "read+inputs": lambda: (buf.sum(), d_p.sum(), d_m.sum()),
    "none": lambda: None,
    "write": lambda: buf.fill_(1.0),
    "read": lambda: buf.sum(),
    "write+read": lambda: (buf.fill_(1.0), buf.sum()),
    "write 64MiB": lambda: buf[: 16 * 1024 * 1024].fill_(1.0),
    "read 16MiB": lambda: buf[: 4 * 1024 * 1024].sum(),
}
only = sys.argv[2].split(",") if len(sys.argv) > 2 else None
for name, fl in modes.items():
    if only and name not in only:
        continue
    ts, ks = [], []
    for i in range(13):
        with torch.cuda.stream(stream):
            fl()
            torch.cuda._sleep(600000)
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        solve()
        with torch.cuda.stream(stream):
            e1.record(stream)
        e1.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1)); ks.append(float(dms[0]))
    print(f"K={K} {name:12s} step {np.median(ts):.4f} ms (min {min(ts):.4f})  solve launches {np.median(ks):.4f} ms", flush=True)
