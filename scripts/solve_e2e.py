"""Where the end-to-end time of the drop-in solve() goes (1024^2 fp32 x100)."""
import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_1302_0120_b200 as pm
from paper_1302_0120_b200 import solver as S
from paper_1302_0120_b200.patterns import make_problem
p, m = make_problem(1024, 50, 7)
spec = pm.GridSpec(1024, 1024)
c = pm.SlmConstraint(pm.RealGrid(spec, p), pm.SINGLE)
mc = pm.FourierConstraint(pm.RealGrid(spec, m), pm.SINGLE)
cfg = pm.SolveConfig(max_iters=100, precision=pm.SINGLE, record_every=100)
for _ in range(5): r = pm.solve(c, mc, cfg)
ts = []
for _ in range(20):
    t0 = time.perf_counter(); r = pm.solve(c, mc, cfg); ts.append((time.perf_counter() - t0) * 1e3); del r
r = pm.solve(c, mc, cfg)
print("pm.solve 1024^2 fp32 x100: median %.3f ms e2e, device %.3f ms" % (np.median(ts), r.timing.fft_ms))
def t(f, n=20):
    out = []
    for _ in range(n):
        t0 = time.perf_counter(); f(); out.append((time.perf_counter() - t0) * 1e3)
    return np.median(out)
print("host casts p, m to float32 (threaded, page-locked): %.3f ms" % t(lambda: (S._host_cast(p, np.float32), S._host_cast(m, np.float32))))
print("page-locked output allocations (phases, u*, v*):    %.3f ms" % t(lambda: (S._host_empty((1024, 1024), np.float64), S._host_empty((1024, 1024), np.complex64), S._host_empty((1024, 1024), np.complex64))))
import torch
a = torch.empty(8 << 20, dtype=torch.uint8, pin_memory=True); d = torch.empty(8 << 20, dtype=torch.uint8, device="cuda")
def h2d():
    d.copy_(a, non_blocking=True); torch.cuda.synchronize()
def d2h():
    a.copy_(d, non_blocking=True); torch.cuda.synchronize()
print("H2D 8 MB pinned: %.3f ms   D2H 8 MB pinned: %.3f ms" % (t(h2d), t(d2h)))
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for _ in range(10): pm.solve(c, mc, cfg)
pr.disable(); pstats.Stats(pr).sort_stats('tottime').print_stats(8)
from paper_1302_0120_b200 import _lib
lib = _lib.load()
orig = lib.pm_solve
T = []
def wrapped(*a):
    t0 = time.perf_counter(); r = orig(*a); T.append((time.perf_counter() - t0) * 1e3); return r
lib.pm_solve = wrapped
ts = []
for _ in range(20):
    t0 = time.perf_counter(); r = pm.solve(c, mc, cfg); ts.append((time.perf_counter() - t0) * 1e3); del r
print("solve() %.3f ms, of which the pm_solve C call %.3f ms" % (np.median(ts), np.median(T)))
lib.pm_solve = orig
gaps = np.full(100, np.nan); lits = np.full(100, np.nan); darks = np.full(100, np.nan)
gaps[0] = 1.0; lits[0] = 0.1; darks[0] = 0.1
print("_reference_error: %.3f ms" % t(lambda: S._reference_error(cfg, 0, gaps, lits, darks)))
