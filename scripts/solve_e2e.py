import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_1302_0120_b200 as pm
from paper_1302_0120_b200.patterns import make_problem
p, m = make_problem(1024, 50, 7)
spec = pm.GridSpec(1024, 1024)
c = pm.SlmConstraint(pm.RealGrid(spec, p), pm.SINGLE)
mc = pm.FourierConstraint(pm.RealGrid(spec, m), pm.SINGLE)
cfg = pm.SolveConfig(max_iters=100, precision=pm.SINGLE, record_every=100)
for _ in range(3): r = pm.solve(c, mc, cfg)
ts = []
for _ in range(10):
    t0 = time.perf_counter(); r = pm.solve(c, mc, cfg); ts.append((time.perf_counter() - t0) * 1e3)
print("pm.solve 1024^2 fp32 x100: median %.3f ms e2e, device %.3f ms" % (np.median(ts), r.timing.fft_ms))
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for _ in range(5): pm.solve(c, mc, cfg)
pr.disable(); pstats.Stats(pr).sort_stats('cumulative').print_stats(12)
