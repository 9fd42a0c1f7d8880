"""Device and end-to-end time of a 1024^2 fp32 x100 solve with and without
host callbacks (record ring), record_every = 1."""
import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_1302_0120_b200 as pm
from paper_1302_0120_b200.patterns import make_problem
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
tag = sys.argv[2] if len(sys.argv) > 2 else "single"
prec = pm.Precision.from_tag(tag)
p, m = make_problem(n, 50, 7)
spec = pm.GridSpec(n, n)
c = pm.SlmConstraint(pm.RealGrid(spec, p), prec)
mm = pm.FourierConstraint(pm.RealGrid(spec, m), prec)
cfg = pm.SolveConfig(max_iters=100, precision=prec, record_every=1)
cases = {"plain": {}, "on_record": {"on_record": lambda r: None},
         "should_abort": {"should_abort": lambda: False},
         "both": {"on_record": lambda r: None, "should_abort": lambda: False}}
for name, kw in cases.items():
    for _ in range(2):
        pm.solve(c, mm, cfg, **kw)
    e2e, dev = [], []
    for _ in range(5):
        t = time.perf_counter()
        r = pm.solve(c, mm, cfg, **kw)
        e2e.append((time.perf_counter() - t) * 1e3)
        dev.append(r.timing.fft_ms)
    print(f"{tag} {n}^2 x100 record_every=1 {name:>13}: e2e median {np.median(e2e):7.2f} ms  device {np.median(dev):7.3f} ms")
