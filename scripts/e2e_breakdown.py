"""Where the end-to-end time of one 1024^2 fp32 solve through the batch API goes."""
import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np
import torch
import paper_1302_0120_b200 as pm
from paper_1302_0120_b200.batch import solve_stack, _maxes
from paper_1302_0120_b200.patterns import make_problem

p, m = make_problem(1024, 50, 7)
cfg = pm.SolveConfig(max_iters=100, precision=pm.SINGLE, record_every=100)
pp = torch.from_numpy(p.astype(np.float32)).pin_memory().numpy()
mm = torch.from_numpy(m[None].astype(np.float32)).pin_memory().numpy()
out = torch.empty((1, 1024, 1024), dtype=torch.float64).pin_memory().numpy()
for _ in range(3):
    r = solve_stack(pp, mm, cfg, out_phases=out)

def t(f, n=20):
    ts = []
    for _ in range(n):
        torch.cuda.synchronize(); t0 = time.perf_counter(); f(); ts.append((time.perf_counter() - t0) * 1e3)
    return np.median(ts)

print("maxes p+m      %.3f ms" % t(lambda: (_maxes(pp, 1), _maxes(mm, 1))))
print("solve_stack    %.3f ms" % t(lambda: solve_stack(pp, mm, cfg, out_phases=out)))
r = solve_stack(pp, mm, cfg, out_phases=out)
print("device_ms      %.3f ms" % r.device_ms)
dp = torch.empty(1024 * 1024, dtype=torch.float32, device="cuda")
print("H2D 4 MB       %.3f ms" % t(lambda: dp.copy_(torch.from_numpy(pp.reshape(-1)), non_blocking=True)))
dq = torch.empty(1024 * 1024, dtype=torch.float64, device="cuda")
print("D2H 8 MB       %.3f ms" % t(lambda: torch.from_numpy(out.reshape(-1)).copy_(dq.cpu() if False else dq.to("cpu", non_blocking=False))))
