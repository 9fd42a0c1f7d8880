"""The paper's own benchmark: 25 GS iterations on an
800x600 SLM in fp32, including the upload of the target (OSP), on one B200.
Times the public batch API end to end (host arrays in, float64 mask out) and
the device solve alone."""
import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np
import torch
import paper_1302_0120_b200 as pm
from paper_1302_0120_b200.batch import solve_stack
from paper_1302_0120_b200.patterns import make_problem

p, m = make_problem(800, 50, 7, n_y=600)
cfg = pm.SolveConfig(max_iters=25, precision=pm.SINGLE, record_every=25)
pp = torch.from_numpy(p.astype(np.float32)).pin_memory().numpy()
mm = torch.from_numpy(m[None].astype(np.float32)).pin_memory().numpy()
out = torch.empty((1, 600, 800), dtype=torch.float64).pin_memory().numpy()
for _ in range(3):
    r = solve_stack(pp, mm, cfg, out_phases=out)
if '--once' in sys.argv:        # for ncu: warm-up solves only
    sys.exit(0)
e2e, dev = [], []
for _ in range(20):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = solve_stack(pp, mm, cfg, out_phases=out)
    e2e.append((time.perf_counter() - t0) * 1e3)
    dev.append(r.device_ms)
print(f"800x600 fp32, 25 GS iterations: e2e {np.median(e2e):.3f} ms (incl. target upload and mask download), "
      f"device {np.median(dev):.3f} ms; paper (Tesla C2070): 45 ms incl. 1 ms upload")
