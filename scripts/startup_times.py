"""Where the persistent solve's fixed cost goes (1024^2 fp32 GS): %globaltimer
stamps at the kernel's start, after the first row phase (tables + initial
iterate + row 1), and at the end (after the final pair), warm and after a
256 MiB L2 flush.

    python scripts/startup_times.py [K]
"""
import sys
sys.path.insert(0, '/root/repo')
import numpy as np
import torch
import paper_1302_0120_b200 as pm
from paper_1302_0120_b200 import _lib
from paper_1302_0120_b200.patterns import make_problem

K = int(sys.argv[1]) if len(sys.argv) > 1 else 4
SPC = 256
n, tag = 1024, 'single'
prec = pm.Precision.from_tag(tag)
p, m = make_problem(n, 50, 7)
spec = pm.GridSpec(n, n)
c = pm.SlmConstraint(pm.RealGrid(spec, p), prec); mm = pm.FourierConstraint(pm.RealGrid(spec, m), prec)
cfg = pm.SolveConfig(max_iters=K, precision=prec, record_every=K, device=0)
buf = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
pm.solve(c, mm, cfg)
plan = pm.transform.get_plan(spec, prec)
for flush in (False, True, False, True):
    plan.lib.pm_debug_phase_stamps(plan.handle, 1, None, 0)
    if flush:
        buf.fill_(1.0); torch.cuda.synchronize()
    r = pm.solve(c, mm, cfg)
    st = np.zeros(1184 * SPC, dtype=np.uint64)
    plan.lib.pm_debug_phase_stamps(plan.handle, 0, st.ctypes.data_as(_lib.C.c_void_p), st.size)
    S = st.reshape(1184, SPC).astype(np.int64)
    S = S[: int((S[:, 0] > 0).sum())]
    S = (S - S[:, 0].min()) / 1e3
    last = 1 + 4 * K
    print(f"flush={flush}: solve {r.timing.fft_ms*1e3:.1f} us on device events; start spread {S[:,0].max():.2f} us; "
          f"first row phase done (tables, u0, z1, row 1) med {np.median(S[:,1]):.2f} max {S[:,1].max():.2f} us; "
          f"iterations 2..K {(S[:, last - 1].max() - S[:, 1].max()) / max(K - 1, 1):.2f} us each; "
          f"final pair {np.median(S[:, last] - S[:, last - 1]):.2f} (max end {S[:, last].max():.2f}) us", flush=True)
