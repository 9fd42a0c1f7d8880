"""Per-phase timing of the persistent solve on a batch (TMA build): the
%globaltimer stamps of CTA phase boundaries, batch B of 1024^2 fp32."""
import sys
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_1302_0120_b200 as pm
from paper_1302_0120_b200 import _lib
from paper_1302_0120_b200.batch import solve_stack
from paper_1302_0120_b200.patterns import make_problem, spot_targets
B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
K = 6
n = 1024
p, _ = make_problem(n, 50, 1000)
ms = spot_targets(n, 50, range(1000, 1000 + B), dtype=np.float32)
cfg = pm.SolveConfig(max_iters=K, precision=pm.SINGLE, record_every=K)
solve_stack(p.astype(np.float32), ms, cfg)
plan = pm.transform.get_plan(pm.GridSpec(n, n), pm.SINGLE)
plan.lib.pm_debug_phase_stamps(plan.handle, 1, None, 0)
r = solve_stack(p.astype(np.float32), ms, cfg)
st = np.zeros(1184 * 256, dtype=np.uint64)
plan.lib.pm_debug_phase_stamps(plan.handle, 0, st.ctypes.data_as(_lib.C.c_void_p), st.size)
S = st.reshape(1184, 256)[:, :128].astype(np.int64)
ncta = int((S[:, 0] > 0).sum())
S = S[:ncta]
S = (S - S[:, 0].min()) / 1e3
print(f"batch {B}: {ncta} CTAs, device {r.device_ms:.3f} ms for K={K} ({r.device_ms / K / B * 1e3:.2f} us per mask-iteration)")
for it in (1, K // 2):
    b = 1 + 4 * it
    prev, row_end, bar1, col_end, bar2 = S[:, b - 1], S[:, b], S[:, b + 1], S[:, b + 2], S[:, b + 3]
    print(f"  it{it+1}: row phase {np.median(row_end - prev):.1f} us (max {np.max(row_end - prev):.1f}), "
          f"col phase {np.median(col_end - bar1):.1f} us (max {np.max(col_end - bar1):.1f}), "
          f"per mask: row {np.median(row_end - prev) / B:.2f} col {np.median(col_end - bar1) / B:.2f} us")
