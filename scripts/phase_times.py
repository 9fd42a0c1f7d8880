"""Per-phase, per-CTA timing of the persistent solve kernel (%globaltimer stamps)."""
import sys
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_1302_0120_b200 as pm
from paper_1302_0120_b200 import _lib
from paper_1302_0120_b200.patterns import make_problem
K = 20
SPC = 256
cases = [(1024, 'single'), (256, 'double'), (1024, 'double'), (4096, 'single')]
sel = [int(x) for x in sys.argv[1].split(',')] if len(sys.argv) > 1 else range(4)
for n, tag in [cases[i] for i in sel]:
    prec = pm.Precision.from_tag(tag)
    p, m = make_problem(n, 50, 7)
    spec = pm.GridSpec(n, n)
    c = pm.SlmConstraint(pm.RealGrid(spec, p), prec); mm = pm.FourierConstraint(pm.RealGrid(spec, m), prec)
    cfg = pm.SolveConfig(max_iters=K, precision=prec, record_every=K)
    pm.solve(c, mm, cfg)
    plan = pm.transform.get_plan(spec, prec)
    plan.lib.pm_debug_phase_stamps(plan.handle, 1, None, 0)
    r = pm.solve(c, mm, cfg)
    st = np.zeros(1184 * SPC, dtype=np.uint64)
    plan.lib.pm_debug_phase_stamps(plan.handle, 0, st.ctypes.data_as(_lib.C.c_void_p), st.size)
    S = st.reshape(1184, SPC).astype(np.int64)
    ncta = int((S[:, 0] > 0).sum())
    S = S[:ncta]
    t0 = S[:, 0].min()
    S = (S - t0) / 1e3
    npts = int((S[0] > -1e-9).sum())
    # points: 0 start, then per iter: 1 after row, 2 after bar, 3 after col, 4 after bar, ... last: end
    print(f"{tag} n={n}: ctas {ncta}, dev {r.timing.fft_ms:.3f} ms, start spread {S[:,0].max():.2f} us", flush=True)
    per = (S[:, 1 + 4 * (K - 1) + 3].max() - S[:, 1 + 4 * 1].min()) / (K - 2)
    print(f"   steady iteration {per:.2f} us", flush=True)
    for it in (1, K // 2):
        b = 1 + 4 * it
        row_end = S[:, b]; bar1 = S[:, b + 1]; col_end = S[:, b + 2]; bar2 = S[:, b + 3]
        prev = S[:, b - 1]
        print(f"   it{it+1}: row work min/med/max {np.min(row_end-prev):.2f}/{np.median(row_end-prev):.2f}/{np.max(row_end-prev):.2f}"
              f"  last-arrive {row_end.max()-prev.min():.2f} release {bar1.min()-row_end.max():.2f}..{bar1.max()-row_end.max():.2f}"
              f" | col work {np.min(col_end-bar1):.2f}/{np.median(col_end-bar1):.2f}/{np.max(col_end-bar1):.2f}"
              f"  release {bar2.min()-col_end.max():.2f}..{bar2.max()-col_end.max():.2f}", flush=True)
