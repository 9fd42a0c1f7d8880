"""Intra-task clock64 breakdown of the persistent solve (library built with
-DPM_FINE=1; PM_LIB points at it). Prints, per stamp transition, the
median / max over CTAs of the SM cycles between consecutive stamps."""
import sys
sys.path.insert(0, '/root/repo')
import collections
import numpy as np
import paper_1302_0120_b200 as pm
from paper_1302_0120_b200 import _lib
from paper_1302_0120_b200.patterns import make_problem

NAMES = {1: "row-phase start", 2: "row-phase end", 3: "bar1 released", 4: "col-phase end", 5: "bar2 released",
         11: "row loads landed", 12: "row FFT1", 14: "row proj", 13: "row FFT2", 15: "row stores issued",
         21: "col loads landed", 22: "col FFT1", 24: "col metrics+proj", 23: "col FFT2", 25: "col stores issued"}
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
tag = sys.argv[2] if len(sys.argv) > 2 else "single"
K = 5
prec = pm.Precision.from_tag(tag)
p, m = make_problem(n, 50, 7)
spec = pm.GridSpec(n, n)
c = pm.SlmConstraint(pm.RealGrid(spec, p), prec)
mm = pm.FourierConstraint(pm.RealGrid(spec, m), prec)
cfg = pm.SolveConfig(max_iters=K, precision=prec, record_every=K)
pm.solve(c, mm, cfg)
plan = pm.transform.get_plan(spec, prec)
for rep in range(3):
    plan.lib.pm_debug_phase_stamps(plan.handle, 1, None, 0)
    r = pm.solve(c, mm, cfg)
st = np.zeros(148 * 1024, dtype=np.uint64)       # PM_FINE rows: 1024 slots per CTA, fine from 128
plan.lib.pm_debug_phase_stamps(plan.handle, 0, st.ctypes.data_as(_lib.C.c_void_p), st.size)
S = st.reshape(148, 1024)[:, 128:].astype(np.int64)
ncta = int((S[:, 1] > 0).sum())
trans = collections.defaultdict(list)
for cta in range(ncta):
    row = S[cta]
    ids, ts = row[0::2], row[1::2]
    k = int((ts > 0).sum())
    ids, ts = ids[:k], ts[:k]
    # skip the init phases: start at the second "row-phase start"
    starts = [i for i in range(k) if ids[i] == 1]
    if len(starts) < 3:
        continue
    for i in range(starts[1], k - 1):
        trans[(int(ids[i]), int(ids[i + 1]))].append(int(ts[i + 1] - ts[i]))
print(f"{tag} n={n}: {ncta} CTAs, {r.timing.fft_ms:.3f} ms for K={K}")
order = sorted(trans, key=lambda t: -len(trans[t]))
for t in order:
    v = np.array(trans[t])
    print(f"  {NAMES.get(t[0], t[0]):>20} -> {NAMES.get(t[1], t[1]):<20} n={len(v):4d}  "
          f"cycles med {np.median(v):7.0f}  p90 {np.percentile(v, 90):7.0f}  max {v.max():7.0f}"
          f"   ({np.median(v) / 1965:.2f} us med)")
