"""Quick GPU diagnostic: transform accuracy per size, solve parity, timings."""
import sys, time, math
sys.path.insert(0, '/root/repo')
import numpy as np, scipy.fft as sfft
import paper_1302_0120_b200 as pm
from paper_1302_0120_b200 import _lib
from paper_1302_0120_b200.patterns import make_problem
from oracle import phasemask_oracle as orc

rng = np.random.default_rng(1)
print("devices", _lib.device_count())
for prec in (pm.SINGLE, pm.DOUBLE):
    for (nx, ny) in [(1,1),(2,2),(4,4),(8,8),(16,16),(32,32),(64,64),(128,128),(256,256),(512,512),(1024,1024),(2048,2048),(4096,4096),(8,256),(1024,16),(4096,2)]:
        x = (rng.standard_normal((ny,nx)) + 1j*rng.standard_normal((ny,nx))).astype(prec.complex_dtype)
        try:
            f = pm.FftProvider(pm.GridSpec(nx,ny), prec)
            y = f.forward(pm.Field(pm.GridSpec(nx,ny), x)).data
            z = f.inverse(pm.Field(pm.GridSpec(nx,ny), y, pm.grid.FOURIER_PLANE)).data
            ref = sfft.fft2(x.astype(np.complex128), norm="ortho")
            e1 = np.linalg.norm(y - ref)/np.linalg.norm(ref); e2 = np.linalg.norm(z - x)/np.linalg.norm(x)
            print(f"fft {prec.tag:6s} {nx}x{ny}: fwd rel {e1:.2e}  roundtrip {e2:.2e}")
        except Exception as e:
            print(f"fft {prec.tag} {nx}x{ny}: ERROR {type(e).__name__}: {e}")

for n, spots, K, tag in [(64, 8, 25, "double"), (256, 8, 100, "double"), (256, 8, 100, "single"), (1024, 50, 100, "single"), (1024, 50, 100, "double")]:
    p, m = make_problem(n, spots, 7)
    prec = pm.Precision.from_tag(tag)
    spec = pm.GridSpec(n, n)
    c = pm.SlmConstraint(pm.RealGrid(spec, p), prec); mm = pm.FourierConstraint(pm.RealGrid(spec, m), prec)
    try:
        t = time.time(); r = pm.solve(c, mm, pm.SolveConfig(max_iters=K, precision=prec)); tg = time.time()-t
        t = time.time(); r = pm.solve(c, mm, pm.SolveConfig(max_iters=K, precision=prec)); tg2 = time.time()-t
        o = orc.solve(p, m, K, tag)
        g = np.array([x.gap for x in r.history]); go = np.array([x[1] for x in o['records']])
        el = np.array([x.err_lit for x in r.history]); elo = np.array([x[2] for x in o['records']])
        print(f"solve {n} {tag} K={K}: u* rel {orc.relative_l2(r.u_star.data, o['u_star']):.2e} v* rel {orc.relative_l2(r.v_star.data, o['v_star']):.2e} "
              f"gap maxrel {np.max(np.abs(g-go)/go):.2e} errlit maxdiff {np.max(np.abs(el-elo)):.2e} mask wpe {orc.weighted_phase_error(r.mask.phases, o['mask'], p):.2e} "
              f"iters {r.iters_run} dev_ms {r.timing.fft_ms:.3f} wall {tg*1e3:.1f}/{tg2*1e3:.1f} ms  gap1 {g[0]:.12f} gapK {g[-1]:.12f}")
    except Exception as e:
        import traceback; traceback.print_exc()

plan = pm.transform.get_plan(pm.GridSpec(1024,1024), pm.SINGLE)
for which in (0,1):
    ms = plan.time_sweep(which, 1, 50)
    print("sweep", which, "ms", ms, "GB/s", 20*1024*1024/ms/1e6)
print("copy HBM GB/s", _lib.measure_copy(1<<30, 5), "L2 GB/s (32MB)", _lib.measure_copy(32<<20, 20), "(8MB)", _lib.measure_copy(8<<20, 20))
