"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
every kernel family once — stand-alone transforms, projections, the sweep
path, the persistent GS and RAAR kernels, the mixed-radix path (register
composite radices), batches, the transposed-m column staging (2048^2),
device random-phase starts and the reconstruction image."""
import sys
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_1302_0120_b200 as pm
from paper_1302_0120_b200.batch import solve_stack
from paper_1302_0120_b200.patterns import make_problem
from paper_1302_0120_b200.metrics import reconstruction_log_image
from paper_1302_0120_b200.projections import project_fourier


def run(nx, ny, tag, algo="gs", K=3, path=0, batch=1, rand=False):
    prec = pm.Precision.from_tag(tag)
    p, m = make_problem(nx, 4 if nx < 128 else 8, 7, n_y=ny)
    spec = pm.GridSpec(nx, ny)
    plan = pm.transform.get_plan(spec, prec)
    plan.set_path(path)
    cfg = pm.SolveConfig(max_iters=K, precision=prec, algorithm=algo, record_every=1,
                         random_phase_init=rand, seed=3)
    if batch == 1:
        r = pm.solve(pm.SlmConstraint(pm.RealGrid(spec, p), prec), pm.FourierConstraint(pm.RealGrid(spec, m), prec), cfg)
        seen = []
        pm.solve(pm.SlmConstraint(pm.RealGrid(spec, p), prec), pm.FourierConstraint(pm.RealGrid(spec, m), prec), cfg,
                 on_record=seen.append)                        # record ring
        polls = []
        pm.solve(pm.SlmConstraint(pm.RealGrid(spec, p), prec), pm.FourierConstraint(pm.RealGrid(spec, m), prec), cfg,
                 on_record=seen.append, should_abort=lambda: polls.append(1) and False)   # lockstep verdicts
        u = pm.Field(spec, r.u_star.data)
        project_fourier(u, pm.FourierConstraint(pm.RealGrid(spec, m), prec), pm.FftProvider(spec, prec))
        reconstruction_log_image(u, pm.FftProvider(spec, prec), float((m ** 2).sum()))
    else:
        ms = np.stack([make_problem(nx, 4, s, n_y=ny)[1] for s in range(batch)])
        solve_stack(p.astype(prec.float_dtype), ms.astype(prec.float_dtype), cfg, levels=True)
    plan.set_path(0)
    print("ok", nx, ny, tag, algo, path, batch, flush=True)


run(64, 64, "double")
run(64, 32, "single")
run(128, 128, "single", path=1)
run(128, 128, "double", path=2)
run(128, 128, "single", algo="raar", path=1)
run(64, 64, "double", algo="raar")
run(128, 128, "single", batch=3)
run(60, 42, "double")
run(30, 40, "single", batch=2)
run(256, 256, "single", batch=24, K=2)            # TMA build (column tiles via cp.async.bulk.tensor)
run(512, 512, "single", algo="raar", batch=5, K=2)
run(60, 42, "double", algo="raar", K=4)          # mixed-radix RAAR (alternating iterate buffers)
run(800, 600, "single", K=2, rand=True)            # mixed radix 16 x 10 x 5 / 12 x 10 x 5, device random start
run(2048, 2048, "single", K=1)                     # persistent column phase staging m from its transposed copy
run(4096, 4096, "single", K=1)                     # TMA build: compact shared twiddles, one-box tiles, tensor stores
run(2048, 2048, "single", algo="raar", K=2)        # TMA build, RAAR (z' stores from the w' input tiles)
