"""phasemask/gpu.py — the binding a `phasemask` maintainer would add to route
the reference's solve() (src/solver.py:111-216) to libphasemask_b200 through
its C ABI (include/phasemask_b200.h). Self-contained: ctypes + numpy + the
reference's own types; it is the documented stub of INTEGRATION.md, kept as a
real file so tests/test_integration_stub.py can check its structure layouts
against the header and against paper_1302_0120_b200/_lib.py.

    from phasemask import gpu
    r = gpu.solve_gpu(c, m, cfg)          # same (c, m, cfg) triple as solve()

The full-featured form (callbacks, batches, streams, plan cache, random-phase
starts) is paper_1302_0120_b200/solver.py + _lib.py in this repository.
"""

import ctypes as C
import os

import numpy as np

try:                                       # inside the reference package
    from .grid import SLM_PLANE, Field, PhaseMask
    from .metrics import ConvergenceRecord
    from .solver import SolveDivergedError, SolveResult
except ImportError:                        # stand-alone (layout checks)
    Field = PhaseMask = ConvergenceRecord = SolveResult = SLM_PLANE = None

    class SolveDivergedError(RuntimeError):
        def __init__(self, iteration):
            super().__init__(f"non-finite values at iteration {iteration}")
            self.iteration = iteration

PM_ERR_DIVERGED = -5


class pm_params(C.Structure):              # include/phasemask_b200.h: typedef struct pm_params
    _fields_ = [("algorithm", C.c_int), ("beta", C.c_double), ("max_iters", C.c_int),
                ("record_every", C.c_int), ("early_stop_tol", C.c_double), ("t_lit", C.c_double),
                ("t_dark", C.c_double), ("p_per_mask", C.c_int), ("init_complex", C.c_int),
                ("init_random", C.c_int), ("rng", C.c_ulonglong * 4)]


class pm_result(C.Structure):              # include/phasemask_b200.h: typedef struct pm_result
    _fields_ = [(n, C.c_void_p) for n in ("phases", "levels", "u_star", "v_star", "gap", "err_lit",
                                          "err_dark", "iters_run", "diverged_iter", "device_ms")]


def load(path=None):
    lib = C.CDLL(path or os.environ.get("PHASEMASK_B200_LIB", "libphasemask_b200.so"))
    lib.pm_plan_create.argtypes = [C.c_int] * 5 + [C.POINTER(C.c_void_p)]
    lib.pm_solve.argtypes = ([C.c_void_p] * 4 + [C.c_int, C.POINTER(pm_params)] + [C.c_void_p] * 3
                             + [C.POINTER(pm_result)])
    lib.pm_last_error.restype = C.c_char_p
    return lib


_lib = None
_plans = {}                                 # PlanCache analogue (src/service.py:65-82)


def solve_gpu(c, m, cfg, device=0):
    global _lib
    _lib = _lib or load()
    spec, prec = c.p.spec, cfg.precision
    key = (spec.n_x, spec.n_y, prec.tag, device)
    if key not in _plans:
        h = C.c_void_p()
        if _lib.pm_plan_create(device, spec.n_x, spec.n_y, int(prec.tag == "double"), 1, C.byref(h)):
            raise RuntimeError(_lib.pm_last_error().decode())
        _plans[key] = h
    f = prec.float_dtype
    p = np.ascontiguousarray(c.p.data, f)
    mm = np.ascontiguousarray(m.m.data, f)
    K = cfg.max_iters
    out = dict(phases=np.empty(spec.shape), u_star=np.empty(spec.shape, prec.complex_dtype),
               v_star=np.empty(spec.shape, prec.complex_dtype), gap=np.full(K, np.nan),
               err_lit=np.full(K, np.nan), err_dark=np.full(K, np.nan),
               iters_run=np.zeros(1, np.int32), diverged_iter=np.zeros(1, np.int32))
    res = pm_result(**{k: v.ctypes.data for k, v in out.items()})
    prm = pm_params(algorithm=0, beta=0.9, max_iters=K, record_every=cfg.record_every,
                    early_stop_tol=-1.0 if cfg.early_stop_tol is None else cfg.early_stop_tol,
                    t_lit=cfg.tolerances.t_lit, t_dark=cfg.tolerances.t_dark, p_per_mask=0,
                    init_complex=0, init_random=0)          # rng stays zero: no random start
    # zero tolerances and sum(m^2) of the caller's arrays, as solve() computes them (:127-136)
    tp, tm = np.array([c.zero_tol]), np.array([m.zero_tol])
    e = np.array([float((m.m.data.astype(np.float64) ** 2).sum())])
    code = _lib.pm_solve(_plans[key], p.ctypes.data, mm.ctypes.data, None, 1, C.byref(prm),
                         tp.ctypes.data, tm.ctypes.data, e.ctypes.data, C.byref(res))
    if code == PM_ERR_DIVERGED:
        raise SolveDivergedError(int(out["diverged_iter"][0]))
    if code:
        raise RuntimeError(_lib.pm_last_error().decode())
    n = int(out["iters_run"][0])
    hist = tuple(ConvergenceRecord(i + 1, out["gap"][i], out["err_lit"][i], out["err_dark"][i])
                 for i in range(n) if not np.isnan(out["gap"][i]))
    return SolveResult(PhaseMask(spec, out["phases"]), Field(spec, out["u_star"], SLM_PLANE),
                       Field(spec, out["v_star"], SLM_PLANE), hist, n, None)
