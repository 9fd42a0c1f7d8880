"""The alternating-projections solver on the GPU — drop-in for the
reference's ``solve`` (src/solver.py:111-216).

``solve(c, m, cfg, provider=None, on_record=None, should_abort=None)`` keeps
the reference's signature, validation messages, record / early-stop / abort
semantics and result type. The iteration itself runs inside
libphasemask_b200 as two fused sweeps per iteration captured in one CUDA
graph (no host round trip per iteration). When ``on_record`` or
``should_abort`` is given, the solve is stepped one iteration at a time so
the callbacks see exactly the reference's sequence.

``SolveConfig`` gains three fields, all defaulting to the reference's
behaviour: ``algorithm`` ("gs"; "raar" is the relaxed variant of SURVEY.md
§8 a15), ``beta`` (RAAR relaxation) and ``device`` (CUDA device index).
"""

from __future__ import annotations

import math
import os
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .backends import BackendSelector, deterministic_sum
from .grid import (DOUBLE, FOURIER_PLANE, SLM_PLANE, Field, PhaseMask, Precision,
                   RealGrid)
from .metrics import ConvergenceRecord, ErrorTolerances
from .projections import FourierConstraint, SlmConstraint
from .transform import FftProvider, PlanMismatchError, get_plan

ALGORITHMS = {"gs": _lib.PM_ALGO_GS, "raar": _lib.PM_ALGO_RAAR}


class SolveDivergedError(RuntimeError):
    """Non-finite values appeared during the iteration (src/solver.py:27-32)."""

    def __init__(self, iteration: int):
        super().__init__(f"non-finite values at iteration {iteration}")
        self.iteration = iteration


def _default_device() -> int:
    from .transform import default_device
    return default_device()


@dataclass(frozen=True)
class SolveConfig:
    """Reference SolveConfig (src/solver.py:35-53) plus algorithm/beta/device."""

    max_iters: int = 25
    precision: Precision = DOUBLE
    record_every: int = 1
    early_stop_tol: float | None = None
    backend: BackendSelector = field(default_factory=BackendSelector)
    random_phase_init: bool = False
    seed: int = 0
    tolerances: ErrorTolerances = field(default_factory=ErrorTolerances)
    algorithm: str = "gs"
    beta: float = 0.9
    device: int | None = None

    def __post_init__(self):
        if self.max_iters < 1:
            raise ValueError("max_iters must be >= 1")
        if self.record_every < 1:
            raise ValueError("record_every must be >= 1")
        if self.early_stop_tol is not None and self.early_stop_tol < 0:
            raise ValueError("early_stop_tol must be nonnegative")
        if self.algorithm not in ALGORITHMS:
            raise ValueError(f"unknown algorithm {self.algorithm!r}")

    @property
    def device_index(self) -> int:
        return _default_device() if self.device is None else self.device


@dataclass(frozen=True)
class Timing:
    """Timing breakdown in ms (src/solver.py:55-68).

    The transforms and projections are fused into the same kernels, so
    ``fft_ms`` carries the fused device time of the whole iteration and
    ``constraint_ms`` / ``metrics_ms`` are 0 (metrics are computed inside
    the sweeps); ``iteration_ms`` is the device time per iteration.
    """

    total_ms: float
    fft_ms: float
    constraint_ms: float
    metrics_ms: float
    iteration_ms: float

    @property
    def per_iter_ms(self) -> float:
        return self.iteration_ms


@dataclass(frozen=True)
class SolveResult:
    mask: PhaseMask
    u_star: Field
    v_star: Field
    history: tuple[ConvergenceRecord, ...]
    iters_run: int
    timing: Timing
    aborted: bool = False

    @property
    def final(self) -> ConvergenceRecord:
        return self.history[-1]


def default_amplitude(m: RealGrid, precision: Precision = DOUBLE) -> RealGrid:
    """Uniform energy-matched p = ||m|| / sqrt(N) (src/solver.py:86-90)."""
    from .grid import norm2
    level = norm2(m.data.astype(np.complex128)) / math.sqrt(m.spec.n)
    return RealGrid(m.spec, np.full(m.spec.shape, level))


def _initial_fourier(m_data: np.ndarray, precision: Precision, random_phases: bool, seed: int,
                     device: int = 0):
    """Fourier-plane start m e^{i phi} for the seeded random branch
    (src/solver.py:100-103), drawn on the device with numpy's PCG64 stream."""
    if random_phases:
        return _lib.random_start(m_data, precision.complex_dtype, seed, device)
    return None


def initial_iterate(m: FourierConstraint, provider: FftProvider,
                    random_phases: bool = False, seed: int = 0) -> Field:
    """u0 = F^-1(m e^{i phi}), phi = 0 unless seeded random (src/solver.py:93-108)."""
    data = _initial_fourier(m.m.data, provider.precision, random_phases, seed,
                            getattr(provider, "device", 0))
    if data is None:
        data = m.m.data.astype(np.complex128).astype(provider.precision.complex_dtype)
    return provider.inverse(Field(m.m.spec, data, FOURIER_PLANE))


def _params(cfg: SolveConfig, p_per_mask: bool, init_complex: bool) -> _lib.pm_params:
    prm = _lib.pm_params()
    prm.algorithm = ALGORITHMS[cfg.algorithm]
    prm.beta = float(cfg.beta)
    prm.max_iters = int(cfg.max_iters)
    prm.record_every = int(cfg.record_every)
    prm.early_stop_tol = -1.0 if cfg.early_stop_tol is None else float(cfg.early_stop_tol)
    prm.t_lit = float(cfg.tolerances.t_lit)
    prm.t_dark = float(cfg.tolerances.t_dark)
    prm.p_per_mask = int(p_per_mask)
    prm.init_complex = int(init_complex)
    if cfg.random_phase_init and not init_complex:
        # phi drawn on the device from the seeded PCG64 stream (src/solver.py:100-103)
        prm.init_random = 1
        prm.rng[:] = [int(v) for v in _lib.pcg64_state(cfg.seed)]
    return prm


_PINNED_MIN, _PINNED_MAX = 1 << 20, 256 << 20


def _host_empty(shape, dtype) -> np.ndarray:
    """An array in page-locked memory (the library's own runtime: full-speed,
    asynchronous copies; the block is reused once the array is dropped) when it
    is between 1 MiB and 256 MiB, else a plain numpy array."""
    n = int(np.prod(shape)) * np.dtype(dtype).itemsize
    if _PINNED_MIN <= n <= _PINNED_MAX:
        try:
            return _lib.host_empty(shape, dtype)
        except (RuntimeError, MemoryError, ImportError):   # no device / no page-locked memory: pageable
            pass
    return np.empty(shape, dtype=dtype)


_CAST_POOL = None
_CAST_THREADED_MIN = 8 << 20


def _host_cast(a: np.ndarray, dtype) -> np.ndarray:
    """`a` as a C-contiguous `dtype` array; when a cast is needed anyway it is
    written into (large: page-locked) memory from _host_empty. Up to 8 MB on
    one thread: a cast spread over several cores leaves the data dirty in their
    caches, and the upload that follows then ran at ~8 GB/s instead of ~50
    (solve() at 1024^2 fp32: 3.9 -> 3.4 ms end to end); larger arrays, whose
    cast dominates, on 8 threads (numpy releases the GIL in the copy)."""
    global _CAST_POOL
    if a.dtype == np.dtype(dtype) and a.flags.c_contiguous:
        return a
    out = _host_empty(a.shape, dtype)
    if out.nbytes < _CAST_THREADED_MIN or a.ndim < 1 or a.shape[0] < 8:
        np.copyto(out, a, casting="unsafe")
        return out
    if _CAST_POOL is None:
        from concurrent.futures import ThreadPoolExecutor
        _CAST_POOL = ThreadPoolExecutor(max(1, min(8, os.cpu_count() or 1)), thread_name_prefix="pm-cast")
    k = _CAST_POOL._max_workers
    bounds = np.linspace(0, a.shape[0], k + 1).astype(int)
    list(_CAST_POOL.map(lambda i: np.copyto(out[bounds[i]:bounds[i + 1]], a[bounds[i]:bounds[i + 1]],
                                            casting="unsafe"), range(k)))
    return out


def _reference_error(cfg: SolveConfig, diverged: int, gaps, lits, darks) -> Exception | None:
    """The exception the reference's solve() raises for this outcome, in its
    order of events (None: it returns normally).

    ``diverged`` is the first iteration whose fields the device found
    non-finite (0: none), i.e. the iteration whose body would raise
    SolveDivergedError (src/solver.py:152-165). The reference evaluates the
    metrics of iteration it-1 before that body when it-1 is recorded or early
    stopping is on (:172-176), and their Field checks see the same non-finite
    transform first: ValueError("field contains non-finite entries") from
    metrics.gap (src/metrics.py:67-71, src/grid.py:108-109). A recorded
    reconstructed intensity that is not finite fails RealGrid's check
    (src/metrics.py:81-88, src/grid.py:128-129).
    """
    early = cfg.early_stop_tol is not None
    last = diverged if diverged else len(gaps)
    for it in range(1, last + 1):
        if it == diverged:
            return SolveDivergedError(it)
        rec = (it - 1) % cfg.record_every == 0
        if (rec or early) and diverged == it + 1 and cfg.algorithm == "gs":
            return ValueError("field contains non-finite entries")
        if rec and not (np.isfinite(lits[it - 1]) and np.isfinite(darks[it - 1])) and not np.isnan(gaps[it - 1]):
            return ValueError("grid contains non-finite entries")
    return None


def _history(it_ms, iters_run, gaps, lits, darks):
    out = []
    for i in range(1, iters_run + 1):
        g = gaps[i - 1]
        if np.isnan(g):
            continue
        out.append(ConvergenceRecord(iter=i, gap=float(g), err_lit=float(lits[i - 1]),
                                     err_dark=float(darks[i - 1]), time_fft_ms=it_ms,
                                     time_constraint_ms=0.0, time_total_ms=it_ms))
    return out


def solve(c: SlmConstraint, m: FourierConstraint, cfg: SolveConfig,
          provider: FftProvider | None = None,
          on_record=None, should_abort=None) -> SolveResult:
    """Alternating projections + best-approximation pair, on the GPU.

    on_record(record) fires for each recorded iteration; should_abort() is
    polled once per iteration for cooperative cancellation, as in the
    reference.

    The physical-error metrics use the target energy sum(m^2) and intensity
    m^2 of the precision-cast m, reduced on the device in a fixed order. The
    reference squares the float64 m (src/solver.py:135-136); in SINGLE
    precision the two differ by at most ~6e-8 relative (the float32 rounding
    of m), far inside the fp32 record tolerance; in DOUBLE they differ only by
    summation order.
    """
    spec = c.p.spec
    if m.m.spec != spec:
        raise ValueError("amplitude and target constraints live on different grids")
    if c.p.max_value == 0.0:            # O(1): the grids' maxima come from their validation
        raise ValueError("SLM amplitude is identically zero")
    if m.m.max_value == 0.0:
        raise ValueError("target pattern is identically zero (all dark)")
    if c.precision is not cfg.precision:
        c = SlmConstraint(c.p, cfg.precision)
    if m.precision is not cfg.precision:
        m = FourierConstraint(m.m, cfg.precision)
    device = cfg.device_index
    if provider is not None:
        if provider.spec != spec:
            raise PlanMismatchError(
                f"field spec {spec.n_x}x{spec.n_y} does not match plan "
                f"{provider.spec.n_x}x{provider.spec.n_y}")
        if cfg.device is None:
            # an explicit SolveConfig.device wins; else the provider's (itself the process default)
            device = getattr(provider, "device", device)

    prec = cfg.precision
    plan = get_plan(spec, prec, device)
    if on_record is not None or should_abort is not None:
        # callbacks run while the solve is in flight: a plan of their own, so a
        # callback may use transforms of this grid (the path setting follows slot 0)
        base, plan = plan, get_plan(spec, prec, device, slot=1)
        plan.set_path(base.path())
    fdt = prec.float_dtype
    p_dev = _host_cast(c.p.data, fdt)
    m_dev = _host_cast(m.m.data, fdt)
    # the zero tolerances 1024 eps max(.) of the precision-cast p and m
    # (src/projections.py:41-43) and the target energy sum(m^2) are reduced on
    # the device from the uploaded arrays, as the batch API does
    tol_p = tol_m = energy = None
    init = None                      # random-phase starts are drawn on the device
    prm = _params(cfg, False, False)

    K = cfg.max_iters
    N = spec.n
    phases = _host_empty(spec.shape, np.float64)
    u_star = _host_empty(spec.shape, prec.complex_dtype)
    v_star = _host_empty(spec.shape, prec.complex_dtype)
    gaps = np.full(K, np.nan)
    lits = np.full(K, np.nan)
    darks = np.full(K, np.nan)
    iters = np.zeros(1, dtype=np.int32)
    div = np.zeros(1, dtype=np.int32)
    dev_ms = np.zeros(1, dtype=np.float32)
    res = _lib.pm_result()
    res.phases, res.u_star, res.v_star = (_lib.ptr(phases), _lib.ptr(u_star), _lib.ptr(v_star))
    res.gap, res.err_lit, res.err_dark = _lib.ptr(gaps), _lib.ptr(lits), _lib.ptr(darks)
    res.iters_run, res.diverged_iter, res.device_ms = _lib.ptr(iters), _lib.ptr(div), _lib.ptr(dev_ms)
    res.levels = None

    aborted = False
    t0 = time.perf_counter()
    lib = plan.lib
    with plan.lock:
        if on_record is None and should_abort is None:
            code = lib.pm_solve(plan.handle, _lib.ptr(p_dev), _lib.ptr(m_dev), _lib.ptr(init), 1,
                                prm, _lib.ptr(tol_p), _lib.ptr(tol_m), _lib.ptr(energy), res)
        else:
            # one enqueued solve; the device streams every decided iteration into
            # a host-mapped ring and, when should_abort is given, waits after each
            # one for its verdict (src/solver.py:188-199) — no launch or copy per
            # iteration. The callbacks run here, in the caller's thread, in the
            # reference's order: on_record, then should_abort unless the
            # iteration stopped early.
            lockstep = should_abort is not None
            _lib.check(lib.pm_solve_async(plan.handle, _lib.ptr(p_dev), _lib.ptr(m_dev), _lib.ptr(init),
                                          prm, _lib.ptr(tol_p), _lib.ptr(tol_m), _lib.ptr(energy),
                                          int(lockstep), res), "pm_solve_async")
            rec = _lib.pm_record()
            failure = None
            # the iterations the device publishes: all of them when it waits for a
            # verdict or stops early, else the recorded ones and the last
            if lockstep or cfg.early_stop_tol is not None:
                published = range(1, K + 1)
            else:
                published = sorted(set(range(1, K + 1, cfg.record_every)) | {K})
            last = 0
            try:
                for it in published:
                    _lib.check(lib.pm_solve_next(plan.handle, it, _lib.C.byref(rec)), "pm_solve_next")
                    fl = rec.flags
                    if not fl or fl & _lib.PM_REC_DIVERGED:
                        break
                    last = it
                    if on_record is not None and fl & _lib.PM_REC_RECORDED:
                        on_record(ConvergenceRecord(iter=it, gap=float(rec.gap), err_lit=float(rec.err_lit),
                                                    err_dark=float(rec.err_dark)))
                    if fl & _lib.PM_REC_EARLY:
                        break
                    if lockstep:
                        stop = bool(should_abort())
                        _lib.check(lib.pm_solve_answer(plan.handle, it, int(stop)), "pm_solve_answer")
                        if stop:
                            aborted = True
                            break
                    elif fl & _lib.PM_REC_STOP:
                        break
                if lockstep and last and not aborted:
                    # a device left without a verdict for 30 s stopped at `last`
                    _lib.check(lib.pm_solve_next(plan.handle, last, _lib.C.byref(rec)), "pm_solve_next")
                    if rec.flags & _lib.PM_REC_TIMEOUT:
                        failure = RuntimeError(
                            f"no should_abort verdict reached the device within 30 s at iteration {last} "
                            "(a callback may not wait for GPU work on the solving device during a solve)")
            except BaseException as exc:            # a callback raised: stop the device, then re-raise
                failure = exc
                if lockstep:
                    lib.pm_solve_answer(plan.handle, 0, 1)
            code = lib.pm_solve_wait(plan.handle, res)
            if failure is not None:
                raise failure
    if code == _lib.PM_ERR_DIVERGED or div[0]:
        raise _reference_error(cfg, int(div[0]) or 1, gaps, lits, darks)
    # the library's messages are the reference's: zero inputs (checked before the
    # loop), then the loop's record checks, then a non-finite pair (after it)
    if code != _lib.PM_OK and "identically zero" in _lib.last_error():
        _lib.check(code)
    err = _reference_error(cfg, 0, gaps[:int(iters[0])], lits, darks)
    if err is not None:
        raise err
    _lib.check(code)
    total_ms = (time.perf_counter() - t0) * 1e3
    iters_run = int(iters[0])
    it_ms = float(dev_ms[0]) / max(iters_run, 1)
    history = _history(it_ms, iters_run, gaps, lits, darks)
    timing = Timing(total_ms=total_ms, fft_ms=float(dev_ms[0]), constraint_ms=0.0,
                    metrics_ms=0.0, iteration_ms=it_ms)
    # device outputs: the mask is in [0, 2pi) by construction and the pair was
    # checked finite on the device (the library fails with the reference's
    # ValueError otherwise), so no O(N) host validation pass
    return SolveResult(mask=PhaseMask._trusted(spec, phases), u_star=Field._trusted(spec, u_star, SLM_PLANE),
                       v_star=Field._trusted(spec, v_star, SLM_PLANE), history=tuple(history),
                       iters_run=iters_run, timing=timing, aborted=aborted)
