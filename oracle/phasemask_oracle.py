"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A numpy/scipy restatement of the reference's phase-retrieval hot path
(``/root/reference/pkg/src/phasemask``; abbreviated ``src/`` below). It is the
checker the GPU path is compared against and the CPU baseline that
``bench.py`` times. Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s cpu_baseline / ``--impl reference`` legs may import it; the
product package never does.

Parity status: PINNED. ``tests/test_oracle_golden.py`` checks every function
here bitwise against golden vectors produced by importing the reference
itself in the build container (``tests/golden/make_golden.py``) and against
the reference's own known-answer tests.

The FFT is third-party in the reference: ``scipy.fft.fft2/ifft2(norm="ortho")``
(scipy 1.18.1 here, DUCC0 backend; reference pins only ``scipy>=1.10`` in
``pkg/pyproject.toml:12``). The oracle calls the same scipy entry points, so
its results are the reference's results on the same machine.

RAAR has no reference implementation (``SPEC.md:16,205,261``); ``solve_raar``
composes the reference's own projections with the Luke (2005) update given in
SURVEY.md §8(a) row a15, and its parity is therefore "restatement only".
"""

from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import scipy.fft as sfft

ZERO_TOL_SCALE = 1024.0                       # src/grid.py:21
REDUCE_BLOCK = 1 << 14                        # src/backends.py:24
MIN_CHUNK = 1 << 12                           # src/backends.py:26
NAIVE_DFT_MAX_PIXELS = 4096                   # src/transform.py:16
T_LIT, T_DARK = 0.1, 3e-4                     # src/metrics.py:24-25

DTYPES = {
    "single": (np.float32, np.complex64, float(np.finfo(np.float32).eps)),
    "double": (np.float64, np.complex128, float(np.finfo(np.float64).eps)),
}


def zero_tol(tag: str, amplitude: np.ndarray) -> float:
    """1024 * eps(prec) * max(amplitude) (src/grid.py:33-34, src/projections.py:29-43)."""
    return ZERO_TOL_SCALE * DTYPES[tag][2] * float(np.max(amplitude, initial=0.0))


# ---------------------------------------------------------------- reductions

def deterministic_sum(values: np.ndarray) -> float:
    """Fixed block tree: np.sum per 16384-block, then np.sum of partials.

    src/backends.py:109-125 (the serial branch; the threaded branch computes
    the same partials in the same order).
    """
    flat = np.ascontiguousarray(values).reshape(-1)
    if flat.size == 0:
        raise ValueError("cannot reduce an empty grid")
    parts = [np.sum(flat[s:s + REDUCE_BLOCK]) for s in range(0, flat.size, REDUCE_BLOCK)]
    return float(np.sum(np.asarray(parts)))


def norm2(data: np.ndarray) -> float:
    """src/grid.py:161-165: |.| in field precision, cast to fp64, squared, summed."""
    mags = np.abs(np.asarray(data).ravel()).astype(np.float64)
    return float(np.sqrt(deterministic_sum(mags * mags)))


# ---------------------------------------------------------------- transforms

def fft2(u: np.ndarray, workers: int = 1) -> np.ndarray:
    """Unitary forward 2D DFT (src/transform.py:47-50)."""
    return sfft.fft2(u, norm="ortho", workers=workers)


def ifft2(u: np.ndarray, workers: int = 1) -> np.ndarray:
    """Unitary inverse 2D DFT (src/transform.py:52-55)."""
    return sfft.ifft2(u, norm="ortho", workers=workers)


def naive_dft(data: np.ndarray, direction: str = "forward") -> np.ndarray:
    """Dense-matrix unitary DFT in fp64, W_rows @ X @ W_cols^T (src/transform.py:58-81)."""
    n_y, n_x = data.shape
    if n_x * n_y > NAIVE_DFT_MAX_PIXELS:
        raise ValueError(f"grid with {n_x * n_y} pixels too large for the O(N^2) oracle "
                         f"(limit {NAIVE_DFT_MAX_PIXELS})")
    sign = {"forward": -1.0, "inverse": 1.0}[direction]

    def mat(n):
        k = np.arange(n)
        return np.exp(sign * 2j * np.pi * np.outer(k, k) / n) / np.sqrt(n)

    return mat(n_y) @ data.astype(np.complex128) @ mat(n_x).T


# ---------------------------------------------------------------- projections

def replace_modulus(u: np.ndarray, target: np.ndarray, tol: float, tag: str) -> np.ndarray:
    """Per-pixel modulus replacement, exact reference op order.

    src/projections.py:46-66: mag=|u|; safe = mag==0 ? 1 : mag;
    out = mag >= tol ? target*(u/safe) : target+0j, all in the precision's
    dtype (the Python-float tolerance is cast to the array dtype by NEP 50).
    """
    fdt, cdt, _ = DTYPES[tag]
    u = np.asarray(u).astype(cdt, copy=False)
    t = np.asarray(target).astype(fdt, copy=False)
    mag = np.abs(u)
    safe = np.where(mag == 0, 1, mag)
    scaled = t * (u / safe)
    return np.where(mag >= tol, scaled, t.astype(cdt)).astype(cdt)


def project_slm(u, p, tag):
    """P_S (src/projections.py:69-74)."""
    return replace_modulus(u, p, zero_tol(tag, p), tag)


def project_modulus(uhat, m, tag):
    """Fourier half of P_M (src/projections.py:77-83)."""
    return replace_modulus(uhat, m, zero_tol(tag, m), tag)


def _field_ok(a):
    """Field's construction check (src/grid.py:100-110)."""
    if not np.isfinite(a).all():
        raise ValueError("field contains non-finite entries")
    return a


def project_fourier(u, m, tag, workers=1):
    """P_M = F^-1 . replace_m . F (src/projections.py:86-91), with the Field
    checks of every intermediate the reference builds."""
    cdt = DTYPES[tag][1]
    vhat = _field_ok(project_modulus(_field_ok(fft2(u.astype(cdt, copy=False), workers)), m, tag))
    return _field_ok(ifft2(vhat, workers))


# ---------------------------------------------------------------- metrics

def gap(u, p, m, tag, workers=1) -> float:
    """G = ||P_S u - P_M u|| (src/metrics.py:67-71)."""
    return norm2(project_slm(u, p, tag) - project_fourier(u, m, tag, workers))


def reconstructed_intensity(u, target_energy, tag, workers=1):
    """|F u|^2 rescaled to the target energy (src/metrics.py:74-88)."""
    cdt = DTYPES[tag][1]
    amps = np.abs(_field_ok(fft2(u.astype(cdt, copy=False), workers))).astype(np.float64)
    inten = amps * amps
    total = deterministic_sum(inten)
    if total == 0:
        raise ValueError("reconstruction carries no energy")
    out = inten * (target_energy / total)
    if not np.isfinite(out).all():                # RealGrid check (src/grid.py:128-129)
        raise ValueError("grid contains non-finite entries")
    return out


def physical_error(inten, target_inten, t_lit=T_LIT, t_dark=T_DARK):
    """Summed lit/dark tolerance violations (src/metrics.py:91-112)."""
    u, m = inten, target_inten
    lit = m > 0
    dev = np.abs(m - u)
    rel = np.where(lit, dev / np.where(lit, m, 1.0), 0.0)
    lit_terms = np.where(lit & (rel > t_lit),
                         t_dark * dev / (t_lit * np.where(lit, m, 1.0)) - t_dark, 0.0)
    dark_terms = np.where(~lit & (u > t_dark), u - t_dark, 0.0)
    return deterministic_sum(lit_terms), deterministic_sum(dark_terms)


def phases_of(u, tol=0.0):
    """arg(u) in [0, 2pi), zero-branch pixels -> 0 (src/grid.py:168-176)."""
    theta = np.mod(np.angle(u.astype(np.complex128)), 2 * np.pi)
    theta[theta >= 2 * np.pi] = 0.0
    if tol > 0:
        theta[np.abs(u) < tol] = 0.0
    return theta


# ---------------------------------------------------------------- solver

def initial_iterate(m, tag, workers=1, random_phases=False, seed=0):
    """u0 = F^-1(m e^{i0}) — not projected onto S (src/solver.py:93-108)."""
    cdt = DTYPES[tag][1]
    if random_phases:
        rng = np.random.default_rng(seed)
        data = m * np.exp(1j * rng.uniform(0.0, 2 * np.pi, m.shape))
    else:
        data = m.astype(np.complex128)
    return ifft2(data.astype(cdt), workers)


def _finish(u, p, m, tag, workers):
    """Best-approximation pair (src/solver.py:201-206)."""
    v_star = ifft2(project_modulus(fft2(u, workers), m, tag), workers)
    u_star = project_slm(v_star, p, tag)
    return v_star, u_star, phases_of(u_star, zero_tol(tag, p))


class Diverged(FloatingPointError):
    """SolveDivergedError of the reference (src/solver.py:27-32,162-165)."""

    def __init__(self, iteration):
        super().__init__(f"non-finite values at iteration {iteration}")
        self.iteration = iteration


def _finite(a, it):
    if not np.isfinite(a).all():
        raise Diverged(it)
    return a


def first_nonfinite_iteration(p, m, max_iters, tag="double", workers=1):
    """The iteration whose loop body (src/solver.py:152-165) first builds a
    non-finite Field — the SolveDivergedError iteration with the metrics path
    left out — or 0. The batch API's per-mask divergence contract."""
    u = initial_iterate(m, tag, workers)
    for it in range(1, max_iters + 1):
        try:
            uhat = _finite(fft2(u, workers), it)
            v = _finite(ifft2(_finite(project_modulus(uhat, m, tag), it), workers), it)
            u = _finite(project_slm(v, p, tag), it)
        except Diverged as e:
            return e.iteration
    return 0


def solve(p, m, max_iters, tag="double", record_every=1, early_stop_tol=None,
          algorithm="gs", beta=0.9, workers=1, random_phase_init=False, seed=0,
          should_abort=None, keep_iterates=False):
    """Alternating projections (src/solver.py:111-216) or RAAR (§8 a15).

    Returns a dict: mask, u_star, v_star, records [(iter, gap, err_lit,
    err_dark)], iters_run, aborted, and (keep_iterates) the per-iteration
    iterates. Records follow the reference exactly: iterations 1, 1+r, ...,
    gap every iteration when early stopping is on.
    """
    if float(np.max(p, initial=0.0)) == 0.0:
        raise ValueError("SLM amplitude is identically zero")
    if float(np.max(m, initial=0.0)) == 0.0:
        raise ValueError("target pattern is identically zero (all dark)")
    target_inten = m.astype(np.float64) ** 2
    energy = float(target_inten.sum())
    u = initial_iterate(m, tag, workers, random_phase_init, seed)
    records, iterates = [], []
    prev, iters_run, aborted = None, 0, False
    cdt = DTYPES[tag][1]
    for it in range(1, max_iters + 1):
        # every Field the reference builds is checked finite (src/grid.py:100-110):
        # uhat, vhat, v and the new iterate (src/solver.py:152-165)
        uhat = _finite(fft2(u, workers), it)
        v = _finite(ifft2(_finite(project_modulus(uhat, m, tag), it), workers), it)
        if algorithm == "gs":
            u = project_slm(v, p, tag)
        elif algorithm == "raar":
            # x+ = b x + b P_S(2v - x) + (1 - 2b) v, v = P_M x (Luke 2005; §8 a15)
            u = (beta * u + beta * project_slm(2 * v - u, p, tag)
                 + (1 - 2 * beta) * v).astype(cdt)
        else:
            raise ValueError(f"unknown algorithm {algorithm!r}")
        _finite(u, it)
        iters_run = it
        if keep_iterates:
            iterates.append(u.copy())
        record_now = (it - 1) % record_every == 0
        if record_now or early_stop_tol is not None:
            g = gap(u, p, m, tag, workers)
            if record_now:
                el, ed = physical_error(reconstructed_intensity(u, energy, tag, workers),
                                        target_inten)
                records.append((it, g, el, ed))
            if (early_stop_tol is not None and prev is not None and g > 0
                    and abs(g - prev) <= early_stop_tol * g):
                break
            prev = g
        if should_abort is not None and should_abort():
            aborted = True
            break
    v_star, u_star, mask = _finish(u, p, m, tag, workers)
    out = dict(mask=mask, u_star=u_star, v_star=v_star, records=records,
               iters_run=iters_run, aborted=aborted)
    if keep_iterates:
        out["iterates"] = iterates
    return out


# ---------------------------------------------------------------- CPU baseline

class ThreadedGS:
    """The reference's ``threaded:N`` strategy for the timed CPU baseline.

    scipy.fft ``workers=N`` for the transforms (src/transform.py:49,54) and a
    thread pool over >=4096-pixel chunks for the per-pixel projections
    (src/backends.py:80-106). Metrics off the timed path, as the reference's
    bench does (``record_every=iters``, src/bench.py:100-102).
    """

    def __init__(self, p, m, tag, workers=None):
        self.workers = workers or os.cpu_count() or 1
        self.tag = tag
        fdt, self.cdt, _ = DTYPES[tag]
        self.p = p.astype(fdt)
        self.m = m.astype(fdt)
        self.tol_p = zero_tol(tag, p)
        self.tol_m = zero_tol(tag, m)
        self.pool = ThreadPoolExecutor(self.workers) if self.workers > 1 else None

    def _replace(self, u, t, tol):
        n = u.size
        if self.pool is None or n < 2 * MIN_CHUNK:
            return replace_modulus(u, t, tol, self.tag)
        fu, ft = u.reshape(-1), t.reshape(-1)
        out = np.empty(n, dtype=self.cdt)
        chunk = max(MIN_CHUNK, -(-n // self.workers))

        def run(s):
            out[s:s + chunk] = replace_modulus(fu[s:s + chunk], ft[s:s + chunk], tol, self.tag)

        list(self.pool.map(run, range(0, n, chunk)))
        return out.reshape(u.shape)

    def run(self, iters):
        w = self.workers
        u = ifft2(self.m.astype(self.cdt), w)
        for _ in range(iters):
            v = ifft2(self._replace(fft2(u, w), self.m, self.tol_m), w)
            u = self._replace(v, self.p, self.tol_p)
        v_star = ifft2(self._replace(fft2(u, w), self.m, self.tol_m), w)
        u_star = self._replace(v_star, self.p, self.tol_p)
        return phases_of(u_star, self.tol_p)

    def close(self):
        if self.pool is not None:
            self.pool.shutdown()


def relative_l2(a, b) -> float:
    a = np.asarray(a, dtype=np.complex128)
    b = np.asarray(b, dtype=np.complex128)
    den = math.sqrt(float(np.sum(np.abs(b) ** 2)))
    return math.sqrt(float(np.sum(np.abs(a - b) ** 2))) / (den if den > 0 else 1.0)


def weighted_phase_error(mask_a, mask_b, weight) -> float:
    """Amplitude-weighted RMS wrapped phase difference."""
    d = np.angle(np.exp(1j * (np.asarray(mask_a) - np.asarray(mask_b))))
    w = np.asarray(weight, dtype=np.float64) ** 2
    return math.sqrt(float(np.sum(w * d * d) / np.sum(w)))
