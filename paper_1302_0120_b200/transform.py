"""Unitary 2-D Fourier transforms on the GPU behind the reference's provider
contract (reference src/transform.py:23-55).

``FftProvider(spec, precision, fft_workers)`` keeps the reference's
signature, checks and errors; ``forward`` / ``inverse`` run the library's
hand-written Stockham transforms (pm_fft2) instead of scipy's DUCC0 FFT.
Both directions carry 1/sqrt(n_x) and 1/sqrt(n_y), so the pair is unitary
and Parseval holds to roundoff (reference ``norm="ortho"``).
"""

from __future__ import annotations

import threading

import numpy as np

from . import _lib
from .grid import DOUBLE, FOURIER_PLANE, SLM_PLANE, Field, GridSpec, Precision

NAIVE_DFT_MAX_PIXELS = 4096


class PlanMismatchError(ValueError):
    """Field spec or plane does not match the provider's plan (src/transform.py:19-20)."""


def default_device() -> int:
    """The process's CUDA device: PM_DEVICE, else LOCAL_RANK (one rank per GPU), else 0."""
    import os
    return int(os.environ.get("PM_DEVICE", os.environ.get("LOCAL_RANK", "0")))


_plans: dict[tuple[int, int, int, int], _lib.Plan] = {}
_plans_lock = threading.Lock()


def get_plan(spec: GridSpec, precision: Precision, device: int = 0, slot: int = 0) -> _lib.Plan:
    """Per-process plan cache keyed (n_x, n_y, precision, device).

    The GPU analogue of the service's PlanCache (src/service.py:65-82).
    ``slot`` 1 is the plan of solves with host callbacks: their callbacks may
    use transforms of the same grid (slot 0) while the solve is in flight.
    """
    key = (spec.n_x, spec.n_y, precision.code, device, slot)
    with _plans_lock:
        plan = _plans.get(key)
        if plan is None:
            plan = _lib.Plan(spec.n_x, spec.n_y, precision.code, device)
            _plans[key] = plan
        return plan


def clear_plans():
    with _plans_lock:
        for plan in _plans.values():
            plan.close()
        _plans.clear()


class FftProvider:
    """GPU transform planned for one grid spec and precision.

    Immutable after construction and safe to share across threads (the
    underlying plan serialises its calls). ``fft_workers`` is accepted for
    signature compatibility; results do not depend on it.
    """

    def __init__(self, spec: GridSpec, precision: Precision = DOUBLE,
                 fft_workers: int = 1, device: int | None = None):
        self.spec = spec
        self.precision = precision
        self.fft_workers = fft_workers
        # None: the process default (PM_DEVICE, else LOCAL_RANK, else 0), as SolveConfig.device
        self.device = default_device() if device is None else int(device)

    @property
    def plan(self) -> _lib.Plan:
        return get_plan(self.spec, self.precision, self.device)

    def _check(self, f: Field, expected_plane: str) -> np.ndarray:
        if f.spec != self.spec:
            raise PlanMismatchError(
                f"field spec {f.spec.n_x}x{f.spec.n_y} does not match plan "
                f"{self.spec.n_x}x{self.spec.n_y}")
        if f.domain_tag != expected_plane:
            raise PlanMismatchError(f"expected a {expected_plane} field, got {f.domain_tag}")
        return f.data.astype(self.precision.complex_dtype, copy=False)

    def forward(self, f: Field) -> Field:
        data = self._check(f, SLM_PLANE)
        return Field(self.spec, self.plan.fft2(data, _lib.PM_FORWARD), FOURIER_PLANE)

    def inverse(self, f: Field) -> Field:
        data = self._check(f, FOURIER_PLANE)
        return Field(self.spec, self.plan.fft2(data, _lib.PM_INVERSE), SLM_PLANE)


def fft2(data: np.ndarray, precision: Precision = DOUBLE, device: int = 0) -> np.ndarray:
    """Unitary forward transform of a (n_y, n_x) or (batch, n_y, n_x) array."""
    spec = GridSpec(data.shape[-1], data.shape[-2])
    return get_plan(spec, precision, device).fft2(data, _lib.PM_FORWARD)


def ifft2(data: np.ndarray, precision: Precision = DOUBLE, device: int = 0) -> np.ndarray:
    """Unitary inverse transform of a (n_y, n_x) or (batch, n_y, n_x) array."""
    spec = GridSpec(data.shape[-1], data.shape[-2])
    return get_plan(spec, precision, device).fft2(data, _lib.PM_INVERSE)


def naive_dft(f: Field, direction: str = "forward") -> Field:
    """The reference's textbook double-sum unitary DFT (src/transform.py:56-81),
    always double precision, guarded to small grids: a correctness oracle, not
    a production transform. Evaluated on the device (pm_naive_dft)."""
    if f.spec.n > NAIVE_DFT_MAX_PIXELS:
        raise ValueError(
            f"grid with {f.spec.n} pixels too large for the O(N^2) oracle "
            f"(limit {NAIVE_DFT_MAX_PIXELS})")
    if direction not in ("forward", "inverse"):
        raise ValueError(f"unknown direction {direction!r}")
    out = _lib.naive_dft(f.data, _lib.PM_FORWARD if direction == "forward" else _lib.PM_INVERSE)
    return Field(f.spec, out, FOURIER_PLANE if direction == "forward" else SLM_PLANE)
