"""Execution-strategy selector kept for API compatibility.

The reference's per-pixel strategies (``serial`` / ``threaded:N``,
src/backends.py:46-106) become the CUDA grid here: every solve and transform
runs on the GPU whatever the selector says, and outputs are bitwise
independent of it (the GPU analogue of the reference's serial-vs-threaded
bitwise guarantee). The selector still parses and validates exactly like the
reference — ``BackendSelector.parse("cuda")`` is rejected, as
tests/test_backends.py:20-22 requires — so configs written for ``phasemask``
load unchanged.

``deterministic_sum`` keeps the reference's contract (a fixed-order fp64
reduction, src/backends.py:109-125) and runs on the GPU.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np

SERIAL = "serial"
THREADED = "threaded"


@dataclass(frozen=True)
class BackendSelector:
    strategy: str = SERIAL
    workers: int = 1

    def __post_init__(self):
        if self.strategy not in (SERIAL, THREADED):
            raise ValueError(f"unknown strategy: {self.strategy!r}")
        if self.workers < 1:
            raise ValueError("worker count must be >= 1")

    @staticmethod
    def parse(text: str) -> "BackendSelector":
        """Parse 'serial' or 'threaded[:N]' (reference src/backends.py:58-67)."""
        if text == SERIAL:
            return BackendSelector(SERIAL)
        if text == THREADED:
            return BackendSelector(THREADED, workers=os.cpu_count() or 1)
        if text.startswith(THREADED + ":"):
            return BackendSelector(THREADED, workers=int(text.split(":", 1)[1]))
        raise ValueError(f"cannot parse strategy {text!r}")

    @property
    def fft_workers(self) -> int:
        return self.workers if self.strategy == THREADED else 1


def deterministic_sum(values: np.ndarray, sel: BackendSelector | None = None) -> float:
    """Fixed-order fp64 sum of a real grid, on the GPU (src/backends.py:109-125)."""
    from . import _lib
    flat = np.ascontiguousarray(values).reshape(-1)
    if flat.size == 0:
        raise ValueError("cannot reduce an empty grid")
    return _lib.fixed_sum(flat.astype(np.float64, copy=False))
