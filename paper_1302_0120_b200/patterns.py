"""Host-side problem construction: spot targets, Gaussian beams, DFT order.

This is input preparation, not the hot path. It restates the reference's
pattern helpers so callers (bench.py, tests, the batch API) can build the
same target moduli ``m`` and SLM amplitudes ``p`` the reference builds:

* ``spot_pattern``            — reference ``src/patterns.py:63-74``
* ``to_fourier_order``        — reference ``src/patterns.py:102-105``
* ``to_centered_order``       — reference ``src/patterns.py:108-111``
* ``modulus_from_intensity``  — reference ``src/patterns.py:114-116``
* ``spot_grid_centers``       — reference ``src/bench.py:78-82``
* ``make_problem``            — the non-degenerate synthetic generator of
  SURVEY.md §8(d) (seeded random spots + energy-matched Gaussian beam), the
  input to every BASELINE.json config.

Everything here is plain numpy on host arrays of shape ``(n_y, n_x)``.
"""

from __future__ import annotations

import math

import numpy as np

from .grid import GridSpec, RealGrid

LOG_FLOOR = 1e-6        # display floor of the log-scale images (src/patterns.py:22)


def spot_grid_centers(spec: GridSpec, cols: int = 3, rows: int = 3):
    """Evenly spaced spot lattice (reference ``src/bench.py:78-82``)."""
    out = []
    for q in range(rows):
        for i in range(cols):
            out.append((round((i + 1) * spec.n_x / (cols + 1)),
                        round((q + 1) * spec.n_y / (rows + 1))))
    return tuple(out)


def spot_pattern(spec: GridSpec, centers, radius: int = 1,
                 intensity: float = 1.0) -> RealGrid:
    """Discs of ``intensity`` on a dark background, centred visual frame.

    Pixel (j, k) is lit when (j-j0)^2 + (k-k0)^2 < radius^2, as in the
    reference (``src/patterns.py:63-74``); overlapping discs are rejected.
    """
    if radius < 1:
        raise ValueError("spot radius must be >= 1 pixel")
    if intensity <= 0:
        raise ValueError("spot intensity must be positive")
    img = np.zeros(spec.shape)
    hits = np.zeros(spec.shape, dtype=np.int32)
    rows, cols = np.mgrid[0:spec.n_y, 0:spec.n_x]
    for j0, k0 in centers:
        if not (0 <= j0 < spec.n_x and 0 <= k0 < spec.n_y):
            raise ValueError(f"spot center ({j0}, {k0}) outside grid")
        lit = (cols - j0) ** 2 + (rows - k0) ** 2 < radius ** 2
        hits += lit
        img[lit] = intensity
    if (hits > 1).any():
        raise ValueError("spot discs overlap")
    return RealGrid(spec, img)


def to_fourier_order(g: RealGrid) -> RealGrid:
    """Centred visual frame -> unshifted DFT order (reference ``:102-105``)."""
    shift = (g.spec.n_y // 2, g.spec.n_x // 2)
    return RealGrid(g.spec, np.roll(g.data, shift, axis=(0, 1)))


def to_centered_order(g: RealGrid) -> RealGrid:
    """Inverse of :func:`to_fourier_order` (reference ``:108-111``)."""
    shift = (-(g.spec.n_y // 2), -(g.spec.n_x // 2))
    return RealGrid(g.spec, np.roll(g.data, shift, axis=(0, 1)))


def modulus_from_intensity(intensity: RealGrid) -> RealGrid:
    """m = sqrt(I) (reference ``src/patterns.py:114-116``)."""
    return RealGrid(intensity.spec, np.sqrt(intensity.data))


def random_spot_centers(spec: GridSpec, n_spots: int, seed: int,
                        min_sep2: int = 16):
    """Rejection-sampled spot centres, SURVEY.md §8(d).

    Centres are drawn uniformly from the inner 3/4 of the grid and kept when
    they are at least sqrt(min_sep2) pixels from every accepted centre.
    """
    rng = np.random.default_rng(seed)
    lo_x, hi_x = spec.n_x // 8, 7 * spec.n_x // 8
    lo_y, hi_y = spec.n_y // 8, 7 * spec.n_y // 8
    chosen: set[tuple[int, int]] = set()
    if spec.n_x == spec.n_y:
        draw = lambda: rng.integers(lo_x, hi_x, 2)  # noqa: E731  (square: one call, as §8d)
    else:
        draw = lambda: (rng.integers(lo_x, hi_x), rng.integers(lo_y, hi_y))  # noqa: E731
    tries = 0
    while len(chosen) < n_spots:
        tries += 1
        if tries > 200 * n_spots + 10000:
            raise ValueError(f"cannot place {n_spots} spots {math.sqrt(min_sep2):g} px apart "
                             f"on a {spec.n_x}x{spec.n_y} grid")
        j, k = draw()
        j, k = int(j), int(k)
        if all((j - a) ** 2 + (k - b) ** 2 >= min_sep2 for a, b in chosen):
            chosen.add((j, k))
    return tuple(sorted(chosen))


def gaussian_beam(spec: GridSpec, waist_frac: float = 0.25) -> np.ndarray:
    """Centred Gaussian amplitude exp(-r^2 / w^2), w = waist_frac * n."""
    y, x = np.mgrid[0:spec.n_y, 0:spec.n_x].astype(np.float64)
    dx = x + 0.5 - spec.n_x / 2
    dy = y + 0.5 - spec.n_y / 2
    if spec.n_x == spec.n_y:
        w2 = (spec.n_x * waist_frac) ** 2
        return np.exp(-(dx ** 2 + dy ** 2) / w2)
    return np.exp(-(dx / (spec.n_x * waist_frac)) ** 2
                  - (dy / (spec.n_y * waist_frac)) ** 2)


def make_problem(n_x: int, n_spots: int = 50, seed: int = 7, n_y: int | None = None):
    """The SURVEY.md §8(d) synthetic problem: (p, m) as float64 host arrays.

    m = sqrt(spot intensity) in DFT order, one lit pixel per spot (radius 1);
    p = Gaussian beam (waist n/4) energy-matched so that sum p^2 = sum m^2,
    mirroring ``default_amplitude`` (reference ``src/solver.py:86-90``).
    """
    spec = GridSpec(n_x, n_x if n_y is None else n_y)
    centers = random_spot_centers(spec, n_spots, seed)
    intensity = spot_pattern(spec, centers, radius=1)
    m = modulus_from_intensity(to_fourier_order(intensity)).data
    g = gaussian_beam(spec)
    p = g * math.sqrt(float(np.sum(m ** 2)) / float(np.sum(g ** 2)))
    return np.ascontiguousarray(p), np.ascontiguousarray(m)


def spot_targets(n_x: int, n_spots: int, seeds, n_y: int | None = None, dtype=np.float64) -> np.ndarray:
    """Stack of the §8(d) targets m for several seeds (BASELINE config 4: 256
    distinct OSPs), equal to ``make_problem(n_x, n_spots, seed)[1]`` for each
    seed, built directly: a radius-1 spot lights its centre pixel only, and m
    is 1 there, rolled into DFT order. Every target has sum m^2 = n_spots, so
    one amplitude p serves the whole stack."""
    spec = GridSpec(n_x, n_x if n_y is None else n_y)
    seeds = list(seeds)
    out = np.zeros((len(seeds), spec.n_y, spec.n_x), dtype=dtype)
    sy, sx = spec.n_y // 2, spec.n_x // 2
    for i, seed in enumerate(seeds):
        for j0, k0 in random_spot_centers(spec, n_spots, seed):
            out[i, (k0 + sy) % spec.n_y, (j0 + sx) % spec.n_x] = 1.0
    return out
