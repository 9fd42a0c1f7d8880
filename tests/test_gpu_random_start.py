"""Seeded random-phase starts drawn on the device.

The reference draws phi = np.random.default_rng(seed).uniform(0, 2 pi) and
starts from m e^{i phi} (src/solver.py:100-103); the device kernel replays
numpy's PCG64 stream with per-thread jump-ahead. CPU tests pin the jump
arithmetic against numpy; GPU tests pin the kernel's draws.
"""

import numpy as np
import pytest

import paper_1302_0120_b200 as pm
from paper_1302_0120_b200 import _lib
from paper_1302_0120_b200.solver import initial_iterate

MULT = (2549297995355413924 << 64) | 4865540595714422341
MASK = (1 << 128) - 1


def _jump(inc, delta):
    """The (mult, plus) of `delta` LCG steps, as pcg_jump in csrc/pm_rng.cuh."""
    cm, cp, am, ap = MULT, inc, 1, 0
    while delta:
        if delta & 1:
            am, ap = (am * cm) & MASK, (ap * cm + cp) & MASK
        cp, cm = ((cm + 1) * cp) & MASK, (cm * cm) & MASK
        delta >>= 1
    return am, ap


def _out(state):
    hi, lo = state >> 64, state & ((1 << 64) - 1)
    x, r = hi ^ lo, hi >> 58
    return ((x >> r) | (x << ((64 - r) & 63))) & ((1 << 64) - 1)


def _numpy_start(m, seed, cdt):
    phi = np.random.default_rng(seed).uniform(0.0, 2 * np.pi, m.shape[-2:])
    return (m * np.exp(1j * phi)).astype(cdt)


def test_pcg64_state_and_jump_match_numpy():
    for seed in (0, 7, 123456789):
        s = [int(v) for v in _lib.pcg64_state(seed)]
        state, inc = (s[0] << 64) | s[1], (s[2] << 64) | s[3]
        ref = np.random.default_rng(seed).random(300)
        # element i uses the state advanced i + 1 steps, as each device thread does
        for i in (0, 1, 2, 37, 255, 299):
            a, c = _jump(inc, i + 1)
            d = (_out((state * a + c) & MASK) >> 11) * (1.0 / 9007199254740992.0)
            assert d == ref[i]
        # grid-stride stepping from element 3 by 64
        a, c = _jump(inc, 4)
        st = (state * a + c) & MASK
        sa, sc = _jump(inc, 64)
        for i in range(3, 300, 64):
            assert (_out(st) >> 11) * (1.0 / 9007199254740992.0) == ref[i]
            st = (st * sa + sc) & MASK


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(8, 8), (37, 53), (600, 800)])
def test_device_draws_match_numpy_fp64(shape):
    rng = np.random.default_rng(3)
    m = rng.random(shape)
    out = _lib.random_start(m, np.complex128, 11)
    ref = _numpy_start(m, 11, np.complex128)
    # same draws; only the device sincos may differ from libm by an ulp
    np.testing.assert_allclose(out, ref, rtol=0, atol=4e-16)


@pytest.mark.gpu
def test_device_draws_match_numpy_fp32_and_batch():
    rng = np.random.default_rng(4)
    m = rng.random((3, 64, 96)).astype(np.float32)
    out = _lib.random_start(m, np.complex64, 5)
    for b in range(3):
        ref = _numpy_start(m[b], 5, np.complex64)
        assert np.mean(out[b] == ref) > 0.999
        np.testing.assert_allclose(out[b], ref, rtol=0, atol=1e-7)


@pytest.mark.gpu
def test_random_init_solve_matches_host_start():
    """solve(random_phase_init) equals a solve seeded with numpy's start."""
    from paper_1302_0120_b200.patterns import make_problem
    from paper_1302_0120_b200.batch import solve_stack
    p, m = make_problem(64, 6, 9)
    cfg = pm.SolveConfig(max_iters=10, precision=pm.DOUBLE, random_phase_init=True, seed=21)
    dev = solve_stack(p, m[None], cfg)
    host = solve_stack(p, m[None], pm.SolveConfig(max_iters=10, precision=pm.DOUBLE),
                       init=_numpy_start(m, 21, np.complex128)[None])
    np.testing.assert_allclose(dev.gap, host.gap, rtol=1e-13)
    np.testing.assert_allclose(dev.phases, host.phases, atol=1e-9)


@pytest.mark.gpu
def test_initial_iterate_random_branch():
    spec = pm.GridSpec(32, 16)
    m = np.abs(np.random.default_rng(1).standard_normal(spec.shape))
    mc = pm.FourierConstraint(pm.RealGrid(spec, m), pm.DOUBLE)
    u0 = initial_iterate(mc, pm.FftProvider(spec), random_phases=True, seed=2)
    ref = np.fft.ifft2(_numpy_start(m, 2, np.complex128), norm="ortho")
    np.testing.assert_allclose(u0.data, ref, atol=1e-14)
