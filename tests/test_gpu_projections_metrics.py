"""GPU: projections and metrics (reference tests/test_projections.py and
tests/test_metrics.py, re-pointed at the CUDA path)."""

import math

import numpy as np
import pytest

import paper_1302_0120_b200 as pm
from conftest import golden, random_field
from oracle import phasemask_oracle as orc
from paper_1302_0120_b200.grid import FOURIER_PLANE
from paper_1302_0120_b200.metrics import (ErrorTolerances, contrast_ratio, gap, physical_error,
                                          reconstructed_intensity)
from paper_1302_0120_b200.projections import project_fourier, project_modulus, project_slm

pytestmark = pytest.mark.gpu
EPS = np.finfo(float).eps


def slm(spec, p):
    return pm.SlmConstraint(pm.RealGrid(spec, p))


def test_project_slm_kats():
    spec = pm.GridSpec(1, 1)
    assert project_slm(pm.Field(spec, np.array([[3 + 4j]])), slm(spec, np.ones((1, 1)))).data[0, 0] == \
        pytest.approx(0.6 + 0.8j, abs=1e-15)
    assert project_slm(pm.Field(spec, np.zeros((1, 1))), slm(spec, np.full((1, 1), 2.0))).data[0, 0] == 2 + 0j


@pytest.mark.parametrize("fn", ["slm", "modulus", "gap"])
def test_single_precision_threshold_is_on_the_modulus(fn):
    """fp32 zero-branch decision is |u| >= zero_tol (src/projections.py:46-55),
    including moduli between zero_tol and sqrt(zero_tol), where a test on |u|^2
    would differ; checked bitwise against the oracle restatement."""
    spec = pm.GridSpec(8, 8)
    t = np.ones(spec.shape)                        # zero_tol = 1024 eps32 = 1.22e-4
    rng = np.random.default_rng(5)
    phase = np.exp(1j * rng.uniform(0, 2 * np.pi, spec.shape))
    mags = np.full(spec.shape, 1e-3)               # >= tol, but |u|^2 = 1e-6 < tol
    mags[0, :4] = [5e-5, 1.2e-4, 1.25e-4, 0.0]     # below / at the threshold / zero
    u = (mags * phase).astype(np.complex64)
    tol = orc.zero_tol("single", t)
    if fn == "slm":
        got = project_slm(pm.Field(spec, u), pm.SlmConstraint(pm.RealGrid(spec, t), pm.SINGLE)).data
    elif fn == "modulus":
        got = project_modulus(pm.Field(spec, u, FOURIER_PLANE),
                              pm.FourierConstraint(pm.RealGrid(spec, t), pm.SINGLE)).data
    else:
        m = np.abs(random_field(spec, rng))
        g = gap(pm.Field(spec, u), pm.SlmConstraint(pm.RealGrid(spec, t), pm.SINGLE),
                pm.FourierConstraint(pm.RealGrid(spec, m), pm.SINGLE), pm.FftProvider(spec, pm.SINGLE))
        assert g == pytest.approx(orc.gap(u, t, m, "single"), rel=1e-5)
        return
    want = orc.replace_modulus(u, t, tol, "single")
    zero = np.abs(want - t) == 0
    np.testing.assert_array_equal(zero, np.abs(got - t) == 0)          # same branch everywhere
    np.testing.assert_allclose(got, want, rtol=2e-7, atol=0)


def test_project_modulus_kats():
    spec = pm.GridSpec(1, 1)
    c = pm.FourierConstraint(pm.RealGrid(spec, np.full((1, 1), math.sqrt(2))))
    assert project_modulus(pm.Field(spec, np.array([[1 - 1j]]), FOURIER_PLANE), c).data[0, 0] == \
        pytest.approx(1 - 1j, abs=1e-15)
    c1 = pm.FourierConstraint(pm.RealGrid(spec, np.ones((1, 1))))
    assert project_modulus(pm.Field(spec, np.array([[-5 + 0j]]), FOURIER_PLANE), c1).data[0, 0] == \
        pytest.approx(-1 + 0j, abs=1e-15)
    c5 = pm.FourierConstraint(pm.RealGrid(spec, np.full((1, 1), 0.5)))
    assert project_modulus(pm.Field(spec, np.zeros((1, 1)), FOURIER_PLANE), c5).data[0, 0] == 0.5 + 0j


def test_fixed_point_feasibility_idempotence(rng):
    spec = pm.GridSpec(16, 16)
    p = rng.uniform(0.5, 2.0, spec.shape)
    u = pm.Field(spec, p * np.exp(1j * rng.uniform(0, 2 * np.pi, spec.shape)))
    assert np.abs(project_slm(u, slm(spec, p)).data - u.data).max() <= 4 * EPS * p.max()
    p2 = rng.uniform(0.1, 3.0, spec.shape)
    out = project_slm(pm.Field(spec, random_field(spec, rng)), slm(spec, p2))
    assert np.all(np.abs(np.abs(out.data) - p2) <= 4 * EPS * p2)
    twice = project_slm(out, slm(spec, p2))
    assert np.abs(twice.data - out.data).max() <= 4 * EPS * p2.max()


def test_nearest_point_spot_check(rng):
    spec = pm.GridSpec(8, 8)
    p = rng.uniform(0.2, 2.0, spec.shape)
    c = slm(spec, p)
    for _ in range(50):
        u = random_field(spec, rng)
        proj = project_slm(pm.Field(spec, u), c).data
        alt = p * np.exp(1j * rng.uniform(0, 2 * np.pi, spec.shape))
        assert np.linalg.norm(u - proj) <= np.linalg.norm(u - alt) + 1e-12


def test_zero_branch_bitwise_idempotent():
    spec = pm.GridSpec(4, 4)
    c = pm.FourierConstraint(pm.RealGrid(spec, np.full(spec.shape, 0.5)))
    z = pm.Field(spec, np.zeros(spec.shape), FOURIER_PLANE)
    once = project_modulus(z, c)
    np.testing.assert_array_equal(once.data, project_modulus(once, c).data)


def test_wrong_plane_and_grid_rejected(rng):
    spec = pm.GridSpec(4, 4)
    with pytest.raises(ValueError):
        project_slm(pm.Field(spec, random_field(spec, rng), FOURIER_PLANE), slm(spec, np.ones(spec.shape)))
    with pytest.raises(ValueError):
        project_slm(pm.Field(spec, random_field(spec, rng)), slm(pm.GridSpec(8, 8), np.ones((8, 8))))


def test_project_fourier_matches_naive_composition(rng):
    spec = pm.GridSpec(8, 8)
    prov = pm.FftProvider(spec)
    for _ in range(10):
        u = random_field(spec, rng)
        m = rng.uniform(0, 2, spec.shape)
        got = project_fourier(pm.Field(spec, u), pm.FourierConstraint(pm.RealGrid(spec, m)), prov).data
        vhat = orc.replace_modulus(orc.naive_dft(u), m, orc.zero_tol("double", m), "double")
        assert np.abs(got - orc.naive_dft(vhat, "inverse")).max() < 1e-12


def test_project_fourier_properties(rng):
    spec = pm.GridSpec(16, 16)
    prov = pm.FftProvider(spec)
    u = random_field(spec, rng)
    m = rng.uniform(0.1, 2, spec.shape)
    out = project_fourier(pm.Field(spec, u), pm.FourierConstraint(pm.RealGrid(spec, m)), prov)
    assert np.linalg.norm(out.data) == pytest.approx(np.linalg.norm(m), rel=16 * EPS)
    mods = np.abs(prov.forward(out).data)
    assert np.all(np.abs(mods - m) <= 32 * EPS * np.maximum(m, 1))
    m_feas = np.abs(prov.forward(pm.Field(spec, u)).data)
    back = project_fourier(pm.Field(spec, u), pm.FourierConstraint(pm.RealGrid(spec, m_feas)), prov)
    assert np.linalg.norm(back.data - u) <= 32 * EPS * np.linalg.norm(u)


@pytest.mark.parametrize("tag", ["double", "single"])
def test_reference_projection_kats(tag):
    k = golden("kats")
    prec = pm.Precision.from_tag(tag)
    u, t = k[f"proj_{tag}_u"], k[f"proj_{tag}_t"]
    spec = pm.GridSpec(32, 32)
    rt = 1e-15 if tag == "double" else 3e-7
    got = project_slm(pm.Field(spec, u), pm.SlmConstraint(pm.RealGrid(spec, t), prec)).data
    np.testing.assert_allclose(got, k[f"proj_{tag}_slm"], rtol=rt, atol=rt)
    mc = pm.FourierConstraint(pm.RealGrid(spec, t), prec)
    got = project_modulus(pm.Field(spec, u, FOURIER_PLANE), mc).data
    np.testing.assert_allclose(got, k[f"proj_{tag}_mod"], rtol=rt, atol=rt)
    got = project_fourier(pm.Field(spec, u), mc, pm.FftProvider(spec, prec)).data
    ref = k[f"proj_{tag}_fourier"]
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= (1e-14 if tag == "double" else 1e-6)
    g = gap(pm.Field(spec, u), pm.SlmConstraint(pm.RealGrid(spec, t), prec), mc, pm.FftProvider(spec, prec))
    assert g == pytest.approx(float(k[f"gap_{tag}"]), rel=1e-13 if tag == "double" else 1e-6)


def test_gap_hand_checked_2x2():
    spec = pm.GridSpec(2, 2)
    u = np.array([[1 + 1j, -1 + 0j], [0 + 2j, 0.5 - 0.5j]])
    p = np.ones(spec.shape)
    m = np.full(spec.shape, 0.75)
    ps = p * u / np.abs(u)
    uh = orc.naive_dft(u)
    pmu = orc.naive_dft(m * uh / np.abs(uh), "inverse")
    want = math.sqrt(sum(abs(d) ** 2 for d in (ps - pmu).ravel()))
    got = gap(pm.Field(spec, u), slm(spec, p), pm.FourierConstraint(pm.RealGrid(spec, m)), pm.FftProvider(spec))
    assert got == pytest.approx(want, rel=1e-12)


def test_gap_zero_at_consistent_point_and_positive_otherwise(rng):
    spec = pm.GridSpec(16, 16)
    prov = pm.FftProvider(spec)
    p = rng.uniform(0.5, 1.5, spec.shape)
    u = pm.Field(spec, p * np.exp(1j * rng.uniform(0, 2 * np.pi, spec.shape)))
    m = np.abs(prov.forward(u).data)
    assert gap(u, slm(spec, p), pm.FourierConstraint(pm.RealGrid(spec, m)), prov) <= 16 * 100 * EPS
    spec8 = pm.GridSpec(8, 8)
    assert gap(pm.Field(spec8, random_field(spec8, rng)), slm(spec8, np.ones((8, 8))),
               pm.FourierConstraint(pm.RealGrid(spec8, rng.uniform(0.1, 1, (8, 8)))), pm.FftProvider(spec8)) > 1e-6


def test_reconstructed_intensity(rng):
    spec = pm.GridSpec(8, 8)
    prov = pm.FftProvider(spec)
    u = pm.Field(spec, random_field(spec, rng))
    m = np.abs(prov.forward(u).data)
    np.testing.assert_allclose(reconstructed_intensity(u, prov, float((m ** 2).sum())).data, m ** 2,
                               rtol=1e-12, atol=1e-14)
    a = reconstructed_intensity(u, prov, 1.0).data
    b = reconstructed_intensity(pm.Field(spec, 2.5 * u.data), prov, 1.0).data
    np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-16)
    raw = np.abs(orc.naive_dft(u.data)) ** 2
    np.testing.assert_allclose(reconstructed_intensity(u, prov, 3.7).data, raw * (3.7 / raw.sum()), rtol=1e-12)
    with pytest.raises(ValueError):
        reconstructed_intensity(pm.Field(pm.GridSpec(4, 4), np.zeros((4, 4))), pm.FftProvider(pm.GridSpec(4, 4)), 1.0)


def test_physical_error_unit_values():
    spec = pm.GridSpec(1, 1)
    tol = ErrorTolerances()

    def g(v):
        return pm.RealGrid(spec, np.array([[v]]))

    lit, dark = physical_error(g(1.2), g(1.0), tol)
    assert lit == pytest.approx(3e-4, rel=1e-12) and dark == 0.0
    lit, dark = physical_error(g(4e-4), g(0.0), tol)
    assert lit == 0.0 and dark == pytest.approx(1e-4, rel=1e-12)
    assert physical_error(g(0.7), g(0.7), tol) == (0.0, 0.0)
    assert physical_error(g(1.05), g(1.0), tol) == (0.0, 0.0)
    assert physical_error(g(0.875), g(1.0), ErrorTolerances(t_lit=0.125))[0] == 0.0


def test_contrast_ratio():
    spec = pm.GridSpec(4, 4)
    t = np.zeros(spec.shape)
    t[1, 1] = t[2, 2] = 1.0
    target = pm.RealGrid(spec, t)
    assert contrast_ratio(target, target) == math.inf
    inten = np.full(spec.shape, 9e-4)
    inten[1, 1] = inten[2, 2] = 0.9
    assert contrast_ratio(pm.RealGrid(spec, inten), target) == pytest.approx(1000.0)


def test_norm2_and_phases_on_gpu(rng):
    x = random_field(pm.GridSpec(300, 7), rng)
    assert pm.norm2(x) == pytest.approx(orc.norm2(x), rel=1e-14)
    assert pm.norm2(x.astype(np.complex64)) == pytest.approx(orc.norm2(x.astype(np.complex64)), rel=1e-6)
    spec = pm.GridSpec(300, 7)
    x[0, :3] = [0, -0.0 - 1e-30j, -1 + 0j]
    f = pm.Field(spec, x)
    # CUDA's atan2 is within 2 ulp of glibc's; zero-branch / wrap decisions exact
    np.testing.assert_allclose(pm.phases_of(f, 1e-12).phases, orc.phases_of(x, 1e-12), rtol=0, atol=4e-15)
    np.testing.assert_allclose(pm.phases_of(f).phases, orc.phases_of(x), rtol=0, atol=4e-15)
    assert pm.phases_of(f, 1e-12).phases[0, :2].tolist() == [0.0, 0.0]
    from paper_1302_0120_b200.backends import deterministic_sum
    v = rng.standard_normal(100000)
    assert deterministic_sum(v) == pytest.approx(orc.deterministic_sum(v), rel=1e-12, abs=1e-12)


# ---------------------------------------------------------------- §8f-2
def _ref_log_u8(intensity, floor=1e-6):
    """service._log_scale_u8 (src/service.py:91-95), restated."""
    import math
    peak = intensity.max()
    data = intensity / peak if peak > 0 else np.zeros_like(intensity)
    data = (np.log10(np.maximum(data, floor)) - math.log10(floor)) / (-math.log10(floor))
    return np.round(data * 255.0).astype(np.uint8)


@pytest.mark.parametrize("prec", [pm.DOUBLE, pm.SINGLE])
@pytest.mark.parametrize("shape", [(64, 64), (48, 80), (600, 800)])
def test_reconstruction_intensity_and_log_image(prec, shape):
    from paper_1302_0120_b200.metrics import reconstruction_log_image, reconstructed_intensity
    from paper_1302_0120_b200.patterns import to_centered_order
    ny, nx = shape
    spec = pm.GridSpec(nx, ny)
    rng = np.random.default_rng(5)
    u = (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)).astype(prec.complex_dtype)
    f = pm.Field(spec, u)
    prov = pm.FftProvider(spec, prec)
    E = 17.0
    F = np.fft.fft2(u.astype(np.complex128), norm="ortho").astype(prec.complex_dtype)
    amps = np.abs(F).astype(np.float64)
    ref = amps * amps
    ref = ref * (E / ref.sum())
    got = reconstructed_intensity(f, prov, E).data
    # fp32: the two fp32 FFTs differ by ~eps |u|, relative to the peak for small bins
    np.testing.assert_allclose(got, ref, rtol=1e-12 if prec is pm.DOUBLE else 2e-5,
                               atol=0 if prec is pm.DOUBLE else 1e-6 * ref.max())
    img = reconstruction_log_image(f, prov, E)
    want = _ref_log_u8(to_centered_order(pm.RealGrid(spec, got)).data)
    # same intensities: only log10 ulps may move a value across a .5 boundary
    assert np.abs(img.astype(int) - want.astype(int)).max() <= 1
    assert np.mean(img == want) > 0.999
    # unscaled intensity; zero energy is rejected with the reference's message
    raw = reconstructed_intensity(f, prov).data
    np.testing.assert_allclose(raw * (E / raw.sum()), got, rtol=1e-12 if prec is pm.DOUBLE else 1e-6)
    with pytest.raises(ValueError, match="reconstruction carries no energy"):
        reconstructed_intensity(pm.Field(spec, np.zeros(shape, prec.complex_dtype)), prov, E)


def test_reconstruction_image_batch_matches_single():
    spec = pm.GridSpec(48, 32)
    plan = pm.transform.get_plan(spec, pm.DOUBLE)
    rng = np.random.default_rng(9)
    u = rng.standard_normal((3, 32, 48)) + 1j * rng.standard_normal((3, 32, 48))
    E = np.array([1.0, 2.0, 3.0])
    inten, img = plan.recon_image(u, E, 1e-6)
    for b in range(3):
        i1, g1 = plan.recon_image(u[b], E[b], 1e-6)
        np.testing.assert_array_equal(inten[b], i1)
        np.testing.assert_array_equal(img[b], g1)


# --- norm homogeneity on the device reduction (reference tests/test_grid.py:81-88) ---
from hypothesis import given, settings, strategies as st  # noqa: E402


@given(st.floats(-1e3, 1e3).filter(lambda a: abs(a) > 1e-6))
@settings(max_examples=25, deadline=None)
def test_norm2_absolute_homogeneity(alpha):
    from paper_1302_0120_b200.grid import norm2
    rng = np.random.default_rng(7)
    spec = pm.GridSpec(8, 8)
    data = rng.standard_normal(spec.shape) + 1j * rng.standard_normal(spec.shape)
    base = norm2(pm.Field(spec, data))
    scaled = norm2(pm.Field(spec, alpha * data))
    assert scaled == pytest.approx(abs(alpha) * base, rel=4 * np.finfo(float).eps * 10)


def _straddle(tag, tol, n, seed):
    """n complex values whose numpy modulus np.abs(u) lies within 2 ulp of
    float(tol) in the precision (the reference compares in the array dtype,
    NEP 50), led by values on which np.abs and hypot fall on opposite sides of
    the tolerance."""
    prec = pm.Precision.from_tag(tag)
    fdt, cdt = np.dtype(prec.float_dtype).type, np.dtype(prec.complex_dtype).type
    itype = np.int32 if fdt == np.float32 else np.int64
    tf = fdt(tol)
    rng = np.random.default_rng(seed)
    k = 2_000_000
    th = rng.uniform(0.05, np.pi / 2 - 0.05, k) + rng.integers(0, 4, k) * (np.pi / 2)
    r = float(tf) * (1.0 + rng.integers(-8, 9, k) * float(np.finfo(fdt).eps) * 0.5)
    z = (r * np.cos(th)).astype(fdt) + 1j * (r * np.sin(th)).astype(fdt)
    z = z.astype(cdt)
    mag = np.abs(z)
    ulps = np.abs(mag.view(itype).astype(np.int64) - np.array(tf).view(itype).astype(np.int64))
    near = ulps <= 2
    hyp = np.hypot(z.real, z.imag).astype(fdt)
    split = near & ((hyp >= tf) != (mag >= tf))
    pick = np.concatenate([np.nonzero(split)[0][: n // 4], np.nonzero(near & ~split)[0]])[:n]
    assert pick.size == n and split.any()
    return z[pick], int(split.sum())


@pytest.mark.parametrize("tag", ["single", "double"])
@pytest.mark.parametrize("which", ["slm", "modulus"])
def test_zero_branch_straddling_tolerance_bitwise(tag, which):
    """Pixels with |u| within +-2 ulp of zero_tol, including ones where numpy's
    |u| and hypot disagree: the GPU takes numpy's decision on every one
    (src/projections.py:49-53) and the replaced values agree to the ulp."""
    prec = pm.Precision.from_tag(tag)
    spec = pm.GridSpec(64, 64)
    rng = np.random.default_rng(3)
    t = rng.uniform(0.25, 1.0, spec.shape)
    t[0, 0] = 1.0 + 2 * float(np.finfo(prec.float_dtype).eps)   # max(t): the tolerance scale
    tol = prec.zero_tol(float(t.max()))
    u, _ = _straddle(tag, tol, spec.n, seed=17 if which == "slm" else 19)
    u = u.reshape(spec.shape)
    if which == "slm":
        got = project_slm(pm.Field(spec, u), pm.SlmConstraint(pm.RealGrid(spec, t), prec)).data
    else:
        got = project_modulus(pm.Field(spec, u, FOURIER_PLANE), pm.FourierConstraint(pm.RealGrid(spec, t), prec)).data
    want = orc.replace_modulus(u, t, tol, tag)
    tq = t.astype(prec.float_dtype)
    zero_got = (got.real == tq) & (got.imag == 0)
    zero_want = (want.real == tq) & (want.imag == 0)
    assert zero_want.any() and (~zero_want).any()
    np.testing.assert_array_equal(zero_got, zero_want)
    np.testing.assert_allclose(got, want, rtol=4 * prec.eps_machine, atol=0)


@pytest.mark.parametrize("tag", ["single", "double"])
def test_phases_zero_decision_straddling(tag):
    """phases_of's `np.abs(u) < zero_tol -> 0` (src/grid.py:174-175) on values at
    the tolerance +-2 ulp: the device decision is numpy's."""
    prec = pm.Precision.from_tag(tag)
    tol = prec.zero_tol(1.0)
    u, _ = _straddle(tag, tol, 4096, seed=23)
    spec = pm.GridSpec(64, 64)
    got = pm.phases_of(pm.Field(spec, u.reshape(spec.shape)), tol).phases
    want = orc.phases_of(u.reshape(spec.shape), tol)
    np.testing.assert_array_equal(got == 0.0, want == 0.0)
