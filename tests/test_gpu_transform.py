"""GPU: the transform provider (reference tests/test_transform.py, re-pointed).

Naive-DFT comparisons use the oracle's dense fp64 DFT; scipy is the
reference FFT for the size sweep.
"""

import numpy as np
import pytest
import scipy.fft as sfft

import paper_1302_0120_b200 as pm
from conftest import golden, random_field
from oracle import phasemask_oracle as orc
from oracle.phasemask_oracle import naive_dft
from paper_1302_0120_b200.grid import FOURIER_PLANE, SLM_PLANE

pytestmark = pytest.mark.gpu
EPS = np.finfo(float).eps


def test_delta_forward():
    spec = pm.GridSpec(4, 4)
    d = np.zeros(spec.shape, complex)
    d[0, 0] = 1
    out = pm.FftProvider(spec).forward(pm.Field(spec, d))
    assert out.domain_tag == FOURIER_PLANE
    np.testing.assert_allclose(out.data, np.full(spec.shape, 0.25), atol=1e-15)


def test_constant_forward_and_inverse():
    spec = pm.GridSpec(8, 8)
    c = 0.3 - 1.1j
    out = pm.FftProvider(spec).forward(pm.Field(spec, np.full(spec.shape, c)))
    assert out.data[0, 0] == pytest.approx(c * 8, rel=1e-14)
    off = out.data.copy()
    off[0, 0] = 0
    assert np.abs(off).max() < 1e-13
    c2 = 1.5 + 0.5j
    inv = pm.FftProvider(spec).inverse(pm.Field(spec, np.full(spec.shape, c2), FOURIER_PLANE))
    assert inv.data[0, 0] == pytest.approx(c2 * 8, rel=1e-14)


def test_matches_naive_oracle(rng):
    spec = pm.GridSpec(8, 8)
    prov = pm.FftProvider(spec)
    f = random_field(spec, rng)
    assert np.abs(prov.forward(pm.Field(spec, f)).data - naive_dft(f)).max() < 1e-12
    g = random_field(spec, rng)
    assert np.abs(prov.inverse(pm.Field(spec, g, FOURIER_PLANE)).data - naive_dft(g, "inverse")).max() < 1e-12


def test_round_trip_and_unitarity(rng):
    for n in (8, 16, 64, 256):
        spec = pm.GridSpec(n, n)
        prov = pm.FftProvider(spec)
        f = random_field(spec, rng)
        fw = prov.forward(pm.Field(spec, f))
        back = prov.inverse(fw).data
        assert np.linalg.norm(back - f) <= 16 * EPS * np.linalg.norm(f)
        ratio = np.linalg.norm(fw.data) / np.linalg.norm(f)
        assert abs(ratio - 1) <= 16 * EPS


def test_single_precision_oracle(rng):
    spec = pm.GridSpec(16, 16)
    f = random_field(spec, rng, np.complex64)
    out = pm.FftProvider(spec, pm.SINGLE).forward(pm.Field(spec, f)).data
    assert out.dtype == np.complex64
    assert np.abs(out - naive_dft(f).astype(np.complex64)).max() <= 1e-4


@pytest.mark.parametrize("tag", ["double", "single"])
def test_every_size_against_scipy(tag, rng):
    prec = pm.Precision.from_tag(tag)
    bound = 1e-14 if tag == "double" else 1e-6
    sizes = [(1, 1), (2, 2), (4, 8), (16, 16), (32, 64), (128, 128), (256, 256), (512, 512), (1024, 1024),
             (2048, 2048), (4096, 4096), (8, 256), (1024, 16), (4096, 2), (2, 4096)]
    for nx, ny in sizes:
        spec = pm.GridSpec(nx, ny)
        x = random_field(spec, rng, prec.complex_dtype)
        prov = pm.FftProvider(spec, prec)
        y = prov.forward(pm.Field(spec, x)).data
        ref = sfft.fft2(x.astype(np.complex128), norm="ortho")
        assert np.linalg.norm(y - ref) / np.linalg.norm(ref) <= bound, (nx, ny)
        z = prov.inverse(pm.Field(spec, x, FOURIER_PLANE)).data
        ref = sfft.ifft2(x.astype(np.complex128), norm="ortho")
        assert np.linalg.norm(z - ref) / np.linalg.norm(ref) <= bound, (nx, ny)


def test_reference_fft_kats():
    k = golden("kats")
    for key in [x for x in k if x.startswith("fft_") and x.endswith("_in")]:
        stem = key[:-3]
        tag = stem.rsplit("_", 1)[1]
        ny, nx = k[key].shape
        spec = pm.GridSpec(nx, ny)
        prec = pm.Precision.from_tag(tag)
        prov = pm.FftProvider(spec, prec)
        bound = 1e-13 if tag == "double" else 2e-6
        f = prov.forward(pm.Field(spec, k[key])).data
        i = prov.inverse(pm.Field(spec, k[key], FOURIER_PLANE)).data
        assert np.abs(f - k[stem + "_fwd"]).max() <= bound * np.abs(k[stem + "_fwd"]).max()
        assert np.abs(i - k[stem + "_inv"]).max() <= bound * np.abs(k[stem + "_inv"]).max()


def test_plan_reuse_is_bitwise(rng):
    spec = pm.GridSpec(32, 32)
    prov = pm.FftProvider(spec)
    f = pm.Field(spec, random_field(spec, rng))
    np.testing.assert_array_equal(prov.forward(f).data, prov.forward(f).data)


def test_mismatch_raises(rng):
    prov = pm.FftProvider(pm.GridSpec(8, 8))
    with pytest.raises(pm.PlanMismatchError):
        prov.forward(pm.Field(pm.GridSpec(4, 4), random_field(pm.GridSpec(4, 4), rng)))
    with pytest.raises(pm.PlanMismatchError):
        prov.forward(pm.Field(pm.GridSpec(8, 8), random_field(pm.GridSpec(8, 8), rng), FOURIER_PLANE))


def test_batched_transform_matches_single(rng):
    from paper_1302_0120_b200.transform import fft2
    x = random_field(pm.GridSpec(64, 32), rng)
    xs = np.stack([x, 2 * x, x.conj()])
    y = fft2(xs)
    for a, b in zip(y, xs):
        np.testing.assert_array_equal(a, fft2(b))


def test_unsupported_prime_factor_is_not_implemented(rng):
    with pytest.raises(NotImplementedError, match="prime factors 2, 3, 5, 7"):
        pm.FftProvider(pm.GridSpec(22, 13)).forward(pm.Field(pm.GridSpec(22, 13), np.zeros((13, 22))))


@pytest.mark.parametrize("nx,ny", [(800, 600), (6, 10), (15, 8), (49, 12), (1000, 90), (3, 1),
                                   # every register composite (6 ... 32) and long chains
                                   (9, 14), (20, 21), (27, 28), (24, 25), (96, 160), (243, 7),
                                   (343, 5), (625, 48), (4050, 3), (3, 3969), (2187, 2)])
@pytest.mark.parametrize("tag", ["double", "single"])
def test_mixed_radix_transform_matches_scipy(nx, ny, tag, rng):
    """Sides with prime factors 2, 3, 5, 7 (the paper's 800x600 SLM) run the
    mixed-radix path; unitary forward / inverse against scipy ortho."""
    prec = pm.Precision.from_tag(tag)
    spec = pm.GridSpec(nx, ny)
    x = random_field(spec, rng, prec.complex_dtype)
    prov = pm.FftProvider(spec, prec)
    tol = 1e-12 if tag == "double" else 2e-6
    fwd = prov.forward(pm.Field(spec, x)).data
    assert orc.relative_l2(fwd, sfft.fft2(x.astype(np.complex128), norm="ortho")) <= tol
    inv = prov.inverse(pm.Field(spec, fwd, FOURIER_PLANE)).data
    assert orc.relative_l2(inv, x) <= tol
    if nx * ny <= 4096:
        assert np.abs(fwd - orc.naive_dft(x)).max() <= (1e-12 if tag == "double" else 1e-5)


@pytest.mark.parametrize("nx,ny", [(8, 8), (16, 4), (64, 64), (60, 42)])
def test_naive_dft_public_name_matches_reference_oracle(nx, ny):
    """pm.naive_dft (the reference's src/transform.py:56-81, exported as in its
    src/__init__.py:13) on the device: equal to the dense-matrix oracle and to
    the provider's transform, both directions, fp64."""
    rng = np.random.default_rng(nx * 100 + ny)
    x = rng.standard_normal((ny, nx)) + 1j * rng.standard_normal((ny, nx))
    spec = pm.GridSpec(nx, ny)
    for d in ("forward", "inverse"):
        plane = pm.grid.SLM_PLANE if d == "forward" else pm.grid.FOURIER_PLANE
        got = pm.naive_dft(pm.Field(spec, x, plane), d)
        assert got.domain_tag == (pm.grid.FOURIER_PLANE if d == "forward" else pm.grid.SLM_PLANE)
        assert orc.relative_l2(got.data, orc.naive_dft(x, d)) <= 1e-13
    prov = pm.FftProvider(spec)
    assert orc.relative_l2(pm.naive_dft(pm.Field(spec, x)).data, prov.forward(pm.Field(spec, x)).data) <= 1e-12


def test_naive_dft_guard_and_direction():
    spec = pm.GridSpec(128, 64)
    with pytest.raises(ValueError, match="too large for the O"):
        pm.naive_dft(pm.Field(spec, np.zeros(spec.shape, complex)))
    with pytest.raises(ValueError, match="unknown direction"):
        pm.naive_dft(pm.Field(pm.GridSpec(4, 4), np.zeros((4, 4), complex)), "sideways")
