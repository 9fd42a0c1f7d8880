"""CPU: pin the oracle (oracle/phasemask_oracle.py) to the reference.

Every fixture in tests/golden was produced by the reference package itself
(tests/golden/make_golden.py). The oracle restates the reference with the
same numpy/scipy calls, so it must reproduce the fixtures bit for bit; the
reference's own known-answer tests are re-run against it as well.
"""

import math

import numpy as np
import pytest

from conftest import GOLDEN as GOLDEN_DIR, golden
from oracle import phasemask_oracle as orc
from paper_1302_0120_b200.patterns import make_problem

SOLVE_FIXTURES = ["gs16_double", "gs32_single", "gs64_double", "gs64x32_double", "gs64_single_rec3",
                  "gs128_double_early", "gs32_double_randinit", "gs256_double", "gs256_single",
                  "lattice64_double"]


@pytest.mark.parametrize("name", SOLVE_FIXTURES)
def test_oracle_reproduces_reference_solve_bitwise(name):
    g = golden(name)
    kw = {}
    if "record_every" in g:
        kw["record_every"] = int(g["record_every"])
    if "early_stop_tol" in g and float(g["early_stop_tol"]) >= 0:
        kw["early_stop_tol"] = float(g["early_stop_tol"])
    if "random_phase_init" in g and int(g["random_phase_init"]):
        kw.update(random_phase_init=True, seed=int(g["seed"]))
    o = orc.solve(g["p"], g["m"], int(g["K"]), str(g["precision"]), **kw)
    np.testing.assert_array_equal(o["mask"], g["mask"])
    np.testing.assert_array_equal(o["u_star"], g["u_star"])
    np.testing.assert_array_equal(o["v_star"], g["v_star"])
    np.testing.assert_array_equal(np.array(o["records"], dtype=np.float64), g["history"])
    assert o["iters_run"] == int(g["iters_run"])


@pytest.mark.parametrize("tag", ["double", "single"])
def test_oracle_iterates_bitwise(tag):
    g = golden(f"iterates64_{tag}")
    for K, u in zip(g["Ks"], g["u_star"]):
        o = orc.solve(g["p"], g["m"], int(K), tag)
        np.testing.assert_array_equal(o["u_star"], u)


def test_early_stop_fixture_actually_stops():
    g = golden("gs128_double_early")
    assert int(g["iters_run"]) < int(g["K"])


def test_generator_matches_fixture():
    g = golden("problem64")
    p, m = make_problem(64, 8, 7)
    np.testing.assert_array_equal(p, g["p"])
    np.testing.assert_array_equal(m, g["m"])
    assert np.isclose((p ** 2).sum(), (m ** 2).sum())
    assert (m > 0).sum() == 8


def test_oracle_kats_against_reference_primitives():
    k = golden("kats")
    for key in [x for x in k if x.startswith("fft_") and x.endswith("_in")]:
        stem = key[:-3]
        tag = stem.rsplit("_", 1)[1]
        x = k[key]
        np.testing.assert_array_equal(orc.fft2(x), k[stem + "_fwd"])
        np.testing.assert_array_equal(orc.ifft2(x), k[stem + "_inv"])
        if stem + "_naive" in k:
            np.testing.assert_allclose(orc.naive_dft(x), k[stem + "_naive"], rtol=0, atol=1e-13)
    for tag in ("double", "single"):
        u, t = k[f"proj_{tag}_u"], k[f"proj_{tag}_t"]
        np.testing.assert_array_equal(orc.project_slm(u, t, tag), k[f"proj_{tag}_slm"])
        np.testing.assert_array_equal(orc.project_modulus(u, t, tag), k[f"proj_{tag}_mod"])
        np.testing.assert_array_equal(orc.project_fourier(u, t, tag), k[f"proj_{tag}_fourier"])
        assert orc.gap(u, t, t, tag) == float(k[f"gap_{tag}"])


# --- the reference's known-answer tests, on the oracle ---------------------

def test_kat_delta_to_constant():
    d = np.zeros((4, 4), complex)
    d[0, 0] = 1
    np.testing.assert_allclose(orc.fft2(d), np.full((4, 4), 0.25), atol=1e-15)
    np.testing.assert_allclose(orc.naive_dft(d), np.full((4, 4), 0.25), atol=1e-14)


def test_kat_projections():
    one = np.ones((1, 1))
    assert orc.project_slm(np.array([[3 + 4j]]), one, "double")[0, 0] == pytest.approx(0.6 + 0.8j, abs=1e-15)
    assert orc.project_slm(np.zeros((1, 1), complex), 2 * one, "double")[0, 0] == 2 + 0j
    assert orc.project_modulus(np.array([[1 - 1j]]), math.sqrt(2) * one, "double")[0, 0] == \
        pytest.approx(1 - 1j, abs=1e-15)
    assert orc.project_modulus(np.array([[-5 + 0j]]), one, "double")[0, 0] == pytest.approx(-1, abs=1e-15)
    assert orc.project_modulus(np.zeros((1, 1), complex), 0.5 * one, "double")[0, 0] == 0.5 + 0j


def test_kat_gap_hand_checked_2x2():
    u = np.array([[1 + 1j, -1 + 0j], [0 + 2j, 0.5 - 0.5j]])
    p = np.ones((2, 2))
    m = np.full((2, 2), 0.75)
    ps = p * u / np.abs(u)
    uh = orc.naive_dft(u)
    pm = orc.naive_dft(m * uh / np.abs(uh), "inverse")
    want = math.sqrt(sum(abs(d) ** 2 for d in (ps - pm).ravel()))
    assert orc.gap(u, p, m, "double") == pytest.approx(want, rel=1e-12)


def test_kat_physical_error_unit_values():
    lit, _ = orc.physical_error(np.array([[1.2]]), np.array([[1.0]]))
    _, dark = orc.physical_error(np.array([[4e-4]]), np.array([[0.0]]))
    assert abs(lit - 3e-4) <= 1e-16 and abs(dark - 1e-4) <= 1e-16
    assert orc.physical_error(np.array([[0.7]]), np.array([[0.7]])) == (0.0, 0.0)


def test_raar_restatement_reproducible():
    g = golden("raar64_double")
    o = orc.solve(g["p"], g["m"], int(g["K"]), "double", algorithm="raar", beta=float(g["beta"]))
    np.testing.assert_array_equal(np.array(o["records"]), g["history"])
    np.testing.assert_array_equal(o["u_star"], g["u_star"])


def test_threaded_baseline_matches_serial_oracle():
    p, m = make_problem(128, 8, 7)
    for tag in ("single", "double"):
        t = orc.ThreadedGS(p, m, tag, workers=4)
        try:
            mask = t.run(5)
        finally:
            t.close()
        ref = orc.solve(p, m, 5, tag)["mask"]
        np.testing.assert_array_equal(mask, ref)


def _np_cabs_formula(z):
    """numpy's SIMD complex absolute value (numpy/_core/src/umath/
    loops_unary_complex.dispatch.c.src): larger * sqrt(fma(r, r, 1)),
    r = smaller / larger, with an exact fma (Fraction) and IEEE ops in the
    array's precision. The CUDA path's np_cabs (csrc/pm_fft.cuh) restates it."""
    from fractions import Fraction
    fdt = np.float32 if z.dtype == np.complex64 else np.float64
    out = np.empty(z.shape, fdt)
    for i, v in enumerate(z.ravel()):
        a, b = abs(v.real), abs(v.imag)
        L, S = max(a, b), min(a, b)
        r = fdt(0) if L == 0 else fdt(S / L)              # IEEE division in fdt
        f = fdt(float(Fraction(float(r)) * Fraction(float(r)) + 1))   # fma, one rounding
        out.flat[i] = fdt(np.sqrt(f) * L)
    return out


@pytest.mark.parametrize("dtype", [np.complex64, np.complex128])
def test_numpy_complex_abs_is_the_simd_formula(dtype):
    """The zero-branch decision of the reference is `np.abs(u) >= zero_tol`
    (src/projections.py:49-53); np.abs is this formula, not hypot, bit for bit
    (the GPU decides with the same formula)."""
    rng = np.random.default_rng(11)
    z = (rng.standard_normal(20000) + 1j * rng.standard_normal(20000)).astype(dtype)
    z[::5] *= 1e-4
    z[::7] = z[::7].real.astype(dtype)                    # exact axis values
    z[:4] = [0, 1e-30, 3 + 4j, -2j]
    np.testing.assert_array_equal(np.abs(z), _np_cabs_formula(z))
    # and it is not hypot: some values differ by an ulp
    assert (np.hypot(z.real, z.imag) != np.abs(z)).any()


def test_oracle_divergence_outcomes_match_reference():
    """The reference's outcome (normal return, SolveDivergedError or the
    metrics' ValueError) on amplitudes scaled towards the float range, for
    every case of tests/golden/divergence_outcomes.json (generated by running
    the reference): the oracle reproduces each."""
    import json
    d = json.loads((GOLDEN_DIR / "divergence_outcomes.json").read_text())
    for (n, ny, tag, c, rec, es), want in zip(d["cases"], d["outcomes"]):
        if n > 128:
            continue                                  # the 256^2 cases run on the GPU box (tests/test_gpu_divergence.py)
        p, m = make_problem(n, d["spots"], d["seed"], n_y=ny)
        p = p / p.max() * c
        try:
            with np.errstate(all="ignore"):
                orc.solve(p, m, d["K"], tag, record_every=rec, early_stop_tol=es)
            got = "ok"
        except orc.Diverged as e:
            got = f"div{e.iteration}"
        except ValueError as e:
            got = f"VE:{e}"
        assert got == want, (n, ny, tag, c, rec, es)
