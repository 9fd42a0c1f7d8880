"""GPU parity: the CUDA solve against the reference's own outputs.

Fixtures come from running the reference (tests/golden/make_golden.py).
Tolerances: fp64 field relL2 <= 1e-10 and gap history
<= 1e-12 relative; fp32 (vs the reference in SINGLE mode) field relL2 <= 1e-4,
mask amplitude-weighted RMS phase error <= 1e-4 rad, gap <= 1e-6 relative.
Both execution paths (persistent cooperative kernel, sweep-per-kernel graph)
are checked where the grid admits both.
"""

import numpy as np
import pytest

import paper_1302_0120_b200 as pm
from conftest import golden
from oracle.phasemask_oracle import relative_l2, weighted_phase_error

pytestmark = pytest.mark.gpu

TOL = {"double": dict(field=1e-10, gap=1e-12, phase=1e-10, err=1e-9),
       "single": dict(field=1e-4, gap=1e-6, phase=1e-4, err=1e-5)}

FIXTURES = ["gs16_double", "gs32_single", "gs64_double", "gs64x32_double", "gs64_single_rec3",
            "gs128_double_early", "gs32_double_randinit", "gs256_double", "gs256_single", "lattice64_double"]


def run(g, path=0):
    tag = str(g["precision"])
    prec = pm.Precision.from_tag(tag)
    ny, nx = g["p"].shape
    spec = pm.GridSpec(nx, ny)
    kw = {}
    if "record_every" in g:
        kw["record_every"] = int(g["record_every"])
    if "early_stop_tol" in g and float(g["early_stop_tol"]) >= 0:
        kw["early_stop_tol"] = float(g["early_stop_tol"])
    if "random_phase_init" in g and int(g["random_phase_init"]):
        kw.update(random_phase_init=True, seed=int(g["seed"]))
    plan = pm.transform.get_plan(spec, prec)
    plan.set_path(path)
    try:
        return pm.solve(pm.SlmConstraint(pm.RealGrid(spec, g["p"]), prec),
                        pm.FourierConstraint(pm.RealGrid(spec, g["m"]), prec),
                        pm.SolveConfig(max_iters=int(g["K"]), precision=prec, **kw))
    finally:
        plan.set_path(0)


def check(g, r):
    tag = str(g["precision"])
    t = TOL[tag]
    assert r.iters_run == int(g["iters_run"])
    assert relative_l2(r.u_star.data, g["u_star"]) <= t["field"]
    assert relative_l2(r.v_star.data, g["v_star"]) <= t["field"]
    assert weighted_phase_error(r.mask.phases, g["mask"], g["p"]) <= t["phase"]
    h = np.array([(x.iter, x.gap, x.err_lit, x.err_dark) for x in r.history])
    assert h.shape == g["history"].shape
    np.testing.assert_array_equal(h[:, 0], g["history"][:, 0])
    np.testing.assert_allclose(h[:, 1], g["history"][:, 1], rtol=t["gap"], atol=0)
    np.testing.assert_allclose(h[:, 2:], g["history"][:, 2:], rtol=t["err"], atol=t["err"] * 1e-3)
    assert r.u_star.dtype == pm.Precision.from_tag(tag).complex_dtype


@pytest.mark.parametrize("name", FIXTURES)
def test_solve_matches_reference(name):
    g = golden(name)
    check(g, run(g))


@pytest.mark.parametrize("name", ["gs256_double", "gs256_single", "gs128_double_early", "lattice64_double"])
def test_sweep_graph_path_matches_reference(name):
    g = golden(name)
    check(g, run(g, path=2))


@pytest.mark.parametrize("tag", ["double", "single"])
def test_per_iteration_iterates(tag):
    g = golden(f"iterates64_{tag}")
    spec = pm.GridSpec(64, 64)
    prec = pm.Precision.from_tag(tag)
    for K, u in zip(g["Ks"], g["u_star"]):
        r = pm.solve(pm.SlmConstraint(pm.RealGrid(spec, g["p"]), prec),
                     pm.FourierConstraint(pm.RealGrid(spec, g["m"]), prec),
                     pm.SolveConfig(max_iters=int(K), precision=prec))
        assert relative_l2(r.u_star.data, u) <= TOL[tag]["field"], K


@pytest.mark.parametrize("name", ["anchor512_double", "anchor1024_single", "anchor1024_double"])
def test_large_anchor_histories(name):
    from paper_1302_0120_b200.patterns import make_problem
    g = golden(name)
    tag = str(g["precision"])
    n = int(g["n"])
    p, m = make_problem(n, int(g["spots"]), int(g["seed"]))
    prec = pm.Precision.from_tag(tag)
    spec = pm.GridSpec(n, n)
    r = pm.solve(pm.SlmConstraint(pm.RealGrid(spec, p), prec), pm.FourierConstraint(pm.RealGrid(spec, m), prec),
                 pm.SolveConfig(max_iters=int(g["K"]), precision=prec))
    gaps = np.array([x.gap for x in r.history])
    np.testing.assert_allclose(gaps, g["history"][:, 1], rtol=TOL[tag]["gap"], atol=0)
    ph = r.mask.phases
    d = np.angle(np.exp(1j * (ph[::64, ::64] - g["mask_sample"])))
    assert np.sqrt(np.mean(d * d)) <= (1e-9 if tag == "double" else 1e-3)


def test_survey_anchor_values():
    """SURVEY.md §8c quotes gap[1], gap[2], gap[10], gap[K] to 13 digits."""
    from paper_1302_0120_b200.patterns import make_problem
    p, m = make_problem(256, 8, 7)
    spec = pm.GridSpec(256, 256)
    r = pm.solve(pm.SlmConstraint(pm.RealGrid(spec, p)), pm.FourierConstraint(pm.RealGrid(spec, m)),
                 pm.SolveConfig(max_iters=100))
    g = [x.gap for x in r.history]
    for got, want in zip((g[0], g[1], g[9], g[-1]),
                         (2.667285880343, 2.667285852468, 2.667285704702, 2.667269502141)):
        assert got == pytest.approx(want, abs=2e-12)
