"""GPU: the relaxed variant (RAAR) against the oracle.

The reference has no RAAR; the oracle composes the
reference's own projections with the Luke (2005) update
x+ = b x + b P_S(2v - x) + (1 - 2b) v, v = P_M x, and records the reference's
gap G(x) = ||P_S x - P_M x|| (src/metrics.py:67-71) on the RAAR iterate.
RAAR is chaotic, so the contract is short-horizon:
fp64 field relL2 <= 1e-10 for K <= 20, fp32 <= 1e-4 for K <= 5; gap
history <= 1e-10 relative (fp64, K <= 50) and <= 1e-2 (fp32, K <= 200).
"""

import os

import numpy as np
import pytest

import paper_1302_0120_b200 as pm
from conftest import golden
from oracle import phasemask_oracle as orc
from oracle.phasemask_oracle import relative_l2, weighted_phase_error
from paper_1302_0120_b200.batch import solve_stack
from paper_1302_0120_b200.patterns import make_problem

pytestmark = pytest.mark.gpu

FIELD = {"double": 1e-10, "single": 1e-4}


def gpu(p, m, tag, path=0, **cfg):
    prec = pm.Precision.from_tag(tag)
    ny, nx = p.shape
    spec = pm.GridSpec(nx, ny)
    plan = pm.transform.get_plan(spec, prec)
    plan.set_path(path)
    try:
        return pm.solve(pm.SlmConstraint(pm.RealGrid(spec, p), prec), pm.FourierConstraint(pm.RealGrid(spec, m), prec),
                        pm.SolveConfig(precision=prec, algorithm="raar", **cfg))
    finally:
        plan.set_path(0)


def history(r):
    return np.array([(x.iter, x.gap, x.err_lit, x.err_dark) for x in r.history])


def check_vs(r, o, tag, gap_rtol, field=True):
    assert r.iters_run == o["iters_run"]
    h, oh = history(r), np.array(o["records"], dtype=np.float64)
    assert h.shape == oh.shape
    np.testing.assert_array_equal(h[:, 0], oh[:, 0])
    np.testing.assert_allclose(h[:, 1], oh[:, 1], rtol=gap_rtol, atol=0)
    if field:
        assert relative_l2(r.u_star.data, o["u_star"]) <= FIELD[tag]
        assert relative_l2(r.v_star.data, o["v_star"]) <= FIELD[tag]
        assert weighted_phase_error(r.mask.phases, o["mask"], np.abs(o["u_star"])) <= FIELD[tag]


@pytest.mark.parametrize("name", ["raar64_double", "raar64_single"])
@pytest.mark.parametrize("path", [0, 2])
def test_raar_golden(name, path):
    g = golden(name)
    tag = str(g["precision"])
    r = gpu(g["p"], g["m"], tag, path=path, max_iters=int(g["K"]), beta=float(g["beta"]))
    o = dict(iters_run=int(g["iters_run"]), records=g["history"], u_star=g["u_star"], v_star=g["v_star"],
             mask=g["mask"])
    check_vs(r, o, tag, 1e-10 if tag == "double" else 1e-5)
    np.testing.assert_allclose(history(r)[:, 2:], g["history"][:, 2:], rtol=1e-6, atol=1e-9)


@pytest.mark.parametrize("n,path", [(256, 0), (256, 2), (512, 0)])
def test_raar_fp64_matches_oracle(n, path):
    p, m = make_problem(n, 8, 7)
    K = 20
    r = gpu(p, m, "double", path=path, max_iters=K, beta=0.9)
    o = orc.solve(p, m, K, "double", algorithm="raar", beta=0.9)
    check_vs(r, o, "double", 1e-10)


@pytest.mark.parametrize("n,tag,K", [(2048, "single", 5), (2048, "double", 6)])
def test_raar_large_field_tma_build_matches_oracle(n, tag, K):
    """2048^2 single masks run the persistent kernel's TMA build (column tiles
    and the z' write-back through the tensor accelerator, rows through the
    tile): RAAR against the oracle, short horizon."""
    p, m = make_problem(n, 8, 7)
    r = gpu(p, m, tag, max_iters=K, beta=0.9)
    o = orc.solve(p, m, K, tag, algorithm="raar", beta=0.9, workers=os.cpu_count() or 1)
    check_vs(r, o, tag, 1e-10 if tag == "double" else 1e-5)


def test_raar512_survey_anchor():
    """RAAR 512², 8 spots, fp64, beta 0.9 — gap[1], gap[10], gap[20]."""
    g = golden("raar512_double_anchor")
    p, m = make_problem(512, 8, 7)
    r = gpu(p, m, "double", max_iters=20, beta=0.9)
    gaps = history(r)[:, 1]
    np.testing.assert_allclose(gaps, g["history"][:, 1], rtol=1e-10, atol=0)
    for got, want in zip((gaps[0], gaps[9], gaps[19]), (2.667628112897, 4.536412167171, 4.284140398013)):
        assert got == pytest.approx(want, abs=2e-12)


def test_raar_fp32_short_horizon_and_long_gap():
    p, m = make_problem(512, 8, 7)
    r5 = gpu(p, m, "single", max_iters=5, beta=0.9)
    o5 = orc.solve(p, m, 5, "single", algorithm="raar", beta=0.9)
    check_vs(r5, o5, "single", 1e-5)
    # config 2: 200 iterations, gap history only (chaotic beyond ~20 iterations)
    r = gpu(p, m, "single", max_iters=200, record_every=10, beta=0.9)
    o = orc.solve(p, m, 200, "single", algorithm="raar", beta=0.9, record_every=10)
    check_vs(r, o, "single", 1e-2, field=False)


@pytest.mark.parametrize("path", [0, 2])
def test_raar_record_every_early_stop_and_callbacks(path):
    p, m = make_problem(128, 4, 3)
    o = orc.solve(p, m, 20, "double", algorithm="raar", beta=0.7, record_every=4)
    check_vs(gpu(p, m, "double", path=path, max_iters=20, beta=0.7, record_every=4), o, "double", 1e-10)
    # early stop: every iteration's gap is computed, the loop ends on |dG| <= tol G
    o = orc.solve(p, m, 200, "double", algorithm="raar", beta=0.6, early_stop_tol=1e-3)
    r = gpu(p, m, "double", path=path, max_iters=200, beta=0.6, early_stop_tol=1e-3)
    assert o["iters_run"] < 200
    check_vs(r, o, "double", 1e-9, field=o["iters_run"] <= 20)
    # the stepped (callback) solve produces the same records and pair
    seen = []
    spec = pm.GridSpec(128, 128)
    plan = pm.transform.get_plan(spec, pm.DOUBLE)
    plan.set_path(path)
    try:
        rc = pm.solve(pm.SlmConstraint(pm.RealGrid(spec, p)), pm.FourierConstraint(pm.RealGrid(spec, m)),
                      pm.SolveConfig(max_iters=12, algorithm="raar", beta=0.8, record_every=2),
                      on_record=seen.append)
        rn = pm.solve(pm.SlmConstraint(pm.RealGrid(spec, p)), pm.FourierConstraint(pm.RealGrid(spec, m)),
                      pm.SolveConfig(max_iters=12, algorithm="raar", beta=0.8, record_every=2))
    finally:
        plan.set_path(0)
    assert [x.iter for x in seen] == [1, 3, 5, 7, 9, 11]
    assert [x.gap for x in seen] == [x.gap for x in rn.history]
    np.testing.assert_array_equal(rc.u_star.data, rn.u_star.data)


def test_raar_abort_after_three_polls():
    p, m = make_problem(128, 4, 3)
    polls = []

    def abort():
        polls.append(1)
        return len(polls) >= 3

    spec = pm.GridSpec(128, 128)
    r = pm.solve(pm.SlmConstraint(pm.RealGrid(spec, p)), pm.FourierConstraint(pm.RealGrid(spec, m)),
                 pm.SolveConfig(max_iters=50, algorithm="raar", beta=0.9), should_abort=abort)
    o = orc.solve(p, m, 3, "double", algorithm="raar", beta=0.9)
    assert r.aborted and r.iters_run == 3
    check_vs(r, o, "double", 1e-10)


def test_raar_batch_is_bitwise_per_mask():
    p = make_problem(256, 8, 7)[0]
    ms = np.stack([make_problem(256, 8, s)[1] for s in (11, 12, 13)])
    cfg = pm.SolveConfig(max_iters=15, algorithm="raar", beta=0.9, precision=pm.SINGLE, record_every=5)
    res = solve_stack(p.astype(np.float32), ms.astype(np.float32), cfg)
    spec = pm.GridSpec(256, 256)
    for i in range(3):
        r = pm.solve(pm.SlmConstraint(pm.RealGrid(spec, p), pm.SINGLE),
                     pm.FourierConstraint(pm.RealGrid(spec, ms[i]), pm.SINGLE), cfg)
        np.testing.assert_array_equal(r.mask.phases, res.phases[i])
        assert [x.gap for x in r.history] == list(res.gap[i][~np.isnan(res.gap[i])])


def test_raar_is_deterministic():
    p, m = make_problem(512, 8, 7)
    a = gpu(p, m, "single", max_iters=30, beta=0.9)
    b = gpu(p, m, "single", max_iters=30, beta=0.9)
    np.testing.assert_array_equal(a.mask.phases, b.mask.phases)
    assert [x.gap for x in a.history] == [x.gap for x in b.history]


# --- mixed-radix grids (pm_generic.cuh: alternating iterate buffers) --------

@pytest.mark.parametrize("nx,ny", [(60, 42), (100, 64), (120, 90)])
def test_raar_mixed_radix_fp64_matches_oracle(nx, ny):
    p, m = make_problem(nx, 6, 5, n_y=ny)
    o = orc.solve(p, m, 20, "double", algorithm="raar", beta=0.9, record_every=3)
    check_vs(gpu(p, m, "double", max_iters=20, beta=0.9, record_every=3), o, "double", 1e-10)


def test_raar_mixed_radix_fp32_paper_grid():
    p, m = make_problem(800, 12, 7, n_y=600)
    o = orc.solve(p, m, 5, "single", algorithm="raar", beta=0.9)
    check_vs(gpu(p, m, "single", max_iters=5, beta=0.9), o, "single", 1e-5)


def test_raar_mixed_radix_early_stop_callbacks_abort_and_batch():
    p, m = make_problem(120, 6, 3, n_y=90)
    spec = pm.GridSpec(120, 90)
    c, mc = pm.SlmConstraint(pm.RealGrid(spec, p)), pm.FourierConstraint(pm.RealGrid(spec, m))
    # early stop on an odd and an even iterate (the two iterate buffers)
    for tol in (1e-3, 3e-3):
        o = orc.solve(p, m, 200, "double", algorithm="raar", beta=0.6, early_stop_tol=tol)
        r = pm.solve(c, mc, pm.SolveConfig(max_iters=200, algorithm="raar", beta=0.6, early_stop_tol=tol))
        assert o["iters_run"] < 200
        check_vs(r, o, "double", 1e-9, field=o["iters_run"] <= 20)
    # stepped solve (callbacks) == one-shot solve
    seen = []
    cfg = pm.SolveConfig(max_iters=11, algorithm="raar", beta=0.8, record_every=2)
    rc = pm.solve(c, mc, cfg, on_record=seen.append)
    rn = pm.solve(c, mc, cfg)
    assert [x.iter for x in seen] == [1, 3, 5, 7, 9, 11]
    assert [x.gap for x in seen] == [x.gap for x in rn.history]
    np.testing.assert_array_equal(rc.u_star.data, rn.u_star.data)
    # abort after three polls: the pair comes from x_3 (odd: second buffer)
    polls = []

    def abort():
        polls.append(1)
        return len(polls) >= 3

    ra = pm.solve(c, mc, pm.SolveConfig(max_iters=50, algorithm="raar", beta=0.9), should_abort=abort)
    o = orc.solve(p, m, 3, "double", algorithm="raar", beta=0.9)
    assert ra.aborted and ra.iters_run == 3
    check_vs(ra, o, "double", 1e-10)
    # a batch equals its single solves bitwise
    ms = np.stack([make_problem(120, 6, s, n_y=90)[1] for s in (3, 4)])
    res = solve_stack(p, ms, cfg)
    np.testing.assert_array_equal(res.phases[0], rn.mask.phases)

