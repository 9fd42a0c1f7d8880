"""GPU: solver contracts, determinism, callbacks, batches, large grids
(reference tests/test_solver.py and tests/test_acceptance.py, re-pointed)."""

import math

import numpy as np
import pytest

import paper_1302_0120_b200 as pm
from oracle import phasemask_oracle as orc
from paper_1302_0120_b200.batch import solve_batch, solve_stack
from paper_1302_0120_b200.patterns import (make_problem, modulus_from_intensity, spot_grid_centers,
                                           spot_pattern, to_fourier_order)
from paper_1302_0120_b200.projections import project_fourier, project_slm

pytestmark = pytest.mark.gpu
EPS = np.finfo(float).eps


def spot_problem(n, precision=pm.DOUBLE):
    """The reference's default fixture: 3x3 lattice, energy-matched uniform p."""
    spec = pm.GridSpec(n, n)
    inten = spot_pattern(spec, spot_grid_centers(spec))
    m = pm.FourierConstraint(modulus_from_intensity(to_fourier_order(inten)), precision)
    c = pm.SlmConstraint(pm.default_amplitude(m.m, precision), precision)
    return spec, c, m, inten


def problem(n, tag="double", spots=8, seed=7):
    prec = pm.Precision.from_tag(tag)
    p, m = make_problem(n, spots, seed)
    spec = pm.GridSpec(n, n)
    return spec, pm.SlmConstraint(pm.RealGrid(spec, p), prec), pm.FourierConstraint(pm.RealGrid(spec, m), prec)


def test_initial_iterate_matches_naive_oracle():
    spec = pm.GridSpec(32, 32)
    md = np.zeros(spec.shape)
    for j, k in ((4, 4), (12, 20), (28, 8)):
        md[k, j] = 1.0
    u = pm.initial_iterate(pm.FourierConstraint(pm.RealGrid(spec, md)), pm.FftProvider(spec))
    assert np.abs(u.data - orc.naive_dft(md.astype(complex), "inverse")).max() < 1e-12
    a = pm.initial_iterate(pm.FourierConstraint(pm.RealGrid(spec, md)), pm.FftProvider(spec), True, 3)
    b = pm.initial_iterate(pm.FourierConstraint(pm.RealGrid(spec, md)), pm.FftProvider(spec), True, 3)
    np.testing.assert_array_equal(a.data, b.data)


def test_single_iteration_pair_matches_composition():
    spec, c, m, _ = spot_problem(32)
    prov = pm.FftProvider(spec)
    r = pm.solve(c, m, pm.SolveConfig(max_iters=1), prov)
    assert r.iters_run == 1 and len(r.history) == 1
    u0 = pm.initial_iterate(m, prov)
    u1 = project_slm(project_fourier(u0, m, prov), c)
    v_star = project_fourier(u1, m, prov)
    u_star = project_slm(v_star, c)
    assert np.abs(r.u_star.data - u_star.data).max() <= 1e-12
    d = np.angle(np.exp(1j * (r.mask.phases - pm.phases_of(u_star, c.zero_tol).phases)))
    assert np.abs(d).max() <= 1e-10


def test_history_length_with_record_every():
    spec, c, m, _ = spot_problem(32)
    r = pm.solve(c, m, pm.SolveConfig(max_iters=25, record_every=2))
    assert len(r.history) == 13
    assert [h.iter for h in r.history][:3] == [1, 3, 5]


def test_iterates_feasible():
    spec, c, m, _ = spot_problem(32)
    prov = pm.FftProvider(spec)
    r = pm.solve(c, m, pm.SolveConfig(max_iters=10), prov)
    p = c.p.data
    assert np.abs(np.abs(r.u_star.data) - p).max() <= 4 * EPS * p.max()
    assert np.linalg.norm(r.u_star.data) == pytest.approx(np.linalg.norm(p), rel=16 * EPS)
    mods = np.abs(prov.forward(r.v_star).data)
    assert np.abs(mods - m.m.data).max() <= 32 * EPS * max(1, m.m.data.max())


def test_gap_sequence_non_increasing_fp64():
    for spec, c, m in (spot_problem(64)[:3], problem(128)):
        gaps = [h.gap for h in pm.solve(c, m, pm.SolveConfig(max_iters=25)).history]
        jitter = 4 * EPS * gaps[0]
        assert all(b <= a + jitter for a, b in zip(gaps, gaps[1:]))


def test_rejections():
    spec, c, m, _ = spot_problem(16)
    with pytest.raises(ValueError, match="identically zero"):
        pm.solve(pm.SlmConstraint(pm.RealGrid(spec, np.zeros(spec.shape))), m, pm.SolveConfig(max_iters=1))
    with pytest.raises(ValueError, match="all dark"):
        pm.solve(c, pm.FourierConstraint(pm.RealGrid(spec, np.zeros(spec.shape))), pm.SolveConfig(max_iters=1))


def test_early_stop():
    spec, c, m, _ = spot_problem(64)
    r = pm.solve(c, m, pm.SolveConfig(max_iters=200, early_stop_tol=1e-6))
    assert r.iters_run < 200


def test_abort_callback_and_on_record():
    spec, c, m, _ = spot_problem(32)
    calls, records = [], []

    def should_abort():
        calls.append(1)
        return len(calls) >= 3

    r = pm.solve(c, m, pm.SolveConfig(max_iters=50), on_record=records.append, should_abort=should_abort)
    assert r.aborted and r.iters_run == 3
    assert [x.iter for x in records] == [1, 2, 3]
    full = pm.solve(c, m, pm.SolveConfig(max_iters=3))
    assert [x.gap for x in records] == [x.gap for x in full.history]
    np.testing.assert_array_equal(r.mask.phases, full.mask.phases)


@pytest.mark.parametrize("path", [1, 2])
def test_identical_runs_bitwise(path):
    spec, c, m = problem(128)
    plan = pm.transform.get_plan(spec, pm.DOUBLE)
    plan.set_path(path)
    try:
        a = pm.solve(c, m, pm.SolveConfig(max_iters=10))
        b = pm.solve(c, m, pm.SolveConfig(max_iters=10))
    finally:
        plan.set_path(0)
    np.testing.assert_array_equal(a.mask.phases, b.mask.phases)
    assert [r.gap for r in a.history] == [r.gap for r in b.history]


def test_transposed_m_column_staging_matches_sweep_path():
    """2048^2 fp32: the persistent kernel stages m from a transposed copy
    (one contiguous run per column task); the sweep path reads m row-major.
    Same iterates to fp32 tolerance, same gap history."""
    spec, c, m = problem(2048, "single", spots=50)
    plan = pm.transform.get_plan(spec, pm.SINGLE)
    cfg = pm.SolveConfig(max_iters=8, precision=pm.SINGLE)
    a = pm.solve(c, m, cfg)
    plan.set_path(2)
    try:
        b = pm.solve(c, m, cfg)
    finally:
        plan.set_path(0)
    assert orc.relative_l2(a.u_star.data, b.u_star.data) <= 1e-5
    np.testing.assert_allclose([r.gap for r in a.history], [r.gap for r in b.history], rtol=1e-6)
    np.testing.assert_allclose([r.err_lit for r in a.history], [r.err_lit for r in b.history], rtol=1e-5)
    # the stepping API (callbacks) keeps the transposed copy across its launches
    seen = []
    c3 = pm.SolveConfig(max_iters=3, precision=pm.SINGLE)
    stepped = pm.solve(c, m, c3, on_record=seen.append)
    whole = pm.solve(c, m, c3)
    assert [x.gap for x in seen] == [x.gap for x in whole.history]
    np.testing.assert_array_equal(stepped.mask.phases, whole.mask.phases)


def test_backend_selector_does_not_change_results():
    spec, c, m, _ = spot_problem(64)
    a = pm.solve(c, m, pm.SolveConfig(max_iters=10, backend=pm.BackendSelector("serial")))
    b = pm.solve(c, m, pm.SolveConfig(max_iters=10, backend=pm.BackendSelector("threaded", 8)))
    np.testing.assert_array_equal(a.mask.phases, b.mask.phases)
    assert [(r.gap, r.err_lit, r.err_dark) for r in a.history] == [(r.gap, r.err_lit, r.err_dark) for r in b.history]


def test_single_precision_stays_single():
    spec, c, m, _ = spot_problem(64, pm.SINGLE)
    r = pm.solve(c, m, pm.SolveConfig(max_iters=3, precision=pm.SINGLE))
    assert r.u_star.dtype == np.complex64 and r.v_star.dtype == np.complex64


@pytest.mark.parametrize("tag", ["double", "single"])
def test_batch_is_bitwise_independent_of_batch_size(tag):
    prec = pm.Precision.from_tag(tag)
    p, _ = make_problem(128, 8, 7)
    ms = np.stack([make_problem(128, 8, s)[1] for s in (11, 12, 13)])
    cfg = pm.SolveConfig(max_iters=12, precision=prec, record_every=1)
    whole = solve_stack(p, ms, cfg)
    for i in range(3):
        one = solve_stack(p, ms[i:i + 1], cfg)
        np.testing.assert_array_equal(whole.phases[i], one.phases[0])
        np.testing.assert_array_equal(whole.gap[i], one.gap[0])
    spec = pm.GridSpec(128, 128)
    r = pm.solve(pm.SlmConstraint(pm.RealGrid(spec, p), prec), pm.FourierConstraint(pm.RealGrid(spec, ms[1]), prec),
                 cfg)
    np.testing.assert_array_equal(r.mask.phases, whole.phases[1])
    assert [h.gap for h in r.history] == list(whole.gap[1])
    multi = solve_batch(p, ms, cfg)
    np.testing.assert_array_equal(multi.phases, whole.phases)


def test_batch_per_mask_amplitude_and_early_stop():
    ps = np.stack([make_problem(64, 4, s)[0] for s in (1, 2)])
    ms = np.stack([make_problem(64, 4, s)[1] for s in (1, 2)])
    cfg = pm.SolveConfig(max_iters=60, early_stop_tol=1e-7)
    res = solve_stack(ps, ms, cfg)
    for i in range(2):
        spec = pm.GridSpec(64, 64)
        r = pm.solve(pm.SlmConstraint(pm.RealGrid(spec, ps[i])), pm.FourierConstraint(pm.RealGrid(spec, ms[i])), cfg)
        assert r.iters_run == res.iters_run[i]
        np.testing.assert_array_equal(r.mask.phases, res.phases[i])


@pytest.mark.parametrize("tag", ["double", "single"])
def test_device_slm_levels_match_to_uint8(tag):
    """uint8 levels computed on the device equal PhaseMask.to_uint8 of the
    float64 mask bitwise (reference src/grid.py:152-154)."""
    prec = pm.Precision.from_tag(tag)
    p, _ = make_problem(256, 8, 7)
    ms = np.stack([make_problem(256, 8, s)[1] for s in (3, 4)])
    res = solve_stack(p.astype(prec.float_dtype), ms.astype(prec.float_dtype),
                      pm.SolveConfig(max_iters=20, precision=prec), levels=True)
    spec = pm.GridSpec(256, 256)
    for i in range(2):
        np.testing.assert_array_equal(res.levels[i], pm.PhaseMask(spec, res.phases[i]).to_uint8())
    assert res.levels.dtype == np.uint8 and res.levels.max() <= 255


@pytest.mark.slow
@pytest.mark.parametrize("n", [2048, 4096])
def test_large_field_properties(n):
    """Size-independent properties at BASELINE config 5 sizes (fp32)."""
    spec, c, m = problem(n, "single", spots=50)
    prov = pm.FftProvider(spec, pm.SINGLE)
    r = pm.solve(c, m, pm.SolveConfig(max_iters=20, precision=pm.SINGLE, record_every=5))
    p = c.p.data
    assert np.abs(np.abs(r.u_star.data) - p).max() <= 8 * np.finfo(np.float32).eps * p.max()
    mods = np.abs(prov.forward(r.v_star).data)
    assert np.abs(mods - m.m.data).max() <= 1e-4 * max(1.0, m.m.data.max())
    gaps = [h.gap for h in r.history]
    assert all(np.isfinite(gaps)) and gaps[-1] <= gaps[0] * (1 + 1e-5)
    assert ((r.mask.phases >= 0) & (r.mask.phases < 2 * np.pi)).all()


# --- acceptance criteria of the reference (tests/test_acceptance.py) --------

def test_acceptance_1_oracle_equivalence():
    rng = np.random.default_rng(101)
    worst = 0.0
    for n in (8, 16):
        spec = pm.GridSpec(n, n)
        prov = pm.FftProvider(spec)
        for _ in range(50):
            u = rng.standard_normal(spec.shape) + 1j * rng.standard_normal(spec.shape)
            m = rng.uniform(0, 2, spec.shape)
            got = project_fourier(pm.Field(spec, u), pm.FourierConstraint(pm.RealGrid(spec, m)), prov).data
            vhat = orc.replace_modulus(orc.naive_dft(u), m, orc.zero_tol("double", m), "double")
            worst = max(worst, float(np.abs(got - orc.naive_dft(vhat, "inverse")).max()))
    assert worst <= 1e-12


def _spot_gaps():
    _, cd, md, _ = spot_problem(256, pm.DOUBLE)
    _, cs, ms, _ = spot_problem(256, pm.SINGLE)
    gd = pm.solve(cd, md, pm.SolveConfig(max_iters=25, record_every=25)).final.gap
    gs = pm.solve(cs, ms, pm.SolveConfig(max_iters=25, record_every=25, precision=pm.SINGLE)).final.gap
    return gd, gs


def test_acceptance_3_and_6_inconsistency_and_precision_agreement():
    gd, gs = _spot_gaps()
    assert gd > 1e6 * EPS and 0.1 <= gs / gd <= 10.0
    assert abs(gs - gd) / gd <= 0.05


def test_acceptance_4_saturation():
    _, c, m, _ = spot_problem(256)
    r = pm.solve(c, m, pm.SolveConfig(max_iters=25))
    by = {h.iter: h for h in r.history}
    e2, e25 = by[2].err_lit + by[2].err_dark, by[25].err_lit + by[25].err_dark
    assert abs(e2 - e25) <= 0.05 * e25
    assert abs(by[2].gap - by[25].gap) <= 0.05 * by[25].gap


def test_acceptance_5_contrast():
    from paper_1302_0120_b200.metrics import contrast_ratio, reconstructed_intensity
    spec, c, m, _ = spot_problem(256)
    prov = pm.FftProvider(spec)
    r = pm.solve(c, m, pm.SolveConfig(max_iters=25, record_every=25), prov)
    target = pm.RealGrid(spec, m.m.data ** 2)
    recon = reconstructed_intensity(r.u_star, prov, float(target.data.sum()))
    assert contrast_ratio(recon, target) >= 1e2


def test_acceptance_8_performance_recorded_and_target():
    """Criterion 8 on the GPU (tests/test_acceptance.py:170-207): the 800x600
    single-precision ms/iter is recorded (not gated); the north-star target of
    a 1024^2 fp32 mask with 100 iterations well under 10 ms is gated."""
    p, m = make_problem(800, 12, 7, n_y=600)
    spec = pm.GridSpec(800, 600)
    cfg = pm.SolveConfig(max_iters=10, precision=pm.SINGLE, record_every=10)
    c, mc = pm.SlmConstraint(pm.RealGrid(spec, p), pm.SINGLE), pm.FourierConstraint(pm.RealGrid(spec, m), pm.SINGLE)
    pm.solve(c, mc, cfg)
    r = pm.solve(c, mc, cfg)
    assert r.timing.per_iter_ms > 0
    print(f"800x600 single {r.timing.per_iter_ms:.4f} ms/iter recorded, not gated")
    p, m = make_problem(1024, 50, 7)
    spec = pm.GridSpec(1024, 1024)
    cfg = pm.SolveConfig(max_iters=100, precision=pm.SINGLE, record_every=100)
    c, mc = pm.SlmConstraint(pm.RealGrid(spec, p), pm.SINGLE), pm.FourierConstraint(pm.RealGrid(spec, m), pm.SINGLE)
    pm.solve(c, mc, cfg)
    best = min(pm.solve(c, mc, cfg).timing.fft_ms for _ in range(3))
    assert best < 10.0, best


@pytest.mark.xfail(reason="known-red in the reference too: AP from the default init does not reach "
                          "sqrt(N)*100*eps on consistent problems (reference README, tests/test_solver.py:170)",
                   strict=False)
def test_acceptance_2_consistency_collapse():
    spec = pm.GridSpec(64, 64)
    prov = pm.FftProvider(spec)
    c = pm.SlmConstraint(pm.RealGrid(spec, np.ones(spec.shape)))
    rng = np.random.default_rng(2024)
    w = pm.Field(spec, np.exp(1j * rng.uniform(0, 2 * np.pi, spec.shape)))
    m = pm.FourierConstraint(pm.RealGrid(spec, np.abs(prov.forward(w).data)))
    r = pm.solve(c, m, pm.SolveConfig(max_iters=50, record_every=50), prov)
    assert r.final.gap <= math.sqrt(spec.n) * 100 * EPS


@pytest.mark.parametrize("nx,ny,tag,K", [(800, 600, "single", 25), (60, 42, "double", 30), (100, 64, "double", 20)])
def test_mixed_radix_solve_matches_oracle(nx, ny, tag, K):
    """Non-power-of-two grids (the paper's 800x600 SLM) on the
    mixed-radix path: GS against the oracle restatement of the reference."""
    prec = pm.Precision.from_tag(tag)
    p, m = make_problem(nx, 12, 7, n_y=ny)
    spec = pm.GridSpec(nx, ny)
    r = pm.solve(pm.SlmConstraint(pm.RealGrid(spec, p), prec), pm.FourierConstraint(pm.RealGrid(spec, m), prec),
                 pm.SolveConfig(max_iters=K, precision=prec, record_every=5))
    o = orc.solve(p, m, K, tag, record_every=5)
    tol = 1e-10 if tag == "double" else 1e-4
    assert r.iters_run == o["iters_run"]
    assert orc.relative_l2(r.u_star.data, o["u_star"]) <= tol
    assert orc.relative_l2(r.v_star.data, o["v_star"]) <= tol
    h = np.array([(x.iter, x.gap, x.err_lit, x.err_dark) for x in r.history])
    oh = np.array(o["records"])
    np.testing.assert_array_equal(h[:, 0], oh[:, 0])
    np.testing.assert_allclose(h[:, 1], oh[:, 1], rtol=1e-12 if tag == "double" else 1e-6)
    np.testing.assert_allclose(h[:, 2:], oh[:, 2:], rtol=1e-6, atol=1e-9)


def test_mixed_radix_early_stop_callbacks_and_batch():
    p, m = make_problem(120, 6, 3, n_y=90)
    spec = pm.GridSpec(120, 90)
    c, mc = pm.SlmConstraint(pm.RealGrid(spec, p)), pm.FourierConstraint(pm.RealGrid(spec, m))
    o = orc.solve(p, m, 300, "double", early_stop_tol=1e-6)
    r = pm.solve(c, mc, pm.SolveConfig(max_iters=300, early_stop_tol=1e-6))
    assert r.iters_run == o["iters_run"] < 300
    assert orc.relative_l2(r.u_star.data, o["u_star"]) <= 1e-10
    seen = []
    rc = pm.solve(c, mc, pm.SolveConfig(max_iters=9, record_every=4), on_record=seen.append)
    rn = pm.solve(c, mc, pm.SolveConfig(max_iters=9, record_every=4))
    assert [x.iter for x in seen] == [1, 5, 9] and [x.gap for x in seen] == [x.gap for x in rn.history]
    np.testing.assert_array_equal(rc.mask.phases, rn.mask.phases)
    ms = np.stack([make_problem(120, 6, s, n_y=90)[1] for s in (3, 4)])
    res = solve_stack(p, ms, pm.SolveConfig(max_iters=9, record_every=4))
    np.testing.assert_array_equal(res.phases[0], rn.mask.phases)


def test_batch_device_tolerances_match_host_and_reject_zero_inputs():
    """solve_stack derives the zero tolerances on the device; results equal a
    solve with host-computed tolerances bitwise, and identically zero inputs
    raise the reference's messages (src/solver.py:122-125)."""
    for tag in ("single", "double"):
        prec = pm.Precision.from_tag(tag)
        p, m = make_problem(256, 8, 7)
        spec = pm.GridSpec(256, 256)
        cfg = pm.SolveConfig(max_iters=15, precision=prec, record_every=5)
        r = pm.solve(pm.SlmConstraint(pm.RealGrid(spec, p), prec), pm.FourierConstraint(pm.RealGrid(spec, m), prec), cfg)
        res = solve_stack(p.astype(prec.float_dtype), m[None].astype(prec.float_dtype), cfg)
        np.testing.assert_array_equal(res.phases[0], r.mask.phases)
        assert [x.gap for x in r.history] == list(res.gap[0][~np.isnan(res.gap[0])])
    p, m = make_problem(128, 4, 3)
    ms = np.stack([m, np.zeros_like(m)])
    with pytest.raises(ValueError, match="all dark"):
        solve_stack(p, ms, pm.SolveConfig(max_iters=3))
    with pytest.raises(ValueError, match="identically zero"):
        solve_stack(np.zeros_like(p), m[None], pm.SolveConfig(max_iters=3))


@pytest.mark.parametrize("n,tag,algo,B", [(1024, "single", "gs", 4), (512, "double", "gs", 6), (256, "single", "gs", 24),
                                          (512, "single", "raar", 5), (2048, "single", "gs", 2),
                                          (2048, "single", "raar", 2), (2048, "double", "gs", 2),
                                          (4096, "single", "gs", 2)])
def test_tma_batch_variant_is_bitwise_equal_to_single_solves(n, tag, algo, B):
    """Batches large enough to give every CTA several column tasks run the
    persistent kernel's TMA variant (tiles streamed by the tensor memory
    accelerator); each mask must equal its own single-mask solve bitwise,
    early stopping included. At 2048^2 / 4096^2 both run the TMA build
    (one-box column tiles, tensor stores of z', row copies through the tile)."""
    prec = pm.Precision.from_tag(tag)
    p, _ = make_problem(n, 8, 7)
    ms = np.stack([make_problem(n, 8, s)[1] for s in range(20, 20 + B)])
    cfg = pm.SolveConfig(max_iters=9, precision=prec, record_every=3, algorithm=algo,
                         early_stop_tol=1e-9 if algo == "gs" else None)
    whole = solve_stack(p.astype(prec.float_dtype), ms.astype(prec.float_dtype), cfg)
    spec = pm.GridSpec(n, n)
    for i in (0, B - 1):
        r = pm.solve(pm.SlmConstraint(pm.RealGrid(spec, p), prec),
                     pm.FourierConstraint(pm.RealGrid(spec, ms[i]), prec), cfg)
        np.testing.assert_array_equal(r.mask.phases, whole.phases[i])
        assert r.iters_run == whole.iters_run[i]
        assert [h.gap for h in r.history] == list(whole.gap[i][~np.isnan(whole.gap[i])])


def test_solve_stream_matches_solve_stack_frame_by_frame():
    """batch.solve_stream (pipelined frames: uploads / downloads overlap the
    solves) returns every frame's solve_stack result bitwise, in order."""
    import torch
    from paper_1302_0120_b200.batch import solve_stream
    p, _ = make_problem(256, 8, 7)
    ms = [make_problem(256, 8, s)[1] for s in (21, 22, 23, 24, 25)]
    cfg = pm.SolveConfig(max_iters=12, precision=pm.SINGLE, record_every=3)
    outs = [torch.empty((1, 256, 256), dtype=torch.float64).pin_memory().numpy() for _ in range(2)]
    for out_phases in (None, outs):
        got = []
        for r in solve_stream(((p, m) for m in ms), cfg, out_phases=out_phases):
            got.append((r.phases.copy(), r.gap.copy(), r.iters_run.copy()))
        assert len(got) == len(ms)
        for (ph, gap, its), m in zip(got, ms):
            ref = solve_stack(p.astype(np.float32), m[None].astype(np.float32), cfg)
            np.testing.assert_array_equal(ph, ref.phases)
            np.testing.assert_array_equal(gap, ref.gap)
            assert its[0] == ref.iters_run[0] == 12
    assert list(solve_stream(iter(()), cfg)) == []
    with pytest.raises(ValueError, match="different grids"):
        list(solve_stream([(p, ms[0]), (p, ms[1][:128])], cfg))


def test_solve_stream_mixed_radix_raar_and_random_start():
    """solve_stream on the mixed-radix path, with RAAR and a seeded random
    start drawn on the device: each frame equals its solve_stack result."""
    from paper_1302_0120_b200.batch import solve_stream
    p, _ = make_problem(120, 6, 3, n_y=90)
    ms = [make_problem(120, 6, s, n_y=90)[1] for s in (5, 6, 7)]
    for cfg in (pm.SolveConfig(max_iters=9, algorithm="raar", beta=0.8, record_every=2),
                pm.SolveConfig(max_iters=9, random_phase_init=True, seed=4, record_every=3)):
        got = [(r.phases.copy(), r.gap.copy()) for r in solve_stream(((p, m) for m in ms), cfg)]
        for (ph, gap), m in zip(got, ms):
            ref = solve_stack(p, m[None], cfg)
            np.testing.assert_array_equal(ph, ref.phases)
            np.testing.assert_array_equal(gap, ref.gap)


def test_solve_stream_consumer_may_stop_early():
    """Breaking out of a solve_stream loop leaves the plan usable (the
    generator's cleanup waits for the copies in flight)."""
    from paper_1302_0120_b200.batch import solve_stream
    p, _ = make_problem(256, 8, 7)
    ms = [make_problem(256, 8, s)[1] for s in (31, 32, 33, 34)]
    cfg = pm.SolveConfig(max_iters=6, precision=pm.SINGLE)
    for i, r in enumerate(solve_stream(((p, m) for m in ms), cfg)):
        if i == 1:
            break
    ref = solve_stack(p.astype(np.float32), ms[2][None].astype(np.float32), cfg)
    again = next(iter(solve_stream([(p, ms[2])], cfg)))
    np.testing.assert_array_equal(again.phases, ref.phases)
