"""CPU: the host layer's contracts that do not touch the device.

Validation, messages and exception types follow the reference
(src/solver.py:35-53,111-125; src/grid.py; src/backends.py; src/metrics.py).
"""

import math

import numpy as np
import pytest

import paper_1302_0120_b200 as pm
from paper_1302_0120_b200.backends import BackendSelector
from paper_1302_0120_b200.grid import FOURIER_PLANE, SLM_PLANE
from paper_1302_0120_b200.metrics import ConvergenceRecord, records_from_text, records_to_text
from paper_1302_0120_b200.patterns import (make_problem, modulus_from_intensity, spot_grid_centers,
                                           spot_pattern, to_centered_order, to_fourier_order)


def test_solve_rejects_zero_amplitude_and_dark_target_before_device():
    spec = pm.GridSpec(16, 16)
    p, m = make_problem(16, 3, 3)
    with pytest.raises(ValueError, match="identically zero"):
        pm.solve(pm.SlmConstraint(pm.RealGrid(spec, np.zeros(spec.shape))),
                 pm.FourierConstraint(pm.RealGrid(spec, m)), pm.SolveConfig(max_iters=1))
    with pytest.raises(ValueError, match="all dark"):
        pm.solve(pm.SlmConstraint(pm.RealGrid(spec, p)),
                 pm.FourierConstraint(pm.RealGrid(spec, np.zeros(spec.shape))), pm.SolveConfig(max_iters=1))
    with pytest.raises(ValueError, match="different grids"):
        pm.solve(pm.SlmConstraint(pm.RealGrid(spec, p)),
                 pm.FourierConstraint(pm.RealGrid(pm.GridSpec(8, 8), np.ones((8, 8)))),
                 pm.SolveConfig(max_iters=1))


def test_solve_config_validation():
    with pytest.raises(ValueError):
        pm.SolveConfig(max_iters=0)
    with pytest.raises(ValueError):
        pm.SolveConfig(record_every=0)
    with pytest.raises(ValueError):
        pm.SolveConfig(early_stop_tol=-1.0)
    with pytest.raises(ValueError):
        pm.SolveConfig(algorithm="hio")
    assert pm.SolveConfig().algorithm == "gs" and pm.SolveConfig().max_iters == 25


def test_backend_selector_parsing_like_reference():
    assert BackendSelector.parse("serial").fft_workers == 1
    sel = BackendSelector.parse("threaded:6")
    assert (sel.strategy, sel.workers, sel.fft_workers) == ("threaded", 6, 6)
    with pytest.raises(ValueError):
        BackendSelector.parse("cuda")            # reference tests/test_backends.py:20-22
    with pytest.raises(ValueError):
        BackendSelector(strategy="threaded", workers=0)


def test_precision_and_zero_tol():
    assert pm.SINGLE.zero_tol(1.0) == pytest.approx(1024 * np.finfo(np.float32).eps)
    assert pm.DOUBLE.zero_tol(2.0) == pytest.approx(2048 * np.finfo(np.float64).eps)
    assert pm.Precision.from_tag("single") is pm.SINGLE
    with pytest.raises(ValueError):
        pm.Precision.from_tag("half")


def test_grid_containers_validate():
    spec = pm.GridSpec(4, 2)
    assert spec.shape == (2, 4) and spec.n == 8
    assert spec.unflatten_index(spec.flatten_index(3, 1)) == (3, 1)
    with pytest.raises(ValueError):
        pm.GridSpec(0, 4)
    with pytest.raises(ValueError, match="non-finite"):
        pm.Field(spec, np.full(spec.shape, np.nan))
    with pytest.raises(ValueError, match="negative"):
        pm.RealGrid(spec, -np.ones(spec.shape))
    with pytest.raises(ValueError):
        pm.Field(spec, np.zeros(spec.shape), "nowhere")
    f = pm.Field(spec, np.zeros(spec.shape))
    assert f.dtype == np.complex128 and f.domain_tag == SLM_PLANE
    with pytest.raises(ValueError):
        f.data[0, 0] = 1                          # immutable, like the reference
    with pytest.raises(ValueError):
        pm.PhaseMask(spec, np.full(spec.shape, 2 * np.pi))


def test_phase_mask_uint8_round_trip():
    spec = pm.GridSpec(4, 1)
    mask = pm.PhaseMask(spec, np.array([[0.0, np.pi, 2 * np.pi * 255 / 256, 2 * np.pi - 1e-9]]))
    lv = mask.to_uint8()
    assert lv.tolist() == [[0, 128, 255, 255]]
    back = pm.PhaseMask.from_uint8(spec, lv)
    assert back.phases[0, 1] == pytest.approx(np.pi)


def test_convergence_record_text_round_trip():
    recs = [ConvergenceRecord(1, 0.5, 1e-3, 2e-4, 1.5, 0.5, 2.1), ConvergenceRecord(2, 0.25, 9e-4, 1e-4)]
    text = records_to_text(recs)
    assert text.splitlines()[0].startswith("iter\tgap")
    assert records_from_text(text) == recs


def test_patterns_match_reference_semantics():
    spec = pm.GridSpec(8, 8)
    img = spot_pattern(spec, [(2, 3)], radius=1)
    assert img.data.sum() == 1.0 and img.data[3, 2] == 1.0
    assert to_centered_order(to_fourier_order(img)).data.tolist() == img.data.tolist()
    assert modulus_from_intensity(pm.RealGrid(spec, np.full(spec.shape, 4.0))).data[0, 0] == 2.0
    assert spot_grid_centers(pm.GridSpec(64, 64)) == ((16, 16), (32, 16), (48, 16), (16, 32), (32, 32),
                                                      (48, 32), (16, 48), (32, 48), (48, 48))
    with pytest.raises(ValueError, match="overlap"):
        spot_pattern(spec, [(2, 2), (2, 2)])


def test_make_problem_is_energy_matched_and_seeded():
    p, m = make_problem(256, 8, 7)
    assert math.isclose(float((p ** 2).sum()), float((m ** 2).sum()), rel_tol=1e-12)
    assert (m > 0).sum() == 8 and p.min() / p.max() > 3e-4
    p2, m2 = make_problem(256, 8, 7)
    assert np.array_equal(m, m2)
    pr, mr = make_problem(64, 4, 11, n_y=32)
    assert pr.shape == mr.shape == (32, 64)


def test_plan_mismatch_error_is_value_error():
    assert issubclass(pm.PlanMismatchError, ValueError)
    f = pm.FftProvider(pm.GridSpec(8, 8))
    with pytest.raises(pm.PlanMismatchError):
        f._check(pm.Field(pm.GridSpec(4, 4), np.zeros((4, 4))), SLM_PLANE)
    with pytest.raises(pm.PlanMismatchError):
        f._check(pm.Field(pm.GridSpec(8, 8), np.zeros((8, 8)), FOURIER_PLANE), SLM_PLANE)


def test_solve_diverged_error_message():
    e = pm.SolveDivergedError(7)
    assert e.iteration == 7 and "iteration 7" in str(e)


# --- property tests of the grid helpers (reference tests/test_grid.py:21-26) ---
from hypothesis import given, settings, strategies as st  # noqa: E402


@given(st.integers(1, 37), st.integers(1, 23))
@settings(max_examples=60, deadline=None)
def test_index_round_trip_property(n_x, n_y):
    spec = pm.GridSpec(n_x, n_y)
    for x in range(0, spec.n, max(1, spec.n // 17)):
        j, k = spec.unflatten_index(x)
        assert spec.flatten_index(j, k) == x
    a = np.arange(spec.n).reshape(spec.shape)
    j, k = n_x - 1, n_y - 1
    assert a[k, j] == spec.flatten_index(j, k)


def test_naive_dft_is_a_public_name_with_the_reference_guard():
    """The reference exports naive_dft (src/__init__.py:13); its size guard
    (src/transform.py:67-70) is checked before any device work."""
    import paper_1302_0120_b200 as pm
    assert "naive_dft" in pm.__all__ and callable(pm.naive_dft)
    spec = pm.GridSpec(128, 64)
    with pytest.raises(ValueError, match="too large for the O"):
        pm.naive_dft(pm.Field(spec, np.zeros(spec.shape, complex)))


def test_spot_targets_equal_make_problem():
    """The config-4 target stack builder equals make_problem's m per seed."""
    from paper_1302_0120_b200.patterns import make_problem, spot_targets
    for n, spots in ((64, 8), (256, 50), (120, 6)):
        seeds = [1000, 1001, 7]
        st = spot_targets(n, spots, seeds)
        for i, sd in enumerate(seeds):
            assert np.array_equal(st[i], make_problem(n, spots, sd)[1])
