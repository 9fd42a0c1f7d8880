"""GPU: levels-only outputs of the batch and streaming APIs (SURVEY.md §8f-2:
the SLM's 8-bit levels computed on the device, 1 byte per pixel downloaded),
and the drop-in's trusted outputs."""

import numpy as np
import pytest

import paper_1302_0120_b200 as pm
from paper_1302_0120_b200.batch import solve_stack, solve_stream
from paper_1302_0120_b200.patterns import make_problem, spot_targets

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,ny", [(256, 256), (120, 90)])
def test_levels_only_equal_the_mask_levels(n, ny):
    p, _ = make_problem(n, 8, 1000, n_y=ny)
    ms = spot_targets(n, 8, [1000, 1001, 1002], n_y=ny)
    cfg = pm.SolveConfig(max_iters=12, precision=pm.SINGLE)
    full = solve_stack(p, ms, cfg)
    lev = solve_stack(p, ms, cfg, phases=False, levels=True)
    assert lev.phases is None and lev.levels.dtype == np.uint8
    want = np.stack([pm.PhaseMask(pm.GridSpec(n, ny), ph).to_uint8() for ph in full.phases])
    np.testing.assert_array_equal(lev.levels, want)
    np.testing.assert_array_equal(lev.gap, full.gap)
    frames = list(solve_stream(((p.astype(np.float32), m.astype(np.float32)) for m in ms), cfg, levels_only=True))
    assert len(frames) == 3
    for i, fr in enumerate(frames):
        assert fr.phases is None
        np.testing.assert_array_equal(fr.levels[0], want[i])
    with pytest.raises(ValueError):
        solve_stack(p, ms, cfg, phases=False)


def test_dropin_outputs_are_the_validated_ones():
    """solve() returns the device's mask / pair without host validation passes;
    they are what the validating constructors accept, read-only."""
    p, m = make_problem(256, 8, 7)
    spec = pm.GridSpec(256, 256)
    r = pm.solve(pm.SlmConstraint(pm.RealGrid(spec, p), pm.SINGLE),
                 pm.FourierConstraint(pm.RealGrid(spec, m), pm.SINGLE),
                 pm.SolveConfig(max_iters=10, precision=pm.SINGLE))
    assert not r.mask.phases.flags.writeable and not r.u_star.data.flags.writeable
    pm.PhaseMask(spec, r.mask.phases)
    pm.Field(spec, r.u_star.data)
    pm.Field(spec, r.v_star.data)
    assert r.u_star.data.dtype == np.complex64 and r.u_star.domain_tag == "slm_plane"


def test_zero_inputs_rejected_with_the_reference_messages():
    spec = pm.GridSpec(64, 64)
    p, m = make_problem(64, 4, 7)
    with pytest.raises(ValueError, match="^SLM amplitude is identically zero$"):
        pm.solve(pm.SlmConstraint(pm.RealGrid(spec, np.zeros_like(p))), pm.FourierConstraint(pm.RealGrid(spec, m)),
                 pm.SolveConfig(max_iters=3))
    with pytest.raises(ValueError, match=r"^target pattern is identically zero \(all dark\)$"):
        pm.solve(pm.SlmConstraint(pm.RealGrid(spec, p)), pm.FourierConstraint(pm.RealGrid(spec, np.zeros_like(m))),
                 pm.SolveConfig(max_iters=3))
