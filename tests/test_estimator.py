"""The sklearn front end (reference src/estimator.py, tests/test_estimator.py
patterns): validation and parameters on CPU; the GPU batch route for 3-D
stacks against one-at-a-time solves (bitwise)."""

import numpy as np
import pytest

from paper_1302_0120_b200.estimator import PhaseMaskTransformer, check_target_image
from paper_1302_0120_b200.patterns import spot_pattern
from paper_1302_0120_b200.grid import GridSpec


def targets(n=64, k=3):
    spec = GridSpec(n, n)
    out = []
    for i in range(k):
        centers = tuple((8 + 9 * i + 5 * s, 12 + 7 * s) for s in range(3))
        out.append(spot_pattern(spec, centers).data)
    return np.stack(out)


@pytest.mark.parametrize("bad,msg", [(np.zeros((2, 2, 2, 2)), "expected a 2D"),
                                     (np.array([[1.0, np.nan]]), "non-finite"),
                                     (np.array([[1.0, -1.0]]), "nonnegative"),
                                     (np.zeros((4, 4)), "all dark")])
def test_check_target_image_rejections(bad, msg):
    with pytest.raises(ValueError, match=msg):
        check_target_image(bad)


def test_params_round_trip():
    t = PhaseMaskTransformer(iters=7, precision="single", seed=3)
    assert t.get_params()["iters"] == 7
    t.set_params(iters=9, early_stop_tol=1e-4)
    assert t.iters == 9 and t._config().early_stop_tol == 1e-4
    with pytest.raises(ValueError):
        PhaseMaskTransformer(strategy="cuda")._config()     # the reference's closed backend seam


def test_transform_rejects_bad_rank():
    with pytest.raises(ValueError, match="2D image or 3D stack"):
        PhaseMaskTransformer().transform(np.ones(5))


@pytest.mark.gpu
@pytest.mark.parametrize("precision,rand", [("double", False), ("single", True)])
def test_stack_transform_matches_single_solves(precision, rand):
    X = targets()
    t = PhaseMaskTransformer(iters=12, precision=precision, random_phase_init=rand, seed=4)
    stack = t.transform(X)
    assert stack.shape == X.shape
    for i in range(X.shape[0]):
        np.testing.assert_array_equal(stack[i], t.transform(X[i]))
    t.fit(X[0])
    np.testing.assert_array_equal(t.mask_.phases, stack[0])
    assert len(t.history_) == 12
