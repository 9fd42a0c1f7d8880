"""GPU parity at the BASELINE.json sizes: the CUDA solve against the oracle
(the reference's solve(), src/solver.py:111-216, restated in oracle/ and
pinned bitwise to the reference by tests/test_oracle_golden.py), both run
on the GPU box on the same seeded SURVEY.md §8(d) inputs.

Config 3 (1024^2, 50 spots, 100 GS iterations) in fp32 and fp64, and
config 5 (2048^2 and 4096^2 fp32). Tolerances (written here):
  fp64: u*/v* relL2 <= 1e-10, amplitude-weighted mask <= 1e-10 rad, gap <= 1e-12 rel
  fp32: u*/v* relL2 <= 1e-4,  amplitude-weighted mask <= 1e-4 rad,  gap <= 1e-6 rel
plus the reference mask checksums of the committed 1024^2 anchors
(tests/golden/make_golden.py) and size-independent properties (|u*| = p on
lit pixels, the mask in [0, 2 pi)).
"""

import os

import numpy as np
import pytest

import paper_1302_0120_b200 as pm
from conftest import golden
from oracle import phasemask_oracle as orc
from paper_1302_0120_b200.patterns import make_problem

pytestmark = pytest.mark.gpu

TOL = {"double": dict(field=1e-10, gap=1e-12, phase=1e-10, err=1e-9),
       "single": dict(field=1e-4, gap=1e-6, phase=1e-4, err=1e-4)}
WORKERS = os.cpu_count() or 1


def gpu_solve(p, m, n, tag, K, record_every):
    prec = pm.Precision.from_tag(tag)
    spec = pm.GridSpec(n, n)
    return pm.solve(pm.SlmConstraint(pm.RealGrid(spec, p), prec), pm.FourierConstraint(pm.RealGrid(spec, m), prec),
                    pm.SolveConfig(max_iters=K, precision=prec, record_every=record_every))


def compare(r, o, p, tag):
    t = TOL[tag]
    assert r.iters_run == o["iters_run"]
    e_u = orc.relative_l2(r.u_star.data, o["u_star"])
    e_v = orc.relative_l2(r.v_star.data, o["v_star"])
    e_ph = orc.weighted_phase_error(r.mask.phases, o["mask"], p)
    assert e_u <= t["field"], e_u
    assert e_v <= t["field"], e_v
    assert e_ph <= t["phase"], e_ph
    h = np.array([(x.iter, x.gap, x.err_lit, x.err_dark) for x in r.history])
    ho = np.array(o["records"], dtype=np.float64)
    assert h.shape == ho.shape
    np.testing.assert_array_equal(h[:, 0], ho[:, 0])
    np.testing.assert_allclose(h[:, 1], ho[:, 1], rtol=t["gap"], atol=0)
    np.testing.assert_allclose(h[:, 2:], ho[:, 2:], rtol=t["err"], atol=t["err"] * 1e-3)
    # size-independent properties: |u*| = p (every pixel is lit for the Gaussian beam), mask range
    prec = pm.Precision.from_tag(tag)
    np.testing.assert_allclose(np.abs(r.u_star.data), p.astype(prec.float_dtype), rtol=8 * prec.eps_machine)
    assert r.mask.phases.min() >= 0.0 and r.mask.phases.max() < 2 * np.pi
    return e_u, e_ph


@pytest.mark.parametrize("tag", ["single", "double"])
def test_config3_1024_vs_oracle(tag):
    """BASELINE config 3: 1024^2, 50 spots, 100 GS iterations; the full pair,
    mask and the gap / physical-error history every 10th iteration."""
    n, K, rec = 1024, 100, 10
    p, m = make_problem(n, 50, 7)
    r = gpu_solve(p, m, n, tag, K, rec)
    o = orc.solve(p, m, K, tag, record_every=rec, workers=WORKERS)
    compare(r, o, p, tag)


@pytest.mark.parametrize("tag", ["single", "double"])
def test_config3_mask_checksum(tag):
    """The reference's own mask checksums at config 3 (tests/golden/make_golden.py:115-123):
    sum, sum of squares and a strided subsample sum of the float64 mask."""
    g = golden(f"anchor1024_{tag}")
    p, m = make_problem(1024, 50, 7)
    r = gpu_solve(p, m, 1024, tag, int(g["K"]), 1)
    ph = r.mask.phases
    got = np.array([ph.sum(), (ph * ph).sum(), ph[::37, ::53].sum()])
    np.testing.assert_allclose(got, g["mask_checksum"], rtol=1e-11 if tag == "double" else 2e-5)


@pytest.mark.parametrize("n,K", [(2048, 100), (4096, 20)])
def test_config5_large_fields_vs_oracle(n, K):
    """BASELINE config 5: 2048^2 (field resident in L2) and 4096^2 (HBM) fp32."""
    p, m = make_problem(n, 50, 7)
    rec = max(1, K // 5)
    r = gpu_solve(p, m, n, "single", K, rec)
    o = orc.solve(p, m, K, "single", record_every=rec, workers=WORKERS)
    compare(r, o, p, "single")


def test_config5_4096_fp64_short():
    """4096^2 in fp64 (the HBM-resident field at 256 MiB), 5 iterations."""
    n, K = 4096, 5
    p, m = make_problem(n, 50, 7)
    r = gpu_solve(p, m, n, "double", K, 1)
    o = orc.solve(p, m, K, "double", record_every=1, workers=WORKERS)
    compare(r, o, p, "double")
