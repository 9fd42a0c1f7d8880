"""Generate the golden fixtures from the REFERENCE implementation.

Run in the build container, where the reference is importable read-only:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``phasemask`` from /root/reference/pkg/src (scipy 1.18.1 / DUCC0
FFT here), builds problems with this repo's §8(d) generator
(paper_1302_0120_b200/patterns.py, itself pinned against the reference's
pattern helpers by the fixtures below) and stores inputs and reference
outputs as small .npz files next to this script. The GPU tests compare the
CUDA path with these fixtures; the CPU tests check the oracle reproduces
them bit for bit. /root/reference does not exist on the GPU box — only the
.npz files travel.

RAAR has no reference implementation; its fixtures (raar_*.npz) come from the
oracle restatement (oracle/phasemask_oracle.py) and are marked as such.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(REPO))

from phasemask import metrics as R_metrics  # noqa: E402  (the reference)
from phasemask import patterns as R_patterns  # noqa: E402
from phasemask.bench import spot_grid_centers as R_centers  # noqa: E402
from phasemask.grid import DOUBLE, FOURIER_PLANE, SINGLE, Field, GridSpec, RealGrid  # noqa: E402
from phasemask.projections import (FourierConstraint, SlmConstraint,  # noqa: E402
                                   project_fourier, project_modulus, project_slm)
from phasemask.solver import SolveConfig, default_amplitude, solve  # noqa: E402
from phasemask.transform import FftProvider, naive_dft  # noqa: E402

from paper_1302_0120_b200.patterns import make_problem  # noqa: E402

PREC = {"double": DOUBLE, "single": SINGLE}


def ref_solve(p, m, tag, K, record_every=1, early_stop_tol=None, random_phase_init=False, seed=0):
    spec = GridSpec(p.shape[1], p.shape[0])
    prec = PREC[tag]
    r = solve(SlmConstraint(RealGrid(spec, p), prec), FourierConstraint(RealGrid(spec, m), prec),
              SolveConfig(max_iters=K, precision=prec, record_every=record_every,
                          early_stop_tol=early_stop_tol, random_phase_init=random_phase_init, seed=seed))
    hist = np.array([(h.iter, h.gap, h.err_lit, h.err_dark) for h in r.history], dtype=np.float64)
    return r, hist


def save(name, **arrays):
    np.savez_compressed(HERE / f"{name}.npz", **arrays)
    size = (HERE / f"{name}.npz").stat().st_size
    print(f"{name}.npz  {size / 1024:.0f} KiB")


def spot_lattice_problem(n_x, n_y):
    """The reference's default fixture (tests/conftest.py:17-24): 3x3 lattice, uniform p."""
    spec = GridSpec(n_x, n_y)
    inten = R_patterns.spot_pattern(R_patterns.SpotSpec(spec, R_centers(spec)))
    m = R_patterns.modulus_from_intensity(R_patterns.to_fourier_order(inten)).data
    p = default_amplitude(RealGrid(spec, m)).data
    return np.ascontiguousarray(p), np.ascontiguousarray(m)


def main():
    rng = np.random.default_rng(20240817)

    # -- generator pin: the §8(d) generator vs the reference's pattern helpers
    n = 64
    p, m = make_problem(n, 8, 7)
    save("problem64", p=p, m=m)

    # -- solver fixtures (full outputs), reference solve()
    cases = [
        ("gs16_double", 16, 16, 3, 3, "double", 10, {}),
        ("gs32_single", 32, 32, 4, 5, "single", 25, {}),
        ("gs64_double", 64, 64, 8, 7, "double", 25, {}),
        ("gs64x32_double", 64, 32, 4, 11, "double", 10, {}),
        ("gs64_single_rec3", 64, 64, 8, 7, "single", 25, {"record_every": 3}),
        ("gs128_double_early", 128, 128, 8, 7, "double", 200, {"early_stop_tol": 1.5e-7}),
        ("gs32_double_randinit", 32, 32, 4, 5, "double", 10, {"random_phase_init": True, "seed": 3}),
        ("gs256_double", 256, 256, 8, 7, "double", 100, {}),
        ("gs256_single", 256, 256, 8, 7, "single", 100, {}),
    ]
    for name, nx, ny, spots, seed, tag, K, kw in cases:
        p, m = make_problem(nx, spots, seed, n_y=ny)
        r, hist = ref_solve(p, m, tag, K, **kw)
        save(name, p=p, m=m, K=K, precision=tag, record_every=kw.get("record_every", 1),
             early_stop_tol=-1.0 if kw.get("early_stop_tol") is None else kw["early_stop_tol"],
             random_phase_init=int(kw.get("random_phase_init", False)), seed=kw.get("seed", 0),
             mask=r.mask.phases, u_star=r.u_star.data, v_star=r.v_star.data, history=hist,
             iters_run=r.iters_run)

    # -- the reference's own degenerate default fixture (3x3 lattice, uniform p)
    p, m = spot_lattice_problem(64, 64)
    r, hist = ref_solve(p, m, "double", 25)
    save("lattice64_double", p=p, m=m, K=25, precision="double", mask=r.mask.phases,
         u_star=r.u_star.data, v_star=r.v_star.data, history=hist, iters_run=r.iters_run)

    # -- per-iteration iterates: solve(K) returns the pair of u_K
    p, m = make_problem(64, 8, 7)
    for tag in ("double", "single"):
        us = []
        for K in (1, 2, 3, 5, 8):
            r, _ = ref_solve(p, m, tag, K)
            us.append(r.u_star.data)
        save(f"iterates64_{tag}", p=p, m=m, Ks=np.array([1, 2, 3, 5, 8]), u_star=np.stack(us))

    # -- large-size anchors: histories only
    for name, n, spots, tag, K in [("anchor512_double", 512, 8, "double", 200),
                                   ("anchor1024_single", 1024, 50, "single", 100),
                                   ("anchor1024_double", 1024, 50, "double", 100)]:
        p, m = make_problem(n, spots, 7)
        r, hist = ref_solve(p, m, tag, K)
        ph = r.mask.phases
        save(name, n=n, spots=spots, seed=7, K=K, precision=tag, history=hist,
             mask_checksum=np.array([ph.sum(), (ph * ph).sum(), ph[::37, ::53].sum()]),
             mask_sample=ph[::64, ::64].copy())

    # -- transform / projection / metric KATs from the reference primitives
    kat = {}
    for nx, ny, tag in ((8, 8, "double"), (16, 16, "single"), (32, 8, "double"), (4, 64, "single")):
        spec = GridSpec(nx, ny)
        prec = PREC[tag]
        x = (rng.standard_normal(spec.shape) + 1j * rng.standard_normal(spec.shape)).astype(prec.complex_dtype)
        prov = FftProvider(spec, prec)
        fwd = prov.forward(Field(spec, x)).data
        inv = prov.inverse(Field(spec, x, FOURIER_PLANE)).data
        kat[f"fft_{nx}x{ny}_{tag}_in"] = x
        kat[f"fft_{nx}x{ny}_{tag}_fwd"] = fwd
        kat[f"fft_{nx}x{ny}_{tag}_inv"] = inv
        if nx * ny <= 4096:
            kat[f"fft_{nx}x{ny}_{tag}_naive"] = naive_dft(Field(spec, x)).data
    for tag in ("double", "single"):
        prec = PREC[tag]
        spec = GridSpec(32, 32)
        u = (rng.standard_normal(spec.shape) + 1j * rng.standard_normal(spec.shape)).astype(prec.complex_dtype)
        u[0, :4] = 0                                     # exact zero branch
        u[1, :4] = 1e-9                                  # below every threshold
        t = rng.uniform(0.1, 2.0, spec.shape)
        t[2, :3] = 0.0
        c = SlmConstraint(RealGrid(spec, t), prec)
        mc = FourierConstraint(RealGrid(spec, t), prec)
        kat[f"proj_{tag}_u"] = u
        kat[f"proj_{tag}_t"] = t
        kat[f"proj_{tag}_slm"] = project_slm(Field(spec, u), c).data
        kat[f"proj_{tag}_mod"] = project_modulus(Field(spec, u, FOURIER_PLANE), mc).data
        kat[f"proj_{tag}_fourier"] = project_fourier(Field(spec, u), mc, FftProvider(spec, prec)).data
        kat[f"gap_{tag}"] = np.array(R_metrics.gap(Field(spec, u), c, mc, FftProvider(spec, prec)))
    save("kats", **kat)

    # -- RAAR: restatement only (no reference implementation exists)
    from oracle import phasemask_oracle as orc
    for name, n, spots, tag, K in [("raar64_double", 64, 8, "double", 20),
                                   ("raar64_single", 64, 8, "single", 5)]:
        p, m = make_problem(n, spots, 7)
        o = orc.solve(p, m, K, tag, algorithm="raar", beta=0.9)
        hist = np.array(o["records"], dtype=np.float64)
        save(name, p=p, m=m, K=K, precision=tag, beta=0.9, mask=o["mask"], u_star=o["u_star"],
             v_star=o["v_star"], history=hist, iters_run=o["iters_run"], source="oracle-restatement")
    p, m = make_problem(512, 8, 7)
    o = orc.solve(p, m, 20, "double", algorithm="raar", beta=0.9)
    save("raar512_double_anchor", K=20, history=np.array(o["records"], dtype=np.float64),
         source="oracle-restatement")


# Outcome of the reference's solve() on amplitudes scaled towards the float
# range (the divergence / non-finite contract, src/solver.py:27-32,152-199,
# src/grid.py:100-110,128-129): "ok", "div<it>" (SolveDivergedError) or
# "VE:<message>" (ValueError from a Field / RealGrid check in the metrics).
DIVERGENCE_CASES = [(n, ny, tag, c, rec, es)
                    for n, ny in ((64, 64), (256, 256), (120, 90))
                    for tag, c in (("single", 1e19), ("single", 1e36), ("single", 1e38),
                                   ("double", 1e160), ("double", 1e308))
                    for rec, es in ((1, None), (100, None), (100, 1e-3))]


def divergence_outcomes():
    from phasemask.solver import SolveDivergedError
    out = []
    for n, ny, tag, c, rec, es in DIVERGENCE_CASES:
        p, m = make_problem(n, 8, 7, n_y=ny)
        p = p / p.max() * c
        try:
            ref_solve(p, m, tag, 6, record_every=rec, early_stop_tol=es)
            o = "ok"
        except SolveDivergedError as e:
            o = f"div{e.iteration}"
        except ValueError as e:
            o = f"VE:{e}"
        out.append(o)
    return out


def main_divergence():
    import json
    with np.errstate(all="ignore"):
        out = divergence_outcomes()
    (HERE / "divergence_outcomes.json").write_text(json.dumps(
        {"cases": [list(c) for c in DIVERGENCE_CASES], "K": 6, "spots": 8, "seed": 7, "outcomes": out}, indent=0))
    print("divergence_outcomes.json", len(out))


if __name__ == "__main__":
    if sys.argv[1:] == ["divergence"]:
        main_divergence()
    else:
        main()
        main_divergence()
