"""Batches of independent masks: one launch per device, shards across GPUs.

A single mask never shards (a 2-D FFT split across GPUs
would need two all-to-all transposes per iteration for microseconds of
work). A batch of masks with distinct targets — the reference's sequential
``PhaseMaskTransformer.transform`` loop (src/estimator.py:85-93) — is
embarrassingly parallel:

* on one GPU, the whole batch runs in one persistent launch (every mask in
  lockstep through the same sweeps, per-mask stop flags and histories);
* across GPUs, masks are split into contiguous blocks of ceil(B / G), one
  host thread and one plan (stream) per device, with no collective on the
  iteration path;
* across processes (one rank per GPU, ``torch.distributed``), each rank
  solves its block and the results are gathered once at the end.

Results are bitwise independent of the batch size and of the device count:
every per-mask reduction runs in a fixed order that does not depend on
which CTA or device handled the mask.
"""

from __future__ import annotations

import warnings
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

from . import _lib
from .grid import GridSpec, Precision
from .solver import SolveConfig, SolveDivergedError, _host_cast, _host_empty, _params
from .transform import get_plan


def shard_bounds(n_items: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block [lo, hi) of rank `rank` out of `world` (ceil split)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    per = -(-n_items // world) if n_items else 0
    lo = min(n_items, rank * per)
    return lo, min(n_items, lo + per)


@dataclass
class BatchResult:
    """Per-mask outputs of a batch solve, stacked along axis 0."""

    phases: np.ndarray | None   # (B, n_y, n_x) float64 in [0, 2pi) (None: levels-only solve)
    gap: np.ndarray             # (B, K) gap history, NaN where not recorded
    err_lit: np.ndarray         # (B, K)
    err_dark: np.ndarray        # (B, K)
    iters_run: np.ndarray       # (B,)
    device_ms: float = 0.0      # device time of the slowest shard
    levels: np.ndarray | None = None   # (B, n_y, n_x) uint8 SLM levels (PhaseMask.to_uint8), when asked

    @staticmethod
    def concat(parts: list["BatchResult"]) -> "BatchResult":
        parts = [q for q in parts if q.iters_run.shape[0]]
        levels = None if any(q.levels is None for q in parts) else np.concatenate([q.levels for q in parts])
        phases = None if any(q.phases is None for q in parts) else np.concatenate([q.phases for q in parts])
        return BatchResult(phases,
                           np.concatenate([q.gap for q in parts]),
                           np.concatenate([q.err_lit for q in parts]),
                           np.concatenate([q.err_dark for q in parts]),
                           np.concatenate([q.iters_run for q in parts]),
                           max(q.device_ms for q in parts), levels)


def _maxes(a: np.ndarray, k: int) -> np.ndarray:
    return np.asarray(a).reshape(k, -1).max(axis=1)


def solve_stack(p: np.ndarray, m_stack: np.ndarray, cfg: SolveConfig, device: int = 0,
                out_phases: np.ndarray | None = None, levels: bool = False,
                init: np.ndarray | None = None, phases: bool = True,
                out_levels: np.ndarray | None = None) -> BatchResult:
    """Solve a stack of targets on one device in one launch.

    p: (n_y, n_x) shared amplitude or (B, n_y, n_x) per mask; m_stack:
    (B, n_y, n_x) target moduli in DFT order. Arrays already in the
    precision's dtype are used without a host copy (pass pinned buffers for
    full-speed transfers); ``out_phases`` (B, n_y, n_x) float64 may be a
    caller-owned (e.g. pinned) buffer for the mask; ``levels=True`` also
    returns the 8-bit SLM levels computed on the device, and with
    ``phases=False`` they are the only per-pixel output (1 byte per pixel
    downloaded instead of 8; ``out_levels`` may be a caller-owned (B, n_y,
    n_x) uint8 buffer); ``init`` (B, n_y, n_x)
    complex are caller-chosen Fourier-plane starts instead of m; without it,
    ``cfg.random_phase_init`` draws the seeded phases on the device
    (src/solver.py:100-103, the same draws for every mask, as a reference
    solve per image re-seeds). The per-mask energy
    sum(m^2) and the zero tolerances are reduced on the device.
    """
    m_stack = np.asarray(m_stack)
    if m_stack.ndim != 3:
        raise ValueError("m_stack must be (batch, n_y, n_x)")
    B, ny, nx = m_stack.shape
    if B == 0:
        z = np.zeros((0, cfg.max_iters))
        return BatchResult(np.zeros((0, ny, nx)), z, z.copy(), z.copy(), np.zeros(0, np.int32))
    p = np.asarray(p)
    per_mask = p.ndim == 3
    if (p.shape[-2:] != (ny, nx)) or (per_mask and p.shape[0] != B):
        raise ValueError("amplitude and target constraints live on different grids")
    prec = cfg.precision
    fdt = prec.float_dtype
    plan = get_plan(GridSpec(nx, ny), prec, device)
    pp = _host_cast(p, fdt)                  # page-locked when a cast is needed anyway
    mm = _host_cast(m_stack, fdt)
    # the zero tolerances 1024 eps max(.) and the "identically zero" checks
    # (src/solver.py:122-125) run on the device, on the uploaded p and m
    tol_p = tol_m = None
    K = cfg.max_iters
    want_phases = phases
    if not want_phases and not levels:
        raise ValueError("phases=False needs levels=True (no per-pixel output otherwise)")
    phases = None
    if want_phases:
        phases = out_phases if out_phases is not None else _host_empty((B, ny, nx), np.float64)
        if phases.shape != (B, ny, nx) or phases.dtype != np.float64 or not phases.flags.c_contiguous:
            raise ValueError("out_phases must be a C-contiguous float64 (batch, n_y, n_x) array")
    out = BatchResult(phases, np.full((B, K), np.nan), np.full((B, K), np.nan),
                      np.full((B, K), np.nan), np.zeros(B, np.int32))
    div = np.zeros(B, np.int32)
    ms = np.zeros(1, np.float32)
    res = _lib.pm_result()
    res.phases = _lib.ptr(out.phases)
    res.gap, res.err_lit, res.err_dark = _lib.ptr(out.gap), _lib.ptr(out.err_lit), _lib.ptr(out.err_dark)
    res.iters_run, res.diverged_iter, res.device_ms = _lib.ptr(out.iters_run), _lib.ptr(div), _lib.ptr(ms)
    if levels:
        # 8-bit SLM levels computed on the device (reference src/grid.py:152-154)
        if out_levels is not None:
            if out_levels.shape != (B, ny, nx) or out_levels.dtype != np.uint8 or not out_levels.flags.c_contiguous:
                raise ValueError("out_levels must be a C-contiguous uint8 (batch, n_y, n_x) array")
            out.levels = out_levels
        else:
            out.levels = _host_empty((B, ny, nx), np.uint8)
        res.levels = _lib.ptr(out.levels)
    init_c = None
    if init is not None:
        init_c = np.ascontiguousarray(init, dtype=prec.complex_dtype)
        if init_c.shape != (B, ny, nx):
            raise ValueError("init must be a (batch, n_y, n_x) complex stack")
    prm = _params(cfg, per_mask, init_c is not None)
    with plan.lock:
        code = plan.lib.pm_solve(plan.handle, _lib.ptr(pp), _lib.ptr(mm), _lib.ptr(init_c), B, prm,
                                 _lib.ptr(tol_p), _lib.ptr(tol_m), None, res)
    if code == _lib.PM_ERR_DIVERGED or div.any():
        raise _diverged(div)
    _lib.check(code, "pm_solve")
    out.device_ms = float(ms[0])
    return out


def _diverged(div: np.ndarray) -> SolveDivergedError:
    """The batch contract: SolveDivergedError of the first mask that diverged,
    carrying the iteration whose loop body went non-finite
    (src/solver.py:152-165) and, in ``per_mask``, every mask's (0 = finite)."""
    bad = div[div > 0]
    e = SolveDivergedError(int(bad[0]) if bad.size else 1)
    e.per_mask = div.copy()
    return e


def solve_stream(items, cfg: SolveConfig, device: int = 0, out_phases: list | None = None,
                 levels_only: bool = False):
    """A real-time sequence of masks on one device (the paper's interactive
    use: a new target pattern per frame), pipelined.

    ``items`` yields ``(p, m)`` pairs of (n_y, n_x) host arrays (pinned for
    full-speed copies), one mask per item. While mask i is solved, the
    upload of item i+1 and the download of mask i-1 run on their own CUDA
    streams, so a frame costs about max(solve, transfers) instead of their
    sum. Yields one :class:`BatchResult` (batch 1) per item, in order, one
    item behind the solve. ``out_phases``: optional two (1, n_y, n_x) float64
    (pinned) host buffers, used alternately for the masks (a yielded mask
    stays valid until two more have been produced); otherwise fresh arrays.
    Every solve is :func:`solve_stack`'s (device tolerances and energy),
    bitwise. ``levels_only``: each frame downloads the uint8 SLM levels (1
    byte per pixel, what an SLM displays) instead of the
    float64 mask (BatchResult.levels set, .phases None); ``out_phases`` then
    holds uint8 buffers.
    """
    import torch                                        # streams and events only (plumbing)

    dev = torch.device("cuda", device)
    it = iter(items)
    first = next(it, None)
    if first is None:
        return
    p0 = np.asarray(first[0])
    ny, nx = p0.shape
    prec = cfg.precision
    fdt = prec.float_dtype
    tdt = torch.float32 if fdt == np.float32 else torch.float64
    plan = get_plan(GridSpec(nx, ny), prec, device)
    K = cfg.max_iters
    prm = _params(cfg, False, False)
    # the solve runs on the plan's own stream; uploads and downloads on two more
    h = _lib.C.c_void_p(0)
    _lib.check(plan.lib.pm_plan_get_stream(plan.handle, _lib.C.byref(h)), "pm_plan_get_stream")
    compute = torch.cuda.ExternalStream(h.value or 0, device=dev)
    up, down = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    d_p = [torch.empty((ny, nx), dtype=tdt, device=dev) for _ in range(2)]
    d_m = [torch.empty((ny, nx), dtype=tdt, device=dev) for _ in range(2)]
    odt = torch.uint8 if levels_only else torch.float64
    d_ph = [torch.empty((ny, nx), dtype=odt, device=dev) for _ in range(2)]
    ev_up = [torch.cuda.Event() for _ in range(2)]
    ev_done = [torch.cuda.Event() for _ in range(2)]
    ev_down = [torch.cuda.Event() for _ in range(2)]
    outs = out_phases or [None, None]

    def upload(slot, item):
        pp = np.ascontiguousarray(item[0], dtype=fdt)
        mm = np.ascontiguousarray(item[1], dtype=fdt)
        if pp.shape != (ny, nx) or mm.shape != (ny, nx):
            raise ValueError("amplitude and target constraints live on different grids")
        with torch.cuda.stream(up), warnings.catch_warnings():
            # read-only host arrays are only read here (torch warns on any non-writable array)
            warnings.simplefilter("ignore", UserWarning)
            up.wait_event(ev_done[slot])               # the solve two frames back read this slot
            d_p[slot].copy_(torch.from_numpy(pp), non_blocking=True)
            d_m[slot].copy_(torch.from_numpy(mm), non_blocking=True)
            ev_up[slot].record(up)
        return pp, mm                                  # keep the host arrays alive until copied

    pending = None                                     # (slot, BatchResult, host phases) of the last frame
    keep = [upload(0, first), None]
    item, i = first, 0
    try:
        while item is not None:
            s = i & 1
            nxt = next(it, None)
            if nxt is not None:
                keep[s ^ 1] = upload(s ^ 1, nxt)
            compute.wait_event(ev_up[s])
            compute.wait_event(ev_down[s])        # d_ph[s] downloaded (frame i-2)
            res_py = BatchResult(None, np.full((1, K), np.nan), np.full((1, K), np.nan),
                                 np.full((1, K), np.nan), np.zeros(1, np.int32))
            div = np.zeros(1, np.int32)
            ms = np.zeros(1, np.float32)
            res = _lib.pm_result()
            if levels_only:
                res.levels = _lib.C.c_void_p(d_ph[s].data_ptr())
            else:
                res.phases = _lib.C.c_void_p(d_ph[s].data_ptr())
            res.gap, res.err_lit, res.err_dark = (_lib.ptr(res_py.gap), _lib.ptr(res_py.err_lit),
                                                  _lib.ptr(res_py.err_dark))
            res.iters_run, res.diverged_iter, res.device_ms = (_lib.ptr(res_py.iters_run), _lib.ptr(div),
                                                               _lib.ptr(ms))
            with plan.lock:
                code = plan.lib.pm_solve_device(plan.handle, _lib.C.c_void_p(d_p[s].data_ptr()),
                                                _lib.C.c_void_p(d_m[s].data_ptr()), None, 1, prm, None, None,
                                                None, res)
            if code == _lib.PM_ERR_DIVERGED or div.any():
                raise _diverged(div)
            _lib.check(code, "pm_solve_device")
            res_py.device_ms = float(ms[0])
            ev_done[s].record(compute)
            host = outs[s] if outs[s] is not None else np.empty((1, ny, nx), np.uint8 if levels_only else np.float64)
            with torch.cuda.stream(down):
                down.wait_event(ev_done[s])
                torch.from_numpy(host).view(ny, nx).copy_(d_ph[s], non_blocking=True)
                ev_down[s].record(down)
            if pending is not None:                # frame i-1: its download ran during this solve
                ps, pres, phost = pending
                ev_down[ps].synchronize()
                if levels_only:
                    pres.levels = phost
                else:
                    pres.phases = phost
                yield pres
            pending = (s, res_py, host)
            item, i = nxt, i + 1
        ps, pres, phost = pending
        ev_down[ps].synchronize()
        if levels_only:
            pres.levels = phost
        else:
            pres.phases = phost
        yield pres
    finally:
        torch.cuda.synchronize(dev)
    del keep


def solve_batch(p: np.ndarray, m_stack: np.ndarray, cfg: SolveConfig,
                devices: list[int] | None = None, **kw) -> BatchResult:
    """Shard a stack of masks across local GPUs (one host thread per device).

    Extra keyword arguments (``levels``, ``init``) go to :func:`solve_stack`;
    a per-mask ``init`` stack is split with the masks.
    """
    if devices is None:
        devices = list(range(max(1, _lib.device_count())))
    m_stack = np.asarray(m_stack)
    B = m_stack.shape[0]
    per_mask = np.ndim(p) == 3
    G = len(devices)
    bounds = [shard_bounds(B, G, r) for r in range(G)]

    init = kw.pop("init", None)

    def run(r):
        lo, hi = bounds[r]
        return solve_stack(p[lo:hi] if per_mask else p, m_stack[lo:hi], cfg, devices[r],
                           init=None if init is None else init[lo:hi], **kw)

    if G == 1:
        return run(0)
    with ThreadPoolExecutor(G) as ex:
        parts = list(ex.map(run, range(G)))
    return BatchResult.concat(parts)


def solve_batch_distributed(p: np.ndarray, m_stack: np.ndarray, cfg: SolveConfig, device: int | None = None,
                            solve_fn=None) -> BatchResult | None:
    """One rank per GPU under torch.distributed: solve this rank's block of
    the stack, gather every block on rank 0 (returns None on other ranks).

    ``solve_fn(p, m_block, cfg, device)`` defaults to :func:`solve_stack`;
    the gather is one all_gather_object at the end, never on the iteration
    path.
    """
    import torch.distributed as dist
    world, rank = dist.get_world_size(), dist.get_rank()
    lo, hi = shard_bounds(np.asarray(m_stack).shape[0], world, rank)
    per_mask = np.ndim(p) == 3
    if device is None:
        import os
        device = int(os.environ.get("LOCAL_RANK", rank))
    fn = solve_fn or solve_stack
    part = fn(p[lo:hi] if per_mask else p, np.asarray(m_stack)[lo:hi], cfg, device)
    gathered = [None] * world
    dist.all_gather_object(gathered, part)
    return BatchResult.concat(gathered) if rank == 0 else None
