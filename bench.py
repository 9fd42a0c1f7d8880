"""Benchmark: ms per 1024^2 phase mask (100 GS iterations, fp32) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 1..5]

Default workload (BASELINE.json configs[2], "config 3"): a 1024x1024 SLM,
50-spot target and Gaussian-beam amplitude from the SURVEY.md §8(d)
generator (synthetic, seeded), 100 Gerchberg-Saxton iterations in fp32, one
mask per GPU per step (weak scaling across ranks, no collective on the
iteration path). Metrics are recorded with record_every = iters, as the
reference's own bench does (src/bench.py:100-102), so the gap and the
physical errors are computed on the first and last iterations only.

value  = device time per mask (inputs resident in HBM, CUDA events on the
         solve's stream, L2 flushed by a 256 MiB write before every step),
         max over ranks, divided by the masks of the whole job.
e2e    = the same through the public host API, frame by frame
         (paper_1302_0120_b200.batch.solve_stream): every step uploads p and m
         from pinned memory and downloads the float64 mask and histories; the
         neighbouring frames' copies overlap each solve. e2e.latency = one
         synchronous solve_stack call per mask; e2e.dropin = the reference's
         entry point solve(c, m, cfg) with float64 host grids, SolveResult out.
roofline = the solve's algorithmic bytes / time against the L2-resident copy
         bandwidth measured in the same run (the field stays in L2), with the
         HBM fraction beside it; cpu_baseline / clocks / gpu_launches: see
         DESIGN.md §8.
--config 1 / 2 / 4 / 5 measure the other BASELINE configs the same way
(4: a 256-mask batch sharded over the ranks).

Under torchrun each rank drives cuda:LOCAL_RANK; rank 0 prints one JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

N_PIX = 1024
ITERS = 100
SPOTS = 50
SEED = 7
METRIC = "ms per 1024² phase mask (100 iters) and AP iterations/s; % of HBM/L2 roofline"
BYTES_PER_ITER = 40 * N_PIX * N_PIX          # fp32 GS, two fused sweeps


def workload_config(world: int, plan_path: str = "persistent") -> dict:
    """The `config` of both arms (ours and --impl reference): the same keys."""
    return {"workload": "gs_1024x1024_fp32_100iter_50spots_single_mask", "n_x": N_PIX, "n_y": N_PIX,
            "iters": ITERS, "spots": SPOTS, "seed": SEED, "masks_per_step": world, "masks_per_rank": 1,
            "record_every": ITERS, "parallelism": f"masks sharded over {world} GPU(s), no collective",
            "l2": "flushed by a 256 MiB write before every timed step; the step is enqueued behind the flush and a 0.3 ms device sleep, both outside the timed region", "path": plan_path}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def measured_peaks():
    try:
        return json.loads((REPO / "MEASURED_PEAKS.json").read_text())
    except (OSError, ValueError):
        return {}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device, self.samples, self.proc = device, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def wait_first(self, timeout=10.0):
        t0 = time.time()
        while self.proc and not self.samples and time.time() - t0 < timeout:
            time.sleep(0.05)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def cpu_baseline(iters_sample=ITERS, reps=3):
    """The reference's CPU path (oracle restatement of solve(), threaded like
    the reference's threaded:N strategy) on this host's cores."""
    from oracle import phasemask_oracle as orc
    from paper_1302_0120_b200.patterns import make_problem
    p, m = make_problem(N_PIX, SPOTS, SEED)
    cores = os.cpu_count() or 1
    gs = orc.ThreadedGS(p, m, "single", workers=cores)
    try:
        gs.run(2)                                   # warm-up (pools, FFT plans)
        times = []
        for _ in range(reps):
            t0 = time.perf_counter()
            gs.run(iters_sample)
            times.append((time.perf_counter() - t0) * 1e3)
    finally:
        gs.close()
    per_mask = statistics.median(times) * ITERS / iters_sample
    return {"value": per_mask, "unit": "ms/mask", "cores": cores, "kind": "port",
            "sample": f"{reps} x {iters_sample}-iteration 1024^2 fp32 GS masks (oracle/phasemask_oracle.py "
                      f"ThreadedGS = reference solve() with scipy.fft workers={cores} + threaded projections), "
                      f"median scaled to {ITERS} iterations"}


def run_reference(args, world, rank):
    """--impl reference: the reference algorithm on host cores (rank 0 only)."""
    if rank != 0:
        return
    from oracle import phasemask_oracle as orc
    from paper_1302_0120_b200.patterns import make_problem
    p, m = make_problem(N_PIX, SPOTS, SEED)
    cores = os.cpu_count() or 1
    gs = orc.ThreadedGS(p, m, "single", workers=cores)
    try:
        for _ in range(args.warmup):
            gs.run(ITERS)
        times = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            gs.run(ITERS)
            times.append((time.perf_counter() - t0) * 1e3)
    finally:
        gs.close()
    ms = sum(times) / len(times)
    line = {"impl": "reference", "metric": METRIC, "value": ms, "unit": "ms/mask", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": dict(workload_config(1), path="host CPU (reference algorithm, scipy.fft)",
                           l2="n/a (host)", parallelism=f"one mask per step on {cores} host threads"),
            "iters_per_s": ITERS / (ms / 1e3),
            "cpu_baseline": {"value": ms, "unit": "ms/mask", "cores": cores, "kind": "port",
                             "sample": f"one full {ITERS}-iteration 1024^2 fp32 mask per step, "
                                       f"reference solve() restated in oracle/ with scipy.fft workers={cores}"},
            "e2e": {"value": ms, "unit": "ms/mask", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def paper_config(device: int) -> dict:
    """Context, not the bench metric: the paper's own benchmark (PAPER:409,
    416-417), 25 GS iterations on an 800x600 SLM in fp32 (mixed-radix path),
    end to end through solve_stack with pinned buffers, median of 10."""
    import torch

    import paper_1302_0120_b200 as pm
    from paper_1302_0120_b200.batch import solve_stack
    from paper_1302_0120_b200.patterns import make_problem
    p, m = make_problem(800, 50, 7, n_y=600)
    cfg = pm.SolveConfig(max_iters=25, precision=pm.SINGLE, record_every=25, device=device)
    from paper_1302_0120_b200 import host_empty
    pp = host_empty(p.shape, np.float32)
    pp[...] = p
    mm = host_empty((1,) + m.shape, np.float32)
    mm[0] = m
    out = host_empty((1, 600, 800), np.float64)
    e2e, dev = [], []
    for i in range(13):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = solve_stack(pp, mm, cfg, device=device, out_phases=out)
        if i >= 3:
            e2e.append((time.perf_counter() - t0) * 1e3)
            dev.append(r.device_ms)
    return {"workload": "gs_800x600_fp32_25iter_50spots (mixed radix)", "device_ms": float(np.median(dev)),
            "e2e_ms": float(np.median(e2e)), "paper_ms": 45.0,
            "paper_hw": "Tesla C2070, incl. ~1 ms target upload (PAPER:416-417)"}


def run_batch(args, world, rank, local):
    """--config 4 (BASELINE.json configs[3]): a batch of 256 independent
    1024^2 masks (distinct 50-spot OSPs, seeds 1000..1255, one shared
    Gaussian p) sharded in contiguous blocks over the N ranks, 100 GS
    iterations fp32, no collective on the iteration path (
    the reference loops the images one by one, src/estimator.py:85-93).
    A step solves the whole job once: value = whole-job ms per mask, i.e.
    max-over-ranks device ms per step / 256; `ms_per_batch` beside it, to
    compare with the HBM-lockstep floors 164 / 82 / 41 / 20.5 ms (§8d)."""
    import torch
    import torch.distributed as dist
    import paper_1302_0120_b200 as pm
    from paper_1302_0120_b200 import _lib
    from paper_1302_0120_b200.batch import shard_bounds, solve_stack
    from paper_1302_0120_b200.patterns import make_problem, spot_targets
    from paper_1302_0120_b200.solver import _params

    total_masks = 256
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    lo, hi = shard_bounds(total_masks, world, rank)
    B = hi - lo
    prec = pm.SINGLE
    p, m0 = make_problem(N_PIX, SPOTS, 1000)
    ms = spot_targets(N_PIX, SPOTS, range(1000 + lo, 1000 + hi), dtype=np.float32)
    if lo == 0:
        assert np.array_equal(ms[0], m0.astype(np.float32))
    spec = pm.GridSpec(N_PIX, N_PIX)
    plan = pm.transform.get_plan(spec, prec, local)
    stream = torch.cuda.Stream(device=local)
    plan.set_stream(stream.cuda_stream)
    d_p = torch.from_numpy(p.astype(np.float32)).cuda(local)
    d_m = torch.from_numpy(ms).cuda(local)
    d_phase = torch.empty((B, N_PIX, N_PIX), dtype=torch.float64, device=f"cuda:{local}")
    tol_p = np.full(B, prec.zero_tol(p.astype(np.float32).max()))
    tol_m = np.full(B, prec.zero_tol(1.0))
    energy = np.full(B, float(SPOTS))               # sum m^2 of every target
    cfg = pm.SolveConfig(max_iters=ITERS, precision=prec, record_every=ITERS, device=local)
    prm = _params(cfg, False, False)
    gaps = np.full(B * ITERS, np.nan)
    iters = np.zeros(B, np.int32)

    def solve_device():
        res = _lib.pm_result()
        res.phases = _lib.C.c_void_p(d_phase.data_ptr())
        res.gap = _lib.ptr(gaps)
        res.iters_run = _lib.ptr(iters)
        _lib.check(plan.lib.pm_solve_device(plan.handle, _lib.C.c_void_p(d_p.data_ptr()),
                                            _lib.C.c_void_p(d_m.data_ptr()), None, B, prm, _lib.ptr(tol_p),
                                            _lib.ptr(tol_m), _lib.ptr(energy), res), "pm_solve_device")

    for _ in range(args.warmup):
        solve_device()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    step_ms = []
    with ClockSampler(local) as clocks:
        clocks.wait_first()
        launches0 = plan.launch_count()
        for _ in range(args.steps):                 # working set 3 GB per GPU: no L2 flush needed
            with torch.cuda.stream(stream):
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            solve_device()
            with torch.cuda.stream(stream):
                e1.record(stream)
            e1.synchronize()
            step_ms.append(e0.elapsed_time(e1))
        launches = plan.launch_count() - launches0
        time.sleep(0.2)
    assert (iters == ITERS).all() and np.isfinite(gaps[::ITERS]).all()
    total = torch.tensor([sum(step_ms)], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        dist.barrier()
        dist.all_reduce(total, op=dist.ReduceOp.MAX)
    ms_per_batch = float(total.item()) / args.steps
    value = ms_per_batch / total_masks

    # end to end through solve_stack: the rank's targets uploaded from pinned
    # memory, the 8-bit SLM levels (what an SLM displays) downloaded
    p_pin = pm.host_empty(p.shape, np.float32)          # page-locked by the library's runtime
    p_pin[...] = p
    m_pin = pm.host_empty(ms.shape, np.float32)
    m_pin[...] = ms
    lv_pin = pm.host_empty((B, N_PIX, N_PIX), np.uint8)
    e2e_ms = []
    for i in range(1 + min(args.steps, 5)):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        r = solve_stack(p_pin, m_pin, cfg, device=local, phases=False, levels=True, out_levels=lv_pin)
        if i:
            e2e_ms.append((time.perf_counter() - t0) * 1e3)
        assert (r.iters_run == ITERS).all()
    e2e = torch.tensor([sum(e2e_ms)], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(e2e, op=dist.ReduceOp.MAX)
    e2e_batch = float(e2e.item()) / len(e2e_ms)
    if rank == 0:
        peaks = measured_peaks()
        hbm = peaks.get("hbm_gbs")
        achieved = BYTES_PER_ITER * ITERS * B / (ms_per_batch * 1e-3) / 1e9   # per GPU (rank 0's share)
        floor = 40 * N_PIX * N_PIX * ITERS * total_masks / world / (6550.7e9) * 1e3
        line = {
            "metric": METRIC, "value": value, "unit": "ms/mask", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_batch, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "gs_1024x1024_fp32_100iter_50spots_batch256", "n_x": N_PIX, "n_y": N_PIX,
                       "iters": ITERS, "spots": SPOTS, "seeds": "1000..1255", "masks_per_step": total_masks,
                       "masks_per_rank": B, "record_every": ITERS,
                       "parallelism": f"256 masks in contiguous blocks over {world} GPU(s), no collective",
                       "l2": "working set 3 GB per GPU (> L2): no flush needed", "path": "persistent (TMA build)"},
            "ms_per_batch": ms_per_batch, "hbm_floor_ms_per_batch": floor,
            "iters_per_s": ITERS * total_masks / (ms_per_batch / 1e3),
            "e2e": {"value": e2e_batch / total_masks, "unit": "ms/mask", "ms_per_batch": e2e_batch,
                    "h2d_bytes_per_step": p_pin.nbytes + m_pin.nbytes, "d2h_bytes_per_step": lv_pin.nbytes,
                    "api": "paper_1302_0120_b200.batch.solve_stack(levels=True, phases=False): pinned "
                           "targets up, uint8 SLM levels down"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm if hbm else None, "traffic": None,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                         "kernel": "solve_kernel TMA build (whole batch in one launch)",
                         "bytes_per_iter": BYTES_PER_ITER},
            "clocks": clocks.summary(), "gpu_launches": launches,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# BASELINE.json configs 1, 2, 5 (single mask per GPU): (name, n, tag, algorithm, iters, spots)
SINGLE_CONFIGS = {
    1: [("gs_256x256_fp64_100iter_8spots", 256, "double", "gs", 100, 8)],
    2: [("raar_b0.9_512x512_fp32_200iter_8spots", 512, "single", "raar", 200, 8),
        ("raar_b0.9_512x512_fp64_200iter_8spots", 512, "double", "raar", 200, 8)],
    5: [("gs_4096x4096_fp32_100iter_50spots", 4096, "single", "gs", 100, 50),
        ("gs_2048x2048_fp32_100iter_50spots", 2048, "single", "gs", 100, 50)],
}


def run_single_configs(args, world, rank, local):
    """--config 1 / 2 / 5: BASELINE.json configs[0], [1], [4] with the same
    rigour as the headline (device time with CUDA events on the solve's
    stream, L2 flushed before every step, clocks sampled under load, max over
    ranks; roofline against the L2 copy roof when the working set fits L2,
    else HBM; e2e through solve() with float64 host grids). The first
    workload is the line's value, the others follow under "also"."""
    import torch
    import torch.distributed as dist
    import paper_1302_0120_b200 as pm
    from paper_1302_0120_b200 import _lib
    from paper_1302_0120_b200.patterns import make_problem
    from paper_1302_0120_b200.solver import _params

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    peaks = measured_peaks()
    hbm = peaks.get("hbm_gbs")
    l2 = _lib.measure_l2(32 << 20, 50, 1, local)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=f"cuda:{local}")
    out = []
    for name, n, tag, algo, K, spots in SINGLE_CONFIGS[args.config]:
        prec = pm.Precision.from_tag(tag)
        fdt = prec.float_dtype
        p, m = make_problem(n, spots, SEED + rank)
        spec = pm.GridSpec(n, n)
        plan = pm.transform.get_plan(spec, prec, local)
        stream = torch.cuda.Stream(device=local)
        plan.set_stream(stream.cuda_stream)
        tdt = torch.float32 if fdt == np.float32 else torch.float64
        d_p = torch.from_numpy(p.astype(fdt)).to(f"cuda:{local}", tdt)
        d_m = torch.from_numpy(m.astype(fdt)).to(f"cuda:{local}", tdt)
        d_phase = torch.empty((n, n), dtype=torch.float64, device=f"cuda:{local}")
        tol_p = np.array([prec.zero_tol(float(p.astype(fdt).max()))])
        tol_m = np.array([prec.zero_tol(float(m.astype(fdt).max()))])
        energy = np.array([float((m ** 2).sum())])
        cfg = pm.SolveConfig(max_iters=K, precision=prec, record_every=K, device=local, algorithm=algo, beta=0.9)
        prm = _params(cfg, False, False)
        iters = np.zeros(1, np.int32)

        def solve_device():
            res = _lib.pm_result()
            res.phases = _lib.C.c_void_p(d_phase.data_ptr())
            res.iters_run = _lib.ptr(iters)
            _lib.check(plan.lib.pm_solve_device(plan.handle, _lib.C.c_void_p(d_p.data_ptr()),
                                                _lib.C.c_void_p(d_m.data_ptr()), None, 1, prm, _lib.ptr(tol_p),
                                                _lib.ptr(tol_m), _lib.ptr(energy), res), "pm_solve_device")

        for _ in range(args.warmup):
            solve_device()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        step_ms = []
        with ClockSampler(local) as clocks:
            clocks.wait_first()
            t_load = time.time()
            while time.time() - t_load < 0.3:
                solve_device()
            launches0 = plan.launch_count()
            for _ in range(args.steps):
                with torch.cuda.stream(stream):
                    flush_l2(flush)
                    hold_device()
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                solve_device()
                with torch.cuda.stream(stream):
                    e1.record(stream)
                e1.synchronize()
                step_ms.append(e0.elapsed_time(e1))
            launches = plan.launch_count() - launches0
            time.sleep(0.2)
        assert iters[0] == K
        total = torch.tensor([sum(step_ms)], dtype=torch.float64, device=f"cuda:{local}")
        if world > 1:
            dist.all_reduce(total, op=dist.ReduceOp.MAX)
        ms = float(total.item()) / args.steps
        # e2e: the drop-in solve() with the caller's float64 grids
        c_in = pm.SlmConstraint(pm.RealGrid(spec, p), prec)
        m_in = pm.FourierConstraint(pm.RealGrid(spec, m), prec)
        e2e_ms = []
        for i in range(args.warmup + min(args.steps, 10)):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = pm.solve(c_in, m_in, cfg)
            if i >= args.warmup:
                e2e_ms.append((time.perf_counter() - t0) * 1e3)
            del r
        e2e_t = torch.tensor([sum(e2e_ms) / len(e2e_ms)], dtype=torch.float64, device=f"cuda:{local}")
        if world > 1:
            dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
        csz = 8 if tag == "single" else 16
        per_iter = (4 * csz + 2 * (csz // 2) + (4 * csz if algo == "raar" else 0)) * n * n
        achieved = per_iter * K / (ms * 1e-3) / 1e9
        working = (2 * csz + 2 * (csz // 2) + (2 * csz if algo == "raar" else 0)) * n * n
        in_l2 = working <= (96 << 20)
        roof = l2 if in_l2 else hbm
        out.append({
            "workload": name, "value": ms / world, "unit": "ms/mask", "ms_per_step": ms,
            "iters_per_s": K * world / (ms / 1e3), "dtype": "f32" if tag == "single" else "f64",
            "config": {"workload": name, "n_x": n, "n_y": n, "iters": K, "spots": spots, "seed": SEED,
                       "algorithm": algo, "beta": 0.9 if algo == "raar" else None, "masks_per_step": world,
                       "masks_per_rank": 1, "record_every": K, "path": "persistent" if plan.path() == 1 else "sweep-graph",
                       "l2": "flushed by a 256 MiB write before every timed step; the step is enqueued behind the flush and a 0.3 ms device sleep, both outside the timed region",
                       "parallelism": f"one mask per GPU over {world} GPU(s), no collective"},
            "e2e": {"value": float(e2e_t.item()) / world, "unit": "ms/mask",
                    "h2d_bytes_per_step": 2 * n * n * (csz // 2),
                    "d2h_bytes_per_step": n * n * (8 + 2 * csz) + 3 * K * 8 + 8,
                    "api": "paper_1302_0120_b200.solve(c, m, cfg), float64 host grids in, SolveResult out"},
            "roofline": {"bound": "l2" if in_l2 else "hbm", "achieved": achieved, "peak": roof, "unit": "GB/s",
                         "frac": achieved / roof if roof else None, "traffic": None,
                         "peak_source": ("measured in this run: pm_measure_l2 32 MiB copy" if in_l2
                                         else "MEASURED_PEAKS.json hbm_gbs"),
                         "bytes_per_iter": per_iter, "working_set_bytes": working,
                         "hbm_frac": achieved / hbm if hbm else None},
            "clocks": clocks.summary(), "gpu_launches": launches})
    if rank == 0:
        first = out[0]
        line = {"metric": METRIC, "value": first["value"], "unit": "ms/mask", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": first["ms_per_step"], "higher_is_better": False,
                "scaling": "weak", "vs_baseline": None, "dtype": first["dtype"], "data": "synthetic",
                "config": first["config"], "iters_per_s": first["iters_per_s"], "e2e": first["e2e"],
                "roofline": first["roofline"], "clocks": first["clocks"], "gpu_launches": first["gpu_launches"],
                "baseline_config": args.config, "also": out[1:]}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def flush_l2(buf):
    buf.fill_(1.0)      # 256 MiB write > the 126 MB L2


def hold_device(us: float = 300.0):
    """Keep the stream busy ~0.3 ms before the start event, so the host has
    enqueued the step's launches by the time the timed region opens: `value`
    is the device time of the solve with its inputs resident, not the
    Python/ctypes enqueue latency (that is in `e2e`)."""
    import torch
    torch.cuda._sleep(int(us * 1965))       # cycles at the B200's 1965 MHz SM clock


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--config", type=int, choices=[1, 2, 3, 4, 5], default=3,
                    help="BASELINE.json config (1-based): 3 = one 1024^2 mask per GPU (default, the headline), "
                         "4 = a 256-mask batch sharded over the GPUs, 1 / 2 / 5 = 256^2 fp64 GS / 512^2 RAAR "
                         "fp32+fp64 / 4096^2 + 2048^2 fp32 GS, one mask per GPU")
    args = ap.parse_args()
    world, rank, local = dist_env()
    if args.config == 4 and args.impl == "ours":
        run_batch(args, world, rank, local)
        return
    if args.config in SINGLE_CONFIGS and args.impl == "ours":
        run_single_configs(args, world, rank, local)
        return

    if args.impl == "reference":
        run_reference(args, world, rank)
        return

    import torch
    import torch.distributed as dist
    import paper_1302_0120_b200 as pm
    from paper_1302_0120_b200 import _lib
    from paper_1302_0120_b200.batch import solve_stack, solve_stream
    from paper_1302_0120_b200.patterns import make_problem

    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (phasemask_b200 has no CPU fallback)")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    prec = pm.SINGLE
    p, m = make_problem(N_PIX, SPOTS, SEED + rank)        # a distinct target per rank
    spec = pm.GridSpec(N_PIX, N_PIX)
    plan = pm.transform.get_plan(spec, prec, local)
    stream = torch.cuda.Stream(device=local)
    plan.set_stream(stream.cuda_stream)
    d_p = torch.from_numpy(p.astype(np.float32)).cuda(local)
    d_m = torch.from_numpy(m.astype(np.float32)).cuda(local)
    d_phase = torch.empty((N_PIX, N_PIX), dtype=torch.float64, device=f"cuda:{local}")
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=f"cuda:{local}")
    tol_p = np.array([prec.zero_tol(p.max())])
    tol_m = np.array([prec.zero_tol(m.max())])
    energy = np.array([float((m ** 2).sum())])
    cfg = pm.SolveConfig(max_iters=ITERS, precision=prec, record_every=ITERS, device=local)
    from paper_1302_0120_b200.solver import _params
    prm = _params(cfg, False, False)
    gaps = np.full(ITERS, np.nan)
    iters = np.zeros(1, np.int32)

    def solve_device():
        res = _lib.pm_result()
        res.phases = _lib.C.c_void_p(d_phase.data_ptr())
        res.gap = _lib.ptr(gaps)
        res.iters_run = _lib.ptr(iters)
        _lib.check(plan.lib.pm_solve_device(plan.handle, _lib.C.c_void_p(d_p.data_ptr()),
                                            _lib.C.c_void_p(d_m.data_ptr()), None, 1, prm, _lib.ptr(tol_p),
                                            _lib.ptr(tol_m), _lib.ptr(energy), res), "pm_solve_device")

    # ---- device-resident timing
    for _ in range(args.warmup):
        with torch.cuda.stream(stream):
            flush_l2(flush)
        solve_device()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    step_ms = []
    with ClockSampler(local) as clocks:
        clocks.wait_first()
        t_load = time.time()
        while time.time() - t_load < 0.5:          # clocks sampled under the same load
            solve_device()
        launches0 = plan.launch_count()
        for _ in range(args.steps):
            with torch.cuda.stream(stream):
                flush_l2(flush)
                hold_device()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            solve_device()
            with torch.cuda.stream(stream):
                e1.record(stream)
            e1.synchronize()
            step_ms.append(e0.elapsed_time(e1))
        torch.cuda.synchronize()
        launches = plan.launch_count() - launches0
        t_load = time.time()
        while time.time() - t_load < 0.5:
            solve_device()
        time.sleep(0.2)
    total = torch.tensor([sum(step_ms)], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        dist.barrier()
        dist.all_reduce(total, op=dist.ReduceOp.MAX)
    ms_per_step = float(total.item()) / args.steps
    value = ms_per_step / world                        # whole-job ms per mask
    assert iters[0] == ITERS and np.isfinite(gaps[0])

    # ---- end to end through the public batch API (host buffers, pinned)
    p_pin = pm.host_empty(p.shape, np.float32)          # page-locked by the library's runtime
    p_pin[...] = p
    m_pin = pm.host_empty((1,) + m.shape, np.float32)
    m_pin[0] = m
    out_pin = pm.host_empty((1, N_PIX, N_PIX), np.float64)
    e2e_ms = []
    for i in range(args.warmup + args.steps):
        with torch.cuda.stream(stream):
            flush_l2(flush)                             # cold L2, as for `value` (outside the timed call)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        r = solve_stack(p_pin, m_pin, cfg, device=local, out_phases=out_pin)
        t1 = time.perf_counter()
        if i >= args.warmup:
            e2e_ms.append((t1 - t0) * 1e3)
    e2e = torch.tensor([sum(e2e_ms)], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(e2e, op=dist.ReduceOp.MAX)
    e2e_latency = float(e2e.item()) / args.steps / world
    h2d = p_pin.nbytes + m_pin.nbytes + 3 * 8
    d2h = r.phases.nbytes + 3 * r.gap.nbytes + 4 * 2 + 40

    # ---- end to end, streamed (batch.solve_stream: the paper's frame-by-frame
    # use): every step uploads p and m and downloads the float64 mask and the
    # histories; step i+1's upload and step i-1's download overlap step i's
    # solve; the 256 MiB L2 flush runs on the solve stream between frames
    outs = [torch.empty((1, N_PIX, N_PIX), dtype=torch.float64).pin_memory().numpy() for _ in range(2)]
    m2 = m_pin[0]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    stamps = []
    n_frames = args.warmup + args.steps
    h = _lib.C.c_void_p(0)
    _lib.check(plan.lib.pm_plan_get_stream(plan.handle, _lib.C.byref(h)), "pm_plan_get_stream")
    plan_stream = torch.cuda.ExternalStream(h.value or 0, device=torch.device("cuda", local))
    for r_s in solve_stream(((p_pin, m2) for _ in range(n_frames)), cfg, device=local, out_phases=outs):
        assert r_s.iters_run[0] == ITERS
        stamps.append(time.perf_counter())
        with torch.cuda.stream(plan_stream):           # L2 flushed before the next frame's solve, as for `value`
            flush_l2(flush)
    stream_ms = torch.tensor([(stamps[-1] - stamps[args.warmup - 1]) * 1e3], dtype=torch.float64,
                             device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(stream_ms, op=dist.ReduceOp.MAX)
    e2e_value = float(stream_ms.item()) / args.steps / world
    h2d_s = p_pin.nbytes + m2.nbytes
    d2h_s = outs[0].nbytes + 3 * ITERS * 8 + 4 * 2

    # ---- end to end through the drop-in itself: the reference's entry point
    # solve(c, m, cfg) (src/solver.py:111-113) with the caller's float64 grids
    # on the host and a SolveResult (mask, u*, v*, history) back
    c_in = pm.SlmConstraint(pm.RealGrid(spec, p), prec)
    m_in = pm.FourierConstraint(pm.RealGrid(spec, m), prec)
    dropin_ms = []
    for i in range(args.warmup + args.steps):
        with torch.cuda.stream(plan_stream):
            flush_l2(flush)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        r_d = pm.solve(c_in, m_in, cfg)
        t1 = time.perf_counter()
        assert r_d.iters_run == ITERS
        if i >= args.warmup:
            dropin_ms.append((t1 - t0) * 1e3)
        del r_d
    dropin = torch.tensor([sum(dropin_ms)], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(dropin, op=dist.ReduceOp.MAX)
    dropin_value = float(dropin.item()) / args.steps / world
    h2d_d = 2 * N_PIX * N_PIX * 4                      # p and m, cast to float32 on the host
    d2h_d = N_PIX * N_PIX * (8 + 8 + 8) + 3 * ITERS * 8 + 8   # mask (float64), u*, v* (complex64), records

    if rank == 0:
        peaks = measured_peaks()
        hbm = peaks.get("hbm_gbs")
        solve_ms = ms_per_step                          # one persistent launch per step
        achieved = BYTES_PER_ITER * ITERS / (solve_ms * 1e-3) / 1e9
        # the roof: the 8 MB field (and p, m) stay in the 126 MB L2 across the
        # solve's iterations, so the bound is the L2-resident copy bandwidth
        # (read + write bytes, as the sweeps' traffic), measured here
        l2 = _lib.measure_l2(32 << 20, 50, 1, local)
        traffic = None
        tfiles = sorted((REPO / "profiles").glob("r*_ncu_traffic.json"))
        if tfiles:
            traffic = json.loads(tfiles[-1].read_text()).get("dram_bytes_per_launch")
        line = {
            "metric": METRIC, "value": value, "unit": "ms/mask", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": workload_config(world, "persistent" if plan.path() == 1 else "sweep-graph"),
            "iters_per_s": ITERS * world / (ms_per_step / 1e3),
            "e2e": {"value": e2e_value, "unit": "ms/mask", "h2d_bytes_per_step": h2d_s, "d2h_bytes_per_step": d2h_s,
                    "api": "paper_1302_0120_b200.batch.solve_stream (pinned host buffers; the uploads and "
                           "downloads of neighbouring frames overlap each solve)",
                    "latency": {"value": e2e_latency, "unit": "ms/mask", "h2d_bytes_per_step": h2d,
                                "d2h_bytes_per_step": d2h,
                                "api": "paper_1302_0120_b200.batch.solve_stack, one synchronous call per mask"},
                    "dropin": {"value": dropin_value, "unit": "ms/mask", "h2d_bytes_per_step": h2d_d,
                               "d2h_bytes_per_step": d2h_d,
                               "api": "paper_1302_0120_b200.solve(c, m, cfg): the reference's entry point, "
                                      "float64 host grids in, SolveResult (mask, u*, v*, history) out"}},
            "roofline": {"bound": "l2", "achieved": achieved, "peak": l2, "unit": "GB/s",
                         "frac": achieved / l2 if l2 else None, "traffic": traffic,
                         "peak_source": "measured in this run: pm_measure_l2, 32 MiB L2-resident copy, "
                                        "50 passes in one launch, read + write bytes",
                         "kernel": "solve_kernel (persistent; whole solve in one launch)",
                         "bytes_per_iter": BYTES_PER_ITER, "hbm_peak": hbm,
                         "hbm_frac": (achieved / hbm) if hbm else None,
                         "hbm_peak_source": "MEASURED_PEAKS.json hbm_gbs" if hbm else None},
            "clocks": clocks.summary(),
            "gpu_launches": launches,
        }
        if world == 1:
            line["paper_config"] = paper_config(local)
        if not args.no_cpu_baseline and world == 1:
            line["cpu_baseline"] = cpu_baseline()
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
