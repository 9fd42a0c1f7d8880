/*
 * phasemask_b200 — C ABI of the B200-native phase-mask solver.
 *
 * This is the drop-in boundary for the reference's hot path, the
 * Gerchberg–Saxton / alternating-projections solver of arXiv 1302.0120
 * (reference package `phasemask`, /root/reference/pkg/src/phasemask; `src/`
 * below). The reference is pure Python, so its "FFI" is the Python call
 * surface; every entry point below names the reference function it replaces.
 * The Python host layer (paper_1302_0120_b200/) binds these with ctypes —
 * see INTEGRATION.md for the binding a `phasemask` maintainer would add.
 *
 * Conventions
 *  - Grids are (n_y, n_x) row-major, flat index k*n_x + j (src/grid.py:1-6).
 *  - Complex data is interleaved re,im (numpy complex64/complex128 layout).
 *  - precision: 0 = single (float/complex64), 1 = double (src/grid.py:24-48).
 *  - Real inputs (p, m) are in the plan precision's float type.
 *  - Transforms are unitary (1/sqrt(N) split over both directions), standard
 *    unshifted frequency order (src/transform.py:1-7).
 *  - n_x and n_y are at most 4096 with prime factors 2, 3, 5, 7; powers of
 *    two run the fused register-resident kernels, other sides the
 *    mixed-radix path (GS and RAAR).
 *  - Every function returns 0 on success or a negative PM_ERR_* code;
 *    pm_last_error() returns the calling thread's last message.
 *  - "_device" variants take device pointers on the plan's device and run
 *    asynchronously on the plan's stream; the others take host pointers,
 *    copy with cudaMemcpyAsync straight from / into the caller's memory and
 *    synchronise before returning (page-locked caller buffers copy at full
 *    speed; pageable ones are staged by the CUDA driver).
 *  - No CPU fallback: without a CUDA device every compute call fails with
 *    PM_ERR_CUDA.
 */
#ifndef PHASEMASK_B200_H
#define PHASEMASK_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PM_OK              0
#define PM_ERR_ARG        -1   /* invalid argument            -> ValueError      */
#define PM_ERR_CUDA       -2   /* CUDA runtime failure        -> RuntimeError    */
#define PM_ERR_NOMEM      -3   /* cudaErrorMemoryAllocation   -> MemoryError     */
#define PM_ERR_UNSUPPORTED -4  /* size/precision not supported -> NotImplementedError */
#define PM_ERR_DIVERGED   -5   /* non-finite iterate          -> SolveDivergedError */

#define PM_SINGLE 0
#define PM_DOUBLE 1

#define PM_FORWARD  (-1)      /* exp(-2 pi i jk/n), FftProvider.forward */
#define PM_INVERSE  (+1)      /* exp(+2 pi i jk/n), FftProvider.inverse */

#define PM_ALGO_GS   0        /* alternating projections, src/solver.py:150-170 */
#define PM_ALGO_RAAR 1        /* Luke 2005 relaxed averaged alternating reflections */

typedef struct pm_plan pm_plan;

/* ------------------------------------------------------------------ misc */

/* Library version as 10000*major + 100*minor + patch. */
int pm_version(void);

/* Number of visible CUDA devices (0 when none). */
int pm_device_count(int *count);

/* Message for the calling thread's most recent failure ("" if none). */
const char *pm_last_error(void);

/* ------------------------------------------------------------------ plans */

/*
 * Create a plan for one grid and precision on `device`, with device buffers
 * for up to `max_batch` masks (grown on demand). Replaces
 * FftProvider(spec, precision, fft_workers) (src/transform.py:23-35) and the
 * service's PlanCache entry (src/service.py:65-82).
 */
int pm_plan_create(int device, int n_x, int n_y, int precision, int max_batch,
                   pm_plan **out);
int pm_plan_destroy(pm_plan *plan);

/* Use an external CUDA stream (cudaStream_t as void*; NULL = plan's own). */
int pm_plan_set_stream(pm_plan *plan, void *stream);
int pm_plan_get_stream(pm_plan *plan, void **stream);
int pm_plan_synchronize(pm_plan *plan);

/*
 * Execution path of pm_solve*: 0 = automatic (the persistent cooperative
 * kernel for square grids n >= 128 when the device supports it, else the
 * sweep-per-kernel CUDA graph), 1 = force persistent (PM_ERR_UNSUPPORTED if
 * unavailable), 2 = force the sweep graph.
 */
int pm_plan_set_path(pm_plan *plan, int path);
int pm_plan_get_path(pm_plan *plan, int *path);

/* Kernel launches issued by this plan since creation (evidence counter). */
int pm_plan_launch_count(pm_plan *plan, long long *count);

/* ------------------------------------------------------------ transforms */

/*
 * Unitary 2-D DFT of `batch` fields, in -> out (may alias).
 * Replaces FftProvider.forward / .inverse (src/transform.py:47-55),
 * i.e. scipy.fft.fft2 / ifft2(norm="ortho").
 */
int pm_fft2(pm_plan *plan, const void *in, void *out, int direction, int batch);
int pm_fft2_device(pm_plan *plan, const void *d_in, void *d_out, int direction,
                   int batch);

/* --------------------------------------------------------- projections */

/*
 * Per-pixel modulus replacement: out = mag >= zero_tol ? t*(u/|u|) : t+0i.
 * Replaces _replace_modulus / _modulus_replace_kernel
 * (src/projections.py:46-66), i.e. project_slm (t = p, :69-74) and
 * project_modulus (t = m, :77-83). `target` has `batch` grids when
 * target_per_field != 0, else one grid shared by the batch.
 */
int pm_replace_modulus(pm_plan *plan, const void *in, const void *target,
                       int target_per_field, double zero_tol, void *out, int batch);
int pm_replace_modulus_device(pm_plan *plan, const void *d_in, const void *d_target,
                              int target_per_field, double zero_tol, void *d_out,
                              int batch);

/*
 * P_M u = F^-1(replace_m(F u)) fused into three sweeps.
 * Replaces project_fourier (src/projections.py:86-91).
 */
int pm_project_fourier(pm_plan *plan, const void *u, const void *m,
                       double zero_tol_m, void *out);

/*
 * G(u) = ||P_S u - P_M u||_2 with a fixed-order fp64 reduction.
 * Replaces metrics.gap (src/metrics.py:67-71).
 */
int pm_gap(pm_plan *plan, const void *u, const void *p, const void *m,
           double zero_tol_p, double zero_tol_m, double *out_gap);

/* --------------------------------------------------------- reductions */

/*
 * sqrt(sum |x|^2): moduli in the data's precision, squared and summed in
 * fp64 in a fixed order. dtype: 0=f32 real, 1=f64 real, 2=c64, 3=c128.
 * Replaces grid.norm2 / backends.deterministic_sum (src/grid.py:161-165,
 * src/backends.py:109-125).
 */
int pm_norm2(int device, const void *data, long long count, int dtype, double *out);

/*
 * Fixed-order fp64 sum of `count` doubles (signed values allowed).
 * Replaces backends.deterministic_sum (src/backends.py:109-125).
 */
int pm_sum(int device, const double *data, long long count, double *out);

/*
 * The reference's O(N^2) correctness oracle naive_dft (src/transform.py:56-81):
 * the unitary DFT as the dense double sum W_rows X W_cols^T in fp64 on the
 * device, for grids of at most 4096 pixels (NAIVE_DFT_MAX_PIXELS, :16; larger
 * grids fail with PM_ERR_ARG and the reference's message). in / out:
 * complex128 host arrays (n_y, n_x); direction PM_FORWARD | PM_INVERSE.
 */
int pm_naive_dft(int device, const void *in, int n_x, int n_y, int direction, void *out);

/*
 * Phase extraction: out = mod(atan2(im, re), 2pi) in fp64, >= 2pi -> 0,
 * |u| < zero_tol -> 0. Replaces grid.phases_of (src/grid.py:168-176).
 */
int pm_phases(int device, const void *u, long long count, int precision,
              double zero_tol, double *out);

/*
 * Seeded random-phase start: out[b] = m[b] e^{i phi}, phi = numpy's
 * default_rng(seed).uniform(0, 2pi, count) draws from the PCG64 state
 * rng = {state hi, lo, inc hi, lo}, generated on the device (one draw per
 * pixel, shared by the `batch` masks). Host buffers; replaces the host side
 * of initial_iterate's random branch (src/solver.py:100-103).
 */
int pm_random_start(int device, const void *m, long long count, int batch, int precision,
                    const unsigned long long rng[4], void *out);

/*
 * Reconstructed intensity and its display image for `batch` fields u
 * (host, complex, plan precision): I = |F u|^2 in fp64, scaled by
 * target_energy[b] / sum(I) when target_energy is non-NULL
 * (metrics.reconstructed_intensity, src/metrics.py:74-87; a zero sum fails
 * with PM_ERR_ARG "reconstruction carries no energy"); intensity (nullable)
 * receives I in DFT order, log_image (nullable) the 8-bit log-scale image in
 * centred order, round(255 (log10(max(I/max I, floor)) - log10 floor) /
 * -log10 floor) (service._log_scale_u8 after to_centered_order,
 * src/service.py:91-95,189-194).
 */
int pm_recon_image(pm_plan *plan, const void *u, int batch, const double *target_energy,
                   double log_floor, uint8_t *log_image, double *intensity);

/* --------------------------------------------------------------- solve */

typedef struct pm_params {
    int    algorithm;        /* PM_ALGO_GS | PM_ALGO_RAAR                       */
    double beta;             /* RAAR relaxation (ignored for GS)                */
    int    max_iters;        /* >= 1                  (SolveConfig.max_iters)   */
    int    record_every;     /* >= 1               (SolveConfig.record_every)   */
    double early_stop_tol;   /* < 0: off          (SolveConfig.early_stop_tol)  */
    double t_lit, t_dark;    /* ErrorTolerances (src/metrics.py:30-39)          */
    int    p_per_mask;       /* p has `batch` grids (1) or one shared grid (0)  */
    int    init_complex;     /* 1: `m_init` holds complex Fourier-plane starts  */
    int    init_random;      /* 1: start from m e^{i phi}, phi drawn on the
                                device from the PCG64 state below exactly as
                                np.random.default_rng(seed).uniform(0, 2pi)
                                (SolveConfig.random_phase_init, :100-103)      */
    unsigned long long rng[4]; /* PCG64 state hi, lo, inc hi, lo after seeding
                                  (bit_generator.state)                        */
} pm_params;

typedef struct pm_result {
    /* host (pm_solve) or device (pm_solve_device) pointers; NULL = skip     */
    double  *phases;         /* batch*N float64 mask in [0, 2pi)              */
    uint8_t *levels;         /* batch*N uint8 SLM levels (PhaseMask.to_uint8) */
    void    *u_star;         /* batch*N complex  (SolveResult.u_star)         */
    void    *v_star;         /* batch*N complex  (SolveResult.v_star)         */
    /* always host pointers, filled after completion (NULL = skip)           */
    double  *gap;            /* batch*max_iters; NaN where not recorded       */
    double  *err_lit;        /* batch*max_iters                               */
    double  *err_dark;       /* batch*max_iters                               */
    int     *iters_run;      /* batch                                         */
    int     *diverged_iter;  /* batch; 0 = finite                             */
    float   *device_ms;      /* 1: device time of the whole solve (events)    */
} pm_result;

/*
 * Run the solver on `batch` independent masks and extract the
 * best-approximation pair and phase mask of each.
 * Replaces solver.solve (src/solver.py:111-216), including
 * initial_iterate (:93-108), the record / early-stop logic (:173-195)
 * and phases_of (:201-206); a batch replaces the sequential loop of
 * PhaseMaskTransformer.transform (src/estimator.py:85-93).
 *   p: real grid(s); m: real target moduli, batch grids;
 *   zero_tol_p / zero_tol_m: per-mask thresholds (1024*eps*max), host arrays,
 *           or both NULL to derive them on the device from p and m (an
 *           identically zero p / all-dark m then fails with PM_ERR_ARG and
 *           the reference's message, after the launch);
 *   energy: per-mask sum(m^2) in fp64 (reconstructed-intensity scale), or
 *           NULL to reduce it on the device from the (precision-cast) m;
 *   m_init: complex starts when params->init_complex, else NULL.
 * Returns PM_ERR_DIVERGED when any mask produced non-finite values
 * (result->diverged_iter says which iteration).
 */
int pm_solve(pm_plan *plan, const void *p, const void *m, const void *m_init,
             int batch, const pm_params *params, const double *zero_tol_p,
             const double *zero_tol_m, const double *energy, pm_result *result);
int pm_solve_device(pm_plan *plan, const void *d_p, const void *d_m,
                    const void *d_m_init, int batch, const pm_params *params,
                    const double *zero_tol_p, const double *zero_tol_m,
                    const double *energy, pm_result *result);

/*
 * Incremental form for per-iteration host callbacks (on_record /
 * should_abort, src/solver.py:188-199): begin, then step() one iteration at
 * a time (records for the iterations stepped become readable), then finish()
 * with abort != 0 to stop at the current iterate.
 */
int pm_solve_begin(pm_plan *plan, const void *p, const void *m, const void *m_init,
                   int batch, const pm_params *params, const double *zero_tol_p,
                   const double *zero_tol_m, const double *energy);
int pm_solve_step(pm_plan *plan, int n_iters, int *all_stopped);
int pm_solve_records(pm_plan *plan, int first_iter, int last_iter, double *gap,
                     double *err_lit, double *err_dark, int *iters_run,
                     int *diverged_iter);
int pm_solve_finish(pm_plan *plan, int abort, pm_result *result);

/*
 * Streamed form for per-iteration host callbacks without a host round trip
 * per launch (src/solver.py:188-199; SURVEY.md §8(b) record_ring /
 * abort_flag). pm_solve_async enqueues the whole single-mask solve (one
 * persistent launch on the fused path) and returns at once; the device
 * publishes every decided iteration into a host-mapped record ring, and with
 * lockstep != 0 it waits after each one for the host's verdict
 * (should_abort), answered through a host-mapped word. The caller then:
 *   for it = 1..: pm_solve_next(it) -> on_record (flags & RECORDED);
 *     stop at flags & STOP (or flags == 0: the solve ended);
 *     lockstep and not (EARLY | DIVERGED): pm_solve_answer(it, should_abort())
 *   pm_solve_wait -> the same outputs / errors as pm_solve.
 * `result` names the wanted outputs at pm_solve_async (its host arrays are
 * written by pm_solve_wait). pm_solve_next blocks without holding the GIL
 * of a ctypes caller; a device that gets no verdict for 30 s stops (TIMEOUT).
 */
typedef struct pm_record {
    double gap, err_lit, err_dark;   /* ConvergenceRecord fields (when RECORDED) */
    int    iter;                     /* 1-based iteration                        */
    int    flags;                    /* PM_REC_* bits                            */
} pm_record;
#define PM_REC_PUBLISHED 1   /* slot valid                                          */
#define PM_REC_RECORDED  2   /* a recorded iteration: on_record                     */
#define PM_REC_EARLY     4   /* early stop here (the reference skips should_abort)  */
#define PM_REC_DIVERGED  8   /* non-finite iterate (pm_solve_wait fails)            */
#define PM_REC_STOP      16  /* last iteration of the solve                         */
#define PM_REC_ABORTED   32  /* the host's abort took effect here                   */
#define PM_REC_TIMEOUT   64  /* no verdict within 30 s: stopped here; a lockstep
                                callback must not wait for work on the solving
                                device (the solve occupies every SM)            */
int pm_solve_async(pm_plan *plan, const void *p, const void *m, const void *m_init,
                   const pm_params *params, const double *zero_tol_p,
                   const double *zero_tol_m, const double *energy, int lockstep,
                   pm_result *result);
int pm_solve_next(pm_plan *plan, int iter, pm_record *record);
int pm_solve_answer(pm_plan *plan, int iter, int abort);
int pm_solve_wait(pm_plan *plan, pm_result *result);

/* ------------------------------------------------------------ measurement */

/*
 * Time `reps` launches of one sweep kernel on the plan's resident buffers
 * with CUDA events on the plan's stream (bench.py's roofline leg).
 * which: 0 = row sweep (IFFT.P_S.FFT), 1 = column sweep (FFT.P_M.IFFT).
 * Requires a prior pm_solve*_on this plan with >= batch masks.
 */
int pm_time_sweep(pm_plan *plan, int which, int batch, int reps, float *avg_ms);

/* Diagnostics: enable (1) per-phase %globaltimer stamps in the persistent
 * solve kernel, or read (0) up to n of them into `out` (ns). */
int pm_debug_phase_stamps(pm_plan *plan, int enable, unsigned long long *out, int n);

/* Device-to-device copy bandwidth over `bytes` (read+write counted), best of
 * `reps`, for the HBM (bytes >> L2) and L2 (bytes << L2) roofs. */
int pm_measure_copy(int device, long long bytes, int reps, double *gbs);

/* Page-locked host memory from the library's own CUDA runtime (transfers from
 * it run at full speed and asynchronously; the host layer's cast and output
 * buffers). Plumbing: no reference counterpart. */
int pm_host_alloc(long long bytes, void **out);
int pm_host_free(void *ptr);

/* L2 roof (SURVEY.md §8(d) "Which roof"): `passes` sweeps over an
 * L2-resident buffer of `bytes` inside one launch, L1 bypassed; mode 0 reads
 * only (bytes read), 1 copies (read + write bytes counted). Best of 4. */
int pm_measure_l2(int device, long long bytes, int passes, int mode, double *gbs);

#ifdef __cplusplus
}
#endif
#endif /* PHASEMASK_B200_H */
