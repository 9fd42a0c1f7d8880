// The solver's kernels.
//
// One Gerchberg–Saxton iteration u <- P_S F^-1 replace_m F u
// (reference src/solver.py:150-170) is executed as TWO fused sweeps over the
// field, which lives in HBM/L2 as interleaved complex (n_y, n_x) row-major:
//
//   column sweep  (col_iter_kernel):  w -> column FFT -> [metrics of u] ->
//                 replace modulus with m -> column IFFT -> z
//   row sweep     (row_iter_kernel):  z -> row IFFT -> P_S with p ->
//                 row FFT -> w
//
// Between sweeps the field is held "row-transformed" (w = RowFFT(u)), so the
// column sweep completes F(u) and the row sweep completes F^-1(v^). Each
// sweep reads and writes the field once and reads one real grid: 40 B/pixel
// per iteration in fp32, 80 B in fp64. The best-approximation
// pair and the mask come from row_final_kernel after the last column sweep.
//
// Convergence metrics (gap, err_lit, err_dark; src/metrics.py:67-112) are
// reduced on the device with a fixed-order tree (per-CTA partials + the last
// CTA of each mask combining them in index order), so they are bitwise
// reproducible run to run and independent of batch size. The last CTA of a
// column sweep also takes the stop decision (max_iters, early stop,
// non-finite), so a whole solve runs without host round trips; sweeps after
// the decision exit at their first instruction.
#pragma once
#include <cuda.h>   // CUtensorMap (the maps are encoded on the host through the driver entry point)

#include "pm_fft.cuh"

// PM_ROLL=1: one rolled copy of the transform per task (half the code);
// 0 (default, measured faster on B200): both trips unrolled.
#ifndef PM_ROLL
#define PM_ROLL 0
#endif

namespace pm {

constexpr double kTwoPi = 6.283185307179586;   // float64(2*np.pi)

// Elements between the exchange buffers of the C columns of a CTA: the
// padded transform plus 128/(E*C) so the C columns of a warp's phase land in
// distinct banks (scripts/bank_sim.py checks every configuration).
template <typename T, int SM>
__host__ __device__ __forceinline__ int col_stride(int C) {
    const int pad = 128 / (int)(sizeof(cx<T>) * C);
    return SM + (pad > 0 ? pad : 1);
}

struct MaskState {
    int stop;        // the current iterate is the last one: sweeps exit, final runs
    int done;        // nothing more to do (diverged): every launch exits
    int iters_run;   // SolveResult.iters_run
    int diverged;    // iteration whose iterate went non-finite (0 = never)
    int aborted;     // host requested stop (should_abort)
    int have_prev;   // early stop: a previous gap exists
    int bad;         // row sweep saw a non-finite value (iteration index)
    int n_records;
    double prev_gap;
    int decided;     // last iteration whose record / stop decision is taken
    int zero;        // device-side validation: 1 = p identically zero, 2 = m all dark
    double pend_lit, pend_dark;   // RAAR, sweep path: physical error of the last column sweep's iterate
    int pair_bad;    // the best-approximation pair v* went non-finite (the reference's Field check
                     // of provider.inverse in the pair, src/solver.py:202-204: a ValueError)
};

// One decided iteration, published to host-mapped memory for the host's
// callbacks (src/solver.py:188-199: on_record per record, should_abort per
// iteration). `flags` is written last, after a system-scope fence.
struct RingSlot {
    double gap, err_lit, err_dark;
    int iter;
    int flags;          // kRec* bits
};
enum : int {
    kRecPublished = 1,  // slot valid
    kRecRecorded = 2,   // a ConvergenceRecord of this iteration (on_record)
    kRecEarly = 4,      // early stop at this iteration: the reference breaks before should_abort
    kRecDiverged = 8,   // the iterate went non-finite (the reference raises)
    kRecStop = 16,      // last iteration of the solve (early stop, max_iters, divergence or abort)
    kRecAborted = 32,   // the host's abort took effect here
    kRecTimeout = 64,   // no verdict within 30 s: stopped here, the solve fails
};

struct SolveCtl {
    int max_iters;
    int record_every;
    double early_tol;   // < 0: early stopping off
    double t_lit, t_dark;
    RingSlot* ring;     // host-mapped [max_iters] (device view), null: no streaming (single mask)
    volatile int* host; // host-mapped {acknowledged iteration, abort request}
    int lockstep;       // every iteration waits for the host's verdict (should_abort)
    int decide_all;     // decide every iterate (the stepping API reads state after each step)
};

// Iterate i needs its gap: recorded, or early stopping is on (src/solver.py:173-174).
__host__ __device__ __forceinline__ bool gap_needed(const SolveCtl& c, int i) {
    return (i - 1) % c.record_every == 0 || c.early_tol >= 0.0;
}
__host__ __device__ __forceinline__ bool recorded(const SolveCtl& c, int i) { return (i - 1) % c.record_every == 0; }
// Iterate i must be decided when it is reached (record, early stop, a host verdict,
// max_iters); other iterates' decisions can wait (a non-finite iterate's first
// iteration stays in MaskState::bad until the next decision).
__host__ __device__ __forceinline__ bool decision_needed(const SolveCtl& c, int i) {
    return gap_needed(c, i) || c.lockstep || c.decide_all || i >= c.max_iters;
}

// Row-sweep modes.
enum RowMode : int {
    kRowInit = 0,    // initial iterate: no projection (src/solver.py:93-108)
    kRowGS = 1,      // GS iterate: u = P_S v
    kRowRaar = 2,    // RAAR iterate: x+ = b x + b P_S(2v - x) + (1 - 2b) v, gap of x
    kRowProbe = 3,   // RAAR: only the gap of the current x (no writes)
};

template <typename T>
struct RowArgs {
    cx<T>* field;             // source z' (and destination of w' for GS)
    cx<T>* out;               // destination of w' (GS: == field; RAAR: the second field buffer)
    const T* p;
    long long p_stride;       // elements between masks' p (0: shared)
    const twe<T>* twf;        // forward twiddles
    const twe<T>* twi;        // inverse twiddles (fp64: same as twf)
    int nx, ny;
    T scale;                  // S = 1/sqrt(nx*ny)
    const double* thr_p;      // [batch] zero tolerance (T-rounded) of P_S
    int mode;                 // RowMode
    int it;                   // index of the iterate this sweep produces
    MaskState* st;
    // RAAR; unused by GS
    cx<T>* x;                 // [batch][N] iterate x (SLM plane, true scale)
    T beta, c1;               // beta and 1 - 2 beta, rounded to T as numpy does (NEP 50)
    const double* thr_x;      // [batch] P_S zero tolerance (T-rounded) on true-scale values
    double* rpart;            // [batch][ny * wpr][2]: gap^2 of x_{it-1}, |x_it|^2, per row warp
    int wpr;                  // partial slots per row: max(1, TG / 32)
    SolveCtl ctl;
    double* hist;
    int hist_stride;
    const double* cpart;      // persistent path: lit/dark partials of the column sweeps
    long long cpart_alt;      // offset of the odd-iteration buffer in cpart
    int tpm;                  // column tasks per mask (persistent path)
    unsigned* ctr;
    int nblk;                 // row CTAs per mask (sweep path ticket)
};

template <typename T>
struct FinalArgs {
    const cx<T>* field;
    const T* p;
    long long p_stride;
    const twe<T>* tw;         // forward row twiddles
    int nx, ny;
    T scale;
    const double* tol_p;      // [batch] reference zero_tol (compared to |u|)
    MaskState* st;
    cx<T>* v_star;            // outputs, nullable
    cx<T>* u_star;
    double* phases;
    uint8_t* levels;
    // RAAR: gap of the last iterate x_K = ||P_S x_K - v*|| (null x for GS)
    const cx<T>* x;
    const double* thr_x;
    double* rpart;
    int wpr;
    SolveCtl ctl;
};

template <typename T>
struct ColArgs {
    cx<T>* field;             // destination z' (and source for GS / init)
    const cx<T>* in;          // source w' of an iterate sweep (GS: == field)
    int raar;                 // RAAR: energy scale from the row partials, lit/dark kept for the row decision
    const double* xpart;      // RAAR: row partials ([batch][ny * wpr][2], component 1 = |x|^2)
    int xparts;               // ny * wpr
    const double* energy;     // [batch] sum m^2
    long long part_alt;       // persistent RAAR: offset of the odd-iteration partial buffer
    const T* m;
    long long m_stride;
    const T* mT;              // persistent column phase: m transposed per mask ([batch][nx][ny], same
                              // stride), so a task's m is one contiguous run (null: stage from m)
    const twe<T>* twf;
    const twe<T>* twi;
    int nx, ny;
    T scale;                  // S = 1/sqrt(nx*ny)
    const double* thr_m;      // [batch] zero tolerance (T-rounded) on u^
    const double* escale;     // [batch] sum m^2 / sum |u|^2 (reconstructed-intensity scale)
    int mode;                 // 0: init from real m, 1: init from complex field, 2: iterate
    int u_iter;               // metrics of iterate u_{u_iter} (0 = none)
    SolveCtl ctl;
    MaskState* st;
    double* hist;             // [batch][hist_stride][4] = gap, err_lit, err_dark, recorded
    int hist_stride;
    double* part;             // [batch][nblk][3]
    unsigned* ctr;
    int nblk;
};

// Lanes 0..nl-1 (every lane of this warp present in the CTA).
__device__ __forceinline__ unsigned lane_mask(int nl) { return nl >= 32 ? 0xffffffffu : (1u << nl) - 1u; }

// Fixed-order warp sum that tolerates partial warps (CTAs of < 32 threads):
// lanes outside the CTA contribute nothing. Lane 0 holds the result.
__device__ __forceinline__ double warp_sum(double x) {
    const int lane = threadIdx.x & 31;
    const int nl = min(32, (int)blockDim.x - (int)(threadIdx.x & ~31u));
    const unsigned mask = lane_mask(nl);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        const double y = __shfl_xor_sync(mask, x, o);
        if ((lane ^ o) < nl) x += y;
    }
    return x;
}

// Fixed-order block reduction of NV fp64 accumulators into this CTA's
// partial slot, then a ticket; returns true in the last CTA of the mask,
// whose thread 0 receives the totals (combined in block-index order).
template <int NV>
__device__ __forceinline__ bool reduce_ticket(double (&acc)[NV], double* part, unsigned* ctr,
                                              int nblk, int blk, double (&tot)[NV]) {
    __shared__ double wsum[32][NV];
    __shared__ int s_last;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nw = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        const double x = warp_sum(acc[v]);
        if (lane == 0) wsum[warp][v] = x;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            double s = 0.0;
            for (int w = 0; w < nw; ++w) s += wsum[w][v];
            part[blk * NV + v] = s;
        }
        __threadfence();
        const unsigned t = atomicAdd(ctr, 1u);
        s_last = (t == (unsigned)(nblk - 1));
    }
    __syncthreads();
    if (!s_last) return false;
    __threadfence();
    if (warp == 0) {
        const int stride = min(32, (int)blockDim.x);
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            double x = 0.0;
            for (int i = lane; i < nblk; i += stride) x += __ldcg(&part[i * NV + v]);
            x = warp_sum(x);
            if (lane == 0) tot[v] = x;
        }
    }
    if (threadIdx.x == 0) *ctr = 0u;
    return true;
}

// Phase of the complex128-cast value, np.mod(., 2pi) semantics, >= 2pi -> 0
// (src/grid.py:168-176).
__device__ __forceinline__ double phase_of(double re, double im) {
#if PM_EXP_NOATAN
    double th = im - re;          // experiment only: the cost of atan2 in the final pass
#else
    double th = atan2(im, re);
#endif
    if (th < 0.0) th = th + kTwoPi;
    else th = th + 0.0;                 // -0 -> +0 as np.mod does
    if (th >= kTwoPi) th = 0.0;
    return th;
}

__device__ __forceinline__ uint8_t level_of(double th) {
    double l = rint(th / kTwoPi * 256.0);   // np.round: half to even
    l = l < 0.0 ? 0.0 : (l > 255.0 ? 255.0 : l);
    return (uint8_t)l;
}

// Groups of <= 32 threads live inside one warp and synchronise with a warp
// barrier; larger groups use the CTA barrier.
template <int TG> struct GroupSync { using type = SyncBlock; };
template <> struct GroupSync<1> { using type = SyncWarp; };
template <> struct GroupSync<2> { using type = SyncWarp; };
template <> struct GroupSync<4> { using type = SyncWarp; };
template <> struct GroupSync<8> { using type = SyncWarp; };
template <> struct GroupSync<16> { using type = SyncWarp; };
template <> struct GroupSync<32> { using type = SyncWarp; };

// The synchroniser of row group g: a warp barrier for TG <= 32, else named
// barrier 1+g over the group's TG threads.
template <int TG>
__device__ __forceinline__ auto group_sync(int g) {
    if constexpr (TG <= 32) return SyncWarp{};
    else return SyncNamed{1 + g, TG};
}

template <typename C> __device__ __forceinline__ auto norm_sq(C u) { return u.x * u.x + u.y * u.y; }

// Per-mask decision after the metrics of iterate u_i are reduced: record,
// early stop, divergence, max_iters (src/solver.py:173-199). Runs in one
// thread; `tot` = {gap^2, err_lit, err_dark}.
__device__ __forceinline__ void decide(MaskState* st, double* hist_row, const SolveCtl& ctl, int i, bool rec,
                                       const double (&tot)[3]) {
    const double g = sqrt(tot[0]);
    int stop = 0;
    // divergence = a non-finite field (the sweeps' explicit checks); an
    // overflowing gap of a finite field is recorded as is, like the reference's
    if (st->bad) {
        st->diverged = st->bad;
        st->done = 1;
        stop = 1;
    }
    if (rec) {
        hist_row[0] = g; hist_row[1] = tot[1]; hist_row[2] = tot[2]; hist_row[3] = 1.0;
        st->n_records += 1;
    }
    bool early = false;
    if (ctl.early_tol >= 0.0) {
        if (st->have_prev && g > 0.0 && fabs(g - st->prev_gap) <= ctl.early_tol * g) stop = 1, early = true;
        st->prev_gap = g;
        st->have_prev = 1;
    }
    if (i >= ctl.max_iters) stop = 1;
    st->decided = i;
    if (ctl.ring) {
        // stream the decision to the host; with lockstep, wait for its verdict
        // (should_abort, polled once per iteration after on_record, unless the
        // iteration stopped early or diverged: src/solver.py:188-199)
        RingSlot* r = ctl.ring + (i - 1);
        r->gap = rec ? hist_row[0] : 0.0;
        r->err_lit = rec ? hist_row[1] : 0.0;
        r->err_dark = rec ? hist_row[2] : 0.0;
        r->iter = i;
        int fl = kRecPublished | (rec ? kRecRecorded : 0) | (early ? kRecEarly : 0) | (st->bad ? kRecDiverged : 0);
        const bool ask = ctl.lockstep && !early && !st->bad;
        if (!ask && stop) fl |= kRecStop;
        __threadfence_system();
        *(volatile int*)&r->flags = fl;
        if (ask) {
            // bounded wait: a host that never answers (e.g. a callback that itself
            // waits for this device) must not hang it; after 30 s the solve stops
            // and reports the timeout
            unsigned long long t0, t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
            int abort = 0;
            for (;;) {
                if (ctl.host[1]) { abort = kRecAborted; break; }
                if (ctl.host[0] >= i) break;
                __nanosleep(200);
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
                if (t - t0 > 30000000000ull) { abort = kRecTimeout; break; }
            }
            if (abort) {
                stop = 1;
                st->aborted = 1;
            }
            if (stop) {
                __threadfence_system();
                *(volatile int*)&r->flags = fl | kRecStop | abort;
            }
        }
    }
    if (stop) {
        st->stop = 1;
        st->iters_run = i;
    }
}

// Fixed-order sum of n values p[0], p[s], p[2s], ... by one warp (the lanes
// present when the CTA is smaller than a warp): lane l takes l, l+nl, ...,
// then a xor tree. Lane 0 holds the total.
__device__ __forceinline__ double warp_sum_strided(const double* p, int n, int s) {
    const int lane = threadIdx.x & 31;
    const int nl = min(32, (int)blockDim.x - (int)(threadIdx.x & ~31u));
    double x = 0.0;
    for (int i = lane; i < n; i += nl) x += __ldcg(p + (size_t)i * s);
    return warp_sum(x);
}

// RAAR decision for iterate i of mask b, by one full warp (SURVEY.md §8 a15:
// the reference's record / early-stop logic applied to the RAAR iterate).
// gap^2 comes from the row partials; lit/dark from `lit_dark` (host of the
// persistent path: column-task partials [tpm][3]; sweep path: MaskState).
__device__ __forceinline__ void decide_raar_warp(MaskState* st, double* hist, int hist_stride, const SolveCtl& ctl,
                                                 int b, int i, const double* gparts, int ngp,
                                                 const double* cparts, int ncp) {
    if (i < 1 || __ldcg(&st->decided) >= i || __ldcg(&st->done)) return;
    const bool rec = recorded(ctl, i);
    double tot[3] = {0.0, 0.0, 0.0};
    if (gap_needed(ctl, i)) tot[0] = warp_sum_strided(gparts, ngp, 2);
    if (rec) {
        if (cparts) {
            tot[1] = warp_sum_strided(cparts + 1, ncp, 3);
            tot[2] = warp_sum_strided(cparts + 2, ncp, 3);
        } else {
            tot[1] = __ldcg(&st->pend_lit);
            tot[2] = __ldcg(&st->pend_dark);
        }
    }
    if ((threadIdx.x & 31) == 0) decide(st, hist + ((size_t)b * hist_stride + (i - 1)) * 4, ctl, i, rec, tot);
}

// Group-wide sums of two per-thread values over the TG threads of a row
// group (xor tree inside each warp); lane 0 of every warp of the group
// stores its warp's sums into dst[w][0..1]. Called by all threads.
template <int TG>
__device__ __forceinline__ void row_partials(double g2, double e2, double* dst, int j, bool store) {
    constexpr int W = TG < 32 ? TG : 32;
    const unsigned mask = lane_mask(min(32, (int)blockDim.x - (int)(threadIdx.x & ~31u)));
#pragma unroll
    for (int o = W / 2; o >= 1; o >>= 1) {
        g2 += __shfl_xor_sync(mask, g2, o);
        e2 += __shfl_xor_sync(mask, e2, o);
    }
    if (store && (j & 31) == 0) {
        dst[(j >> 5) * 2 + 0] = g2;
        dst[(j >> 5) * 2 + 1] = e2;
    }
}

// Round-to-nearest complex helpers with no FMA contraction, for the RAAR
// combine, which must follow numpy's operation order.
__device__ __forceinline__ float2 cmul_rn(float2 a, float s) { return mul2(a, make_float2(s, s)); }
__device__ __forceinline__ double2 cmul_rn(double2 a, double s) { return make_double2(__dmul_rn(a.x, s), __dmul_rn(a.y, s)); }
__device__ __forceinline__ float2 cadd_rn(float2 a, float2 b) { return add2(a, b); }
__device__ __forceinline__ double2 cadd_rn(double2 a, double2 b) { return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y)); }
__device__ __forceinline__ float2 csub_rn(float2 a, float2 b) { return sub2(a, b); }
__device__ __forceinline__ double2 csub_rn(double2 a, double2 b) { return make_double2(__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y)); }

template <typename C> __device__ __forceinline__ double norm_sq_d(C u) {
    return (double)u.x * (double)u.x + (double)u.y * (double)u.y;
}

// Non-finite detector of the reference's Field checks (src/grid.py:100-110):
// chk stays 0 while every value folded in is finite (v * 0 is NaN for inf or
// NaN), one packed FMA per complex value; magnitudes are never squared, so
// large finite fields (|u|^2 beyond the float range) are not flagged.
__device__ __forceinline__ void fold_finite(float2& chk, float2 v) { chk = fma2(v, make_float2(0.f, 0.f), chk); }
__device__ __forceinline__ void fold_finite(double2& chk, double2 v) {
    chk.x = fma(v.x, 0.0, chk.x);
    chk.y = fma(v.y, 0.0, chk.y);
}
template <typename C> __device__ __forceinline__ bool all_finite(C chk) { return chk.x == 0 && chk.y == 0; }

// Record the first iteration whose iterate went non-finite (decisions may be
// taken only every few iterations; the reference reports the first).
__device__ __forceinline__ void first_bad(int* bad, int it) {
    if (__ldcg(bad) == 0) atomicCAS(bad, 0, it);
}

template <typename T> __device__ __forceinline__ T min_normal();
template <> __device__ __forceinline__ float min_normal<float>() { return 1.17549435e-38f; }
template <> __device__ __forceinline__ double min_normal<double>() { return 2.2250738585072014e-308; }

// Cross-CTA field loads bypass L1 (the field is rewritten between phases).
template <typename C> __device__ __forceinline__ C ld_field(const C* p) { return __ldcg(p); }

// Fine-grained clock64 stamps inside tasks (experiments only: PM_FINE=1):
// CTA thread 0 writes the SM clock into slots 128.. of its stamp row.
#ifndef PM_FINE
#define PM_FINE 0
#endif

struct FineState {
    unsigned long long* p;
    int i;
};
__device__ __forceinline__ FineState& fine_state() {
    __shared__ FineState s;
    return s;
}
__device__ __forceinline__ void fine_init(unsigned long long* stamps) {
    if constexpr (PM_FINE) {
        if (threadIdx.x == 0) {
            fine_state().p = stamps ? stamps + (size_t)blockIdx.x * 1024 + 128 : nullptr;
            fine_state().i = 0;
        }
        __syncthreads();
    }
}
__device__ __forceinline__ void fine_stamp(int id) {
    if constexpr (PM_FINE) {
        if (threadIdx.x == 0) {
            FineState& s = fine_state();
            if (s.p && s.i < 894) {
                s.p[s.i] = id;
                s.p[s.i + 1] = clock64();
                s.i += 2;
            }
        }
    }
}
// A stamp taken once value x has arrived (forces the scoreboard wait).
template <typename V>
__device__ __forceinline__ void fine_stamp_after(V x, int id) {
    if constexpr (PM_FINE) {
        if (threadIdx.x == 0) {
            FineState& s = fine_state();
            if (s.p && x.x == 1.2345e-30f && x.y == 5.4321e-30f) s.p[895] = 0;
        }
        fine_stamp(id);
    }
}

// ------------------------------------------------------------------ tasks
// Scaling convention: the unitary factor S = 1/sqrt(n_x n_y) is applied
// once per half iteration, at the projections, as the targets' scale: P_S
// writes S u (p pre-scaled by S on the device once per solve; RAAR scales
// its combine), the column replace writes S v^. The field between phases
// is then w'' = RowFFT(S u) = S RowFFT(u) and conj(z'') with
// z'' = S ColIFFT(v^) (unnormalised transforms of the scaled values), so the
// column phase's ColFFT(w'') IS u^ = F(u) and the row phase's RowFFT(conj z'')
// IS conj(v): both projections decide on the normalised values against the
// reference's zero_tol itself, and every intermediate stays within
// sqrt(n) of a normalised transform, as scipy's (DUCC scales by S after
// the first axis), so overflow happens where the reference's does.

// ------------------------------------------------------- shared staging
// cp.async copies of a task's real grid (p or m) into shared memory, issued
// with the field loads so their latency overlaps the first transform
// (persistent kernel; the sweep kernels read the grid from global memory).
template <int BYTES>
__device__ __forceinline__ void cp_async(void* dst, const void* src) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    if constexpr (BYTES == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(d), "l"(src), "n"(BYTES) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
// Wait until at most N of this thread's most recent groups are pending
// (groups complete in commit order).
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// ---------------------------------------------------------------- TMA
// Tensor-memory-accelerator copies (cp.async.bulk.tensor) completing on an
// mbarrier: one elected thread moves a whole column tile into shared memory
// while the CTA computes, with no load instructions on the LSU path.
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z,
                                            unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
        ::"r"(smem_u32(dst)), "l"(map), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}

// Copies completed on each row group's mbarrier (row TMA; their parity),
// zeroed at kernel start.
__device__ __forceinline__ unsigned* row_loads() {
    __shared__ unsigned s[16];
    return s;
}

// Contiguous global -> shared copy by the tensor accelerator (bytes % 16 == 0).
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// TMA tensor store from shared memory (bulk async-group of the issuing thread).
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int x, int y, int z) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];"
                 ::"l"(map), "r"(x), "r"(y), "r"(z), "r"(smem_u32(src)) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// the issuing thread's stores have read their shared-memory source
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
// ... and are complete in global memory (then ordered before the generic
// proxy's later accesses: the grid barrier's release publishes them)
__device__ __forceinline__ void bulk_wait_all() {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

// No prefetch: the sweep kernels and single-task phases.
struct NoPrefetch {
    __device__ __forceinline__ void operator()() const {}
};

// Copy `rows` runs of `run` contiguous elements (global stride `gstride`)
// into a dense [rows][run] shared array, with `nthr` threads (thread `t`),
// in copies of CH bytes (CH divides run * sizeof(T)).
template <typename T, int CH>
__device__ __forceinline__ void stage_runs(T* dst, const T* src, int rows, int run, size_t gstride, int t,
                                           int nthr) {
    constexpr int EPC = CH / (int)sizeof(T);                     // elements per copy
    const int cpr = run / EPC;                                   // copies per run
    for (int i = t; i < rows * cpr; i += nthr) {
        const int r = i / cpr, q = i - r * cpr;
        cp_async<CH>(dst + (size_t)r * run + q * EPC, src + r * gstride + q * EPC);
    }
}

// Conjugate storage. Between a column sweep and the next row sweep the field
// holds conj(z'), z' = ColIFFT(v^) unnormalised; both sweeps then run only
// FORWARD transforms, because IFFT(x) = conj(FFT(conj(x))):
//   row:    y = RowFFT(conj z') = conj(v')   -> u = conj(P_S(y)) = P_S(v')
//           (the conjugation folds into the projection's multiply) -> RowFFT(u)
//   column: u^ = S ColFFT(w') -> conj(v^) = conj(replace_m(u^)) (folded again)
//           -> ColFFT(conj v^) = conj(ColIFFT(v^)) = conj(z').
// One transform direction means one copy of the FFT code per task (a
// two-trip loop, not unrolled, keeps the hot loop inside the instruction
// cache) and one twiddle table.

// stage_runs with every extent known at compile time (power-of-two copies per
// run): no division, a fixed trip count per thread.
template <typename E, int ROWS, int RUN, int NTHR>
__device__ __forceinline__ void stage_tile(E* dst, const E* src, size_t gstride, int t) {
    constexpr int CH = RUN * (int)sizeof(E) >= 16 ? 16 : RUN * (int)sizeof(E);
    constexpr int EPC = CH / (int)sizeof(E);
    constexpr int CPR = RUN / EPC;
    constexpr int TOT = ROWS * CPR;
    static_assert(CPR * EPC == RUN && (CPR & (CPR - 1)) == 0, "runs must split into power-of-two copies");
#pragma unroll 4
    for (int i = t; i < TOT; i += NTHR) {
        const int r = i / CPR, q = i % CPR;
        cp_async<CH>(dst + (size_t)r * RUN + q * EPC, src + r * gstride + q * EPC);
    }
}

// stage_tile into rows of DSTR elements (DSTR >= RUN; DSTR * sizeof(E) a
// multiple of the copy size).
template <typename E, int ROWS, int RUN, int DSTR, int NTHR>
__device__ __forceinline__ void stage_tile_s(E* dst, const E* src, size_t gstride, int t) {
    constexpr int CH = RUN * (int)sizeof(E) >= 16 ? 16 : RUN * (int)sizeof(E);
    constexpr int EPC = CH / (int)sizeof(E);
    constexpr int CPR = RUN / EPC;
    constexpr int TOT = ROWS * CPR;
    static_assert(CPR * EPC == RUN && (CPR & (CPR - 1)) == 0 && (DSTR * (int)sizeof(E)) % CH == 0,
                  "runs must split into power-of-two aligned copies");
#pragma unroll 4
    for (int i = t; i < TOT; i += NTHR) {
        const int r = i / CPR, q = i % CPR;
        cp_async<CH>(dst + (size_t)r * DSTR + q * EPC, src + r * gstride + q * EPC);
    }
}

// Row stride of the transposed m tile of a column task: ny plus a pad that
// spreads the C columns of a warp over distinct banks (and keeps 16-byte rows).
template <typename T, int NY, int CC>
struct MtStride {
    static constexpr int PAD0 = CC > 0 ? 32 / CC : 1;
    static constexpr int Q = 16 / (int)sizeof(T);
    static constexpr int PAD = (PAD0 + Q - 1) / Q * Q;
    static constexpr int V = NY + PAD;
};

// A row task: the TG threads of group g transform one row. `inb` == false
// (row beyond the batch) runs the same instruction stream on zeros without
// touching memory, so group barriers stay aligned when a CTA has fewer rows
// than groups; `live` == false (mask already stopped) loads but stores
// nothing. `tw` is the forward row table (a shared copy when TS); `ps`, when
// PS, is this row's slice of p staged in shared memory.
// ALG selects the code compiled in: 0 GS modes only, 1 RAAR modes only,
// -1 both (the persistent kernel instantiates one algorithm at a time so the
// other's registers do not count against it).
//
// Cross-task prefetch (persistent kernel, PF): when `tile` is non-null the
// row's input was copied into shared memory by the previous task through
// cp.async; `prefetch()` starts the copy of the next task's input. cp.async
// groups per task, in commit order: [p of this task] [next task's field],
// so the projection waits for one group and leaves the prefetch in flight.
// `xs` (XS, RAAR): this row's slice of x staged with p.
template <typename T, int LG_L, int LG_R, class Sync, int ALG = -1, int TS = 0, bool PS = false,
          class Prefetch = NoPrefetch, bool XS = false>
__device__ __forceinline__ void row_task(const RowArgs<T>& a, int b, int row, int j, cx<T>* sm,
                                         const twe<T>* tw, T* ps, bool inb_arg, bool live, Sync sync,
                                         const cx<T>* tile = nullptr, Prefetch prefetch = Prefetch{},
                                         cx<T>* xs = nullptr, bool stage_p = true,
                                         unsigned long long* tbar = nullptr, unsigned tpar = 0) {
    using F = FftShape<LG_L, LG_R>;
    const size_t N = (size_t)a.nx * a.ny;
    // whole-warp groups never run out of bounds (the row phase skips them)
    const bool inb = F::TG >= 32 ? true : inb_arg;
    const bool act = inb && live;
    cx<T>* f = a.field + b * N + (size_t)row * a.nx + j;
    const T* p = a.p + b * a.p_stride + (size_t)row * a.nx + j;
    // the mask's zero tolerance, loaded with the field (its L2 latency then
    // overlaps the loads instead of stalling the projection)
    const double thr_b = (ALG != 1 && a.mode == kRowGS) ? __ldcg(a.thr_p + b)
                       : (ALG != 0 && (a.mode == kRowRaar || a.mode == kRowProbe)) ? __ldcg(a.thr_x + b) : 0.0;
    cx<T> v[F::R];
    if (tile) {
        // tbar: the tile was copied by the tensor accelerator (row TMA); else by cp.async (PF)
        if (tbar) mbar_wait(tbar, tpar);
        else cp_async_wait<0>();
        sync();
#pragma unroll
        for (int k = 0; k < F::R; ++k) v[k] = tile[j + F::TG * k];                           // conj(z')
        sync();                                                                               // tile free
    } else {
#pragma unroll
        for (int k = 0; k < F::R; ++k) v[k] = inb ? ld_field(f + F::TG * k) : mk<T>(T(0), T(0));   // conj(z')
    }
    fine_stamp_after(v[F::R - 1], 11);   // row: loads landed
    if constexpr (PS) {
        if (inb && a.mode != kRowInit && stage_p) stage_tile<T, 1, (1 << LG_L), F::TG>(ps, p - j, 0, j);
        if constexpr (XS) {
            if (inb && (a.mode == kRowRaar || a.mode == kRowProbe))
                stage_tile<cx<T>, 1, (1 << LG_L), F::TG>(xs, a.x + b * N + (size_t)row * a.nx, 0, j);
        }
        cp_async_commit();
    }
    prefetch();
    cp_async_commit();
    auto p_at = [&](int k) -> T {
        if constexpr (PS) return ps[j + F::TG * k];
        else return p[F::TG * k];
    };
    // two trips through one copy of the transform; the trip count is opaque
    // to the compiler (a.ny >= 1 at run time) so it keeps the loop rolled
#if PM_ROLL
    const int trips = 1 + (a.ny > 0);
#pragma unroll 1
#else
    constexpr int trips = 2;
#pragma unroll
#endif
    for (int h = 0; h < trips; ++h) {
        if (h) fine_stamp_after(v[F::R - 1], 14);               // row: after the projection
        fft1d<T, LG_L, LG_R, -1, TS>(v, sm, tw, j, sync);     // h = 0: y = conj(v'); h = 1: w' = RowFFT(u)
        fine_stamp_after(v[F::R - 1], 12 + h);   // row: after FFT 1 / 2
        if (h) break;
        if constexpr (PS) {
            if (stage_p || XS) {                     // (resident p: nothing was copied for this task)
                cp_async_wait<1>();                  // p of this task (the prefetch may stay in flight)
                sync();
            }
        }
        if (ALG != 1 && a.mode == kRowGS) {
            // S u = S P_S v = conj(P_S(y; S p)) (src/projections.py:69-74): y = conj(v) is
            // the normalised field, decided against zero_tol itself; p arrives pre-scaled by S
            const ZThr<T> z = zthr<T>(T(thr_b));
            auto t_of = [&](int k) -> T { return inb ? p_at(k) : T(0); };
            auto keep = [](int, cx<T>, cx<T> o) { return o; };
            // false: v = F^-1 v^ was not finite (the reference's Field check)
            const bool fin = project_regs<true>(v, z, t_of, keep);
            if (act && !fin) first_bad(&a.st[b].bad, a.it);
        } else if (a.mode == kRowInit) {
            cx<T>* xp = (ALG != 0 && a.x) ? a.x + b * N + (size_t)row * a.nx + j : nullptr;
#pragma unroll
            for (int k = 0; k < F::R; ++k) {
                const cx<T> u0 = cconj(v[k]);                             // u0 = F^-1 m (src/solver.py:105-108)
                if (xp && act) xp[F::TG * k] = u0;                        // RAAR: x_0 = u0
                v[k] = cscale(u0, a.scale);                               // the row FFT of S u0 follows
            }
        } else if (ALG != 0) {
            // RAAR, v = P_M x_{it-1} = conj(y), p at true scale:
            //   gap of x_{it-1} = ||P_S x_{it-1} - v|| (src/metrics.py:67-71), when needed;
            //   x_it = beta x + beta P_S(2v - x) + (1 - 2 beta) v, numpy's operation order.
            const int gi = a.it - 1;
            const bool gneed = act && gi >= 1 && gap_needed(a.ctl, gi) && __ldcg(&a.st[b].decided) < gi;
            const bool upd = a.mode == kRowRaar;
            const ZThr<T> z = zthr<T>(T(thr_b));
            cx<T>* xp = a.x + b * N + (size_t)row * a.nx + j;
            double g2 = 0.0, e2 = 0.0;
#pragma unroll
            for (int k = 0; k < F::R; ++k) {
                const cx<T> vv = cconj(v[k]);
                cx<T> xo;
                if constexpr (XS) xo = inb ? xs[j + F::TG * k] : mk<T>(T(0), T(0));
                else xo = inb ? ld_field(xp + F::TG * k) : mk<T>(T(0), T(0));
                const T pk = inb ? p_at(k) : T(0);
                if (gneed) g2 += norm_sq_d(csub_rn(replace_mod(xo, pk, z), vv));
                if (upd) {
                    const cx<T> py = replace_mod(csub_rn(cscale(vv, T(2)), xo), pk, z);
                    const cx<T> xn = cadd_rn(cadd_rn(cmul_rn(xo, a.beta), cmul_rn(py, a.beta)), cmul_rn(vv, a.c1));
                    if (act) xp[F::TG * k] = xn;
                    e2 += norm_sq_d(xn);
                    v[k] = cscale(xn, a.scale);                           // the row FFT of S x_it follows
                }
            }
            if (upd && act && !isfinite(e2)) first_bad(&a.st[b].bad, a.it);
            row_partials<F::TG>(g2, e2, a.rpart + ((size_t)b * a.ny + row) * a.wpr * 2, j, act);
            if (!upd) {
                if constexpr (PS) sync();              // ps is restaged by the next task
                return;
            }
        }
    }
    if (act) {
        cx<T>* o = a.out + (f - a.field);
#pragma unroll
        for (int k = 0; k < F::R; ++k) o[F::TG * k] = v[k];
    }
    fine_stamp(15);   // row: stores issued
}

// Best-approximation pair for one row: v* = P_M u_K = S * RowIFFT(z')
// = S * conj(RowFFT(conj z')), u* = P_S v*, mask = phases_of(u*, zero_tol_p)
// (src/solver.py:201-206, src/grid.py:168-176).
template <typename T, int LG_L, int LG_R, int TS = 0, class Sync>
__device__ __forceinline__ void final_task(const FinalArgs<T>& a, int b, int row, int j, cx<T>* sm,
                                           const twe<T>* tw, bool act, Sync sync) {
    using F = FftShape<LG_L, LG_R>;
    const size_t N = (size_t)a.nx * a.ny;
    const size_t o = b * N + (size_t)row * a.nx + j;
    const T* p = a.p + b * a.p_stride + (size_t)row * a.nx + j;
    cx<T> v[F::R];
#pragma unroll
    for (int k = 0; k < F::R; ++k) v[k] = act ? ld_field(a.field + o + F::TG * k) : mk<T>(T(0), T(0));
    fft1d<T, LG_L, LG_R, -1, TS>(v, sm, tw, j, sync);
    cx<T> chk = mk<T>(T(0), T(0));
#pragma unroll
    for (int k = 0; k < F::R; ++k) {
        v[k] = cconj(v[k]);                                                // v* (normalised)
        fold_finite(chk, v[k]);
    }
    if (act && !all_finite(chk)) a.st[b].pair_bad = 1;
    if (a.x) {
        // RAAR: gap of the last iterate, ||P_S x_K - P_M x_K|| with P_M x_K = v*
        const int i = a.ctl.max_iters;
        const bool gneed = act && !__ldcg(&a.st[b].stop) && gap_needed(a.ctl, i) && __ldcg(&a.st[b].decided) < i;
        double g2 = 0.0;
        if (gneed) {
            const ZThr<T> z = zthr<T>(T(a.thr_x[b]));
#pragma unroll
            for (int k = 0; k < F::R; ++k)
                g2 += norm_sq_d(csub_rn(replace_mod(ld_field(a.x + o + F::TG * k), p[F::TG * k], z), v[k]));
        }
        row_partials<F::TG>(g2, 0.0, a.rpart + ((size_t)b * a.ny + row) * a.wpr * 2, j, gneed);
    }
    if (!act) return;
    const T tol = T(a.tol_p[b]);
    if constexpr (F::TG <= 32 && F::SM >= F::L && F::R >= 8) {
        // warp-synchronous rows: the epilogue (u*, the fp64 phase) rolled over
        // the row through the group's exchange buffer, four elements in flight
        // per thread. One copy of its code instead of R: fully unrolled, the
        // fp64 atan2 made the final pass most of the kernel's cold instruction
        // footprint (fetched from HBM after an L2 flush; profiles/r02_startup_times.txt).
        sync();
#pragma unroll
        for (int k = 0; k < F::R; ++k) sm[j + F::TG * k] = v[k];
        sync();
#pragma unroll 1
        for (int k0 = 0; k0 < F::R; k0 += 4) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int k = k0 + q;
                const size_t x = o + F::TG * k;
                const cx<T> vs = sm[j + F::TG * k];
                if (a.v_star) a.v_star[x] = vs;
                const cx<T> us = replace_mod_exact<T>(vs, p[F::TG * k], tol);
                if (a.u_star) a.u_star[x] = us;
                if (a.phases || a.levels) {
                    double th = phase_of((double)us.x, (double)us.y);
                    if (tol > T(0) && np_cabs(us) < tol) th = 0.0;        // np.abs(u*) < zero_tol
                    if (a.phases) a.phases[x] = th;
                    if (a.levels) a.levels[x] = level_of(th);
                }
            }
        }
        return;
    }
#pragma unroll
    for (int k = 0; k < F::R; ++k) {
        const size_t x = o + F::TG * k;
        const cx<T> vs = v[k];
        if (a.v_star) a.v_star[x] = vs;
        const cx<T> us = replace_mod_exact<T>(vs, p[F::TG * k], tol);
        if (a.u_star) a.u_star[x] = us;
        if (a.phases || a.levels) {
            double th = phase_of((double)us.x, (double)us.y);
            if (tol > T(0) && np_cabs(us) < tol) th = 0.0;        // np.abs(u*) < zero_tol
            if (a.phases) a.phases[x] = th;
            if (a.levels) a.levels[x] = level_of(th);
        }
    }
}

// A column task: C interleaved transforms (thread c + C*j) over columns
// col0..col0+C-1 of mask b. NX > 0 fixes n_x at compile time (square
// persistent path) so every column access is base + immediate offset.
// `tw` is the forward column table (a shared copy when TS); `ms`, when PS,
// receives this task's [n_y][C] slice of m through cp.async.
// `tile` / `prefetch()`: cross-task prefetch as in row_task (the tile holds
// this task's [n_y][C] input, written by the previous task's cp.async).
// TM (TMA): the input arrived in shared memory through the tensor
// accelerator: `tma` holds the tiles, their mbarriers and the parity of this
// task; the task issues the next task's copies (next_f / next_m) as soon as
// its own tiles are consumed.
template <typename T>
struct TmaTask {
    const cx<T>* ft;              // [n_y][C] input
    const T* mt;                  // [n_y][MC] m (null: m staged by cp.async, TMA_F)
    unsigned long long* bars;     // [0] input, [1] m
    unsigned parity;
    int MC;
    const CUtensorMap* out;       // the output z' is stored by TMA through the exchange buffer (null: st.global)
    int ox, oz;                   // its box origin (float column 2*col0, mask)
};

template <typename T, int LG_L, int LG_R, int NX, int TS = 0, bool PS = false, int CC = 0,
          class Prefetch = NoPrefetch, bool TM = false, class NextF = NoPrefetch, class NextM = NoPrefetch>
__device__ __forceinline__ void col_task(const ColArgs<T>& a, int b, int col0, int C, cx<T>* smbase,
                                         const twe<T>* tw, T* ms, bool live, double (&acc)[3],
                                         const cx<T>* tile = nullptr, Prefetch prefetch = Prefetch{},
                                         TmaTask<T> tma = TmaTask<T>{}, NextF next_f = NextF{},
                                         NextM next_m = NextM{}, bool stage_m = true) {
    using F = FftShape<LG_L, LG_R>;
    const int c = threadIdx.x % C, j = threadIdx.x / C;
    const size_t nx = NX > 0 ? (size_t)NX : (size_t)a.nx;
    const size_t N = nx * a.ny;
    const size_t rs = nx * F::TG;                    // stride between a thread's elements
    cx<T>* sm = smbase + c * col_stride<T, F::SM>(C);
    cx<T>* f = a.field + b * N + (size_t)j * nx + col0 + c;
    const T* m = a.m + b * a.m_stride + (size_t)j * nx + col0 + c;
    const bool act = live;
    acc[0] = acc[1] = acc[2] = 0.0;
    // per-mask constants, loaded with the field (see row_task)
    const double thr_b = a.mode == 2 ? __ldcg(a.thr_m + b) : 0.0;
    const double esc_b = (a.mode == 2 && !a.raar && a.u_iter >= 1 && a.escale) ? __ldcg(a.escale + b) : 0.0;

    cx<T> v[F::R];
    if (a.mode == 0) {
        // u0 = F^-1(m e^{i0}) (src/solver.py:93-108): m is real, so the stored
        // conj(ColIFFT(m)) is ColFFT(m); the row phase finishes u0
#pragma unroll
        for (int k = 0; k < F::R; ++k) v[k] = mk<T>(m[k * rs] * a.scale, T(0));
    } else if (TM && a.mode == 2) {
        mbar_wait(&tma.bars[0], tma.parity);
#pragma unroll
        for (int k = 0; k < F::R; ++k) v[k] = tma.ft[(j + F::TG * k) * C + c];
        fine_stamp_after(v[F::R - 1], 21);                                     // col: tile landed
        if (tma.out && threadIdx.x == 0) bulk_wait_read();                     // previous task's output read
        __syncthreads();                                                         // tile free, exchange buffer free
        if (threadIdx.x == 0) next_f();
    } else if (tile) {
        cp_async_wait<0>();
        __syncthreads();
#pragma unroll
        for (int k = 0; k < F::R; ++k) v[k] = tile[(j + F::TG * k) * C + c];
        __syncthreads();                                                         // tile free
    } else {
        const cx<T>* src = (a.mode == 2 ? a.in : a.field) + (f - a.field);
#pragma unroll
        for (int k = 0; k < F::R; ++k) v[k] = ld_field(src + k * rs);
        if (a.mode == 2) fine_stamp_after(v[F::R - 1], 21);          // col: loads landed
        if (a.mode == 1) {
#pragma unroll
            for (int k = 0; k < F::R; ++k) v[k] = cscale_conj(v[k], a.scale);   // complex start: conj in, conj(IFFT) out
        }
    }
    if (a.mode < 2) {
        fft1d<T, LG_L, LG_R, -1, TS>(v, sm, tw, j, SyncBlock{});
        if (act) {
#pragma unroll
            for (int k = 0; k < F::R; ++k) f[k * rs] = v[k];
        }
        return;
    }
    if constexpr (PS) {
      if (!TM || !tma.mt) {
        // CC: the persistent kernel's compile-time column count (division-free copy loop)
        static_assert(CC > 0, "staged m needs the compile-time column count");
        if (!stage_m) {
            // resident: loaded by this CTA's first column phase of the launch
        } else if (a.mT)     // transposed m: the task's CC columns are one contiguous run
            stage_tile_s<T, CC, (1 << LG_L), MtStride<T, (1 << LG_L), CC>::V, CC * F::TG>(
                ms, a.mT + b * a.m_stride + (size_t)col0 * (1 << LG_L), (size_t)(1 << LG_L), threadIdx.x);
        else
            stage_tile<T, (1 << LG_L), CC, CC * F::TG>(ms, a.m + b * a.m_stride + col0, nx, threadIdx.x);
        cp_async_commit();
      }
    }
    prefetch();
    cp_async_commit();
    const bool metr = a.u_iter >= 1;
    const bool rec = metr && recorded(a.ctl, a.u_iter);
    const bool gneed = metr && !a.raar && gap_needed(a.ctl, a.u_iter);
#if PM_ROLL
    const int trips = 1 + (a.ny > 0);         // 2, opaque: one rolled copy of the transform
#pragma unroll 1
#else
    constexpr int trips = 2;
#pragma unroll
#endif
    for (int h = 0; h < trips; ++h) {
        if (h) fine_stamp_after(v[F::R - 1], 24);                    // col: after metrics + projection
        fft1d<T, LG_L, LG_R, -1, TS>(v, sm, tw, j, SyncBlock{});   // h = 0: ColFFT(w'); h = 1: conj(z')
        fine_stamp_after(v[F::R - 1], 22 + h);                       // col: after FFT 1 / 2
        if (h) break;
        // u^ = F(u) = ColFFT(w''), w'' = S RowFFT(u): normalised, decided against zero_tol itself
        const ZThr<T> z = zthr<T>(T(thr_b));
        T mm[F::R];
        if (TM && tma.mt) {
            mbar_wait(&tma.bars[1], tma.parity);
#pragma unroll
            for (int k = 0; k < F::R; ++k) mm[k] = tma.mt[(j + F::TG * k) * tma.MC + c];
            __syncthreads();                                                     // m tile free
            if (threadIdx.x == 0) next_m();
        } else {
            if constexpr (PS) {
                if (stage_m) {                       // (resident m: nothing was copied for this task)
                    cp_async_wait<1>();              // m of this task (the prefetch may stay in flight)
                    __syncthreads();
                }
            }
            if constexpr (PS) {
                if (a.mT) {
#pragma unroll
                    for (int k = 0; k < F::R; ++k) mm[k] = ms[c * MtStride<T, (1 << LG_L), CC>::V + j + F::TG * k];
                } else {
#pragma unroll
                    for (int k = 0; k < F::R; ++k) mm[k] = ms[(j + F::TG * k) * C + c];
                }
            } else {
#pragma unroll
                for (int k = 0; k < F::R; ++k) mm[k] = m[k * rs];
            }
        }
        if (rec && act) {
            // reconstructed intensity and physical error (src/metrics.py:74-112);
            // the energy scale is sum m^2 / sum |u|^2 (Parseval: sum |F u|^2 = sum |u|^2).
            // GS: u is on S, so sum |u|^2 = sum p^2 (precomputed). RAAR: sum |x|^2
            // from the row sweep's partials, in a fixed order.
            double sc;
            if (a.raar) {
                __shared__ double s_sc;
                if (threadIdx.x < 32) {
                    const double e = warp_sum_strided(a.xpart + (size_t)b * a.xparts * 2 + 1, a.xparts, 2);
                    if (threadIdx.x == 0) s_sc = a.energy[b] / e;
                }
                __syncthreads();
                sc = s_sc;
                __syncthreads();
            } else {
                sc = esc_b;
            }
#pragma unroll
            for (int k = 0; k < F::R; ++k) {
                const double inten = norm_sq_d(v[k]) * sc;    // fp64 square: no overflow for large fp32 fields
                const double m2 = (double)mm[k] * (double)mm[k];
                if (!(inten <= 1.7976931348623157e308)) {
                    acc[1] = __longlong_as_double(0x7ff8000000000000LL);   // RealGrid's check (src/grid.py:128-129)
                } else if (m2 > 0.0) {
                    const double dev = fabs(m2 - inten);
                    if (dev > a.ctl.t_lit * m2 && dev / m2 > a.ctl.t_lit)
                        acc[1] += a.ctl.t_dark * dev / (a.ctl.t_lit * m2) - a.ctl.t_dark;
                } else if (inten > a.ctl.t_dark) {
                    acc[2] += inten - a.ctl.t_dark;
                }
            }
        }
        double g2 = 0.0;                              // fp64: |u^ - v^|^2 of a large finite field stays finite
        // conj(v^), v^ = replace_m(u^); G(u) = ||P_S u - P_M u|| = ||u^ - v^|| (Parseval; u is on S);
        // the column FFT of S conj(v^) follows
        auto t_of = [&](int k) -> T { return mm[k]; };
        auto epi_gap = [&](int, cx<T> u, cx<T> vh) -> cx<T> {
            g2 += norm_sq_d(csub(u, cconj(vh)));
            return cscale(vh, a.scale);
        };
        auto epi = [&](int, cx<T>, cx<T> vh) -> cx<T> { return cscale(vh, a.scale); };
        // false: u^ = F(u_{u_iter}) was not finite, the reference's Field check of iteration u_iter + 1.
        bool fin;
        // iterations without a gap take a copy of the loop with no fp64 work in it
        // (predicated conversions and squares would still take issue slots)
        if (gneed) fin = project_regs<true>(v, z, t_of, epi_gap);
        else fin = project_regs<true>(v, z, t_of, epi);
        if (act && !fin) first_bad(&a.st[b].bad, a.u_iter + 1);
        acc[0] = act ? g2 : 0.0;
    }
    if constexpr (TM) {
        if (tma.out) {
            // stage [n_y][C] in the exchange buffer; the tensor accelerator
            // writes it out while the next task computes
            if (act) {
                constexpr int NY = 1 << LG_L;                      // TMA builds: NY >= 256 (blocked maps)
                __syncthreads();                                   // FFT 2's last exchange reads are done
#pragma unroll
                for (int k = 0; k < F::R; ++k) smbase[(j + F::TG * k) * C + c] = v[k];
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncthreads();
                if (threadIdx.x == 0) {
                    tma_store_3d(tma.out, smbase, tma.ox, 0, tma.oz * (NY / 256));
                    bulk_commit();
                }
            }
            fine_stamp(25);
            return;
        }
    }
    if (act) {
#pragma unroll
        for (int k = 0; k < F::R; ++k) f[k * rs] = v[k];
    }
    fine_stamp(25);                                                     // col: stores issued
}

// Fixed-order CTA sum of NV accumulators; thread 0 gets the totals.
template <int NV>
__device__ __forceinline__ void block_reduce(double (&acc)[NV], double (&tot)[NV]) {
    __shared__ double wsum[32][NV];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nw = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        const double x = warp_sum(acc[v]);
        if (lane == 0) wsum[warp][v] = x;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            double s = 0.0;
            for (int w = 0; w < nw; ++w) s += wsum[w][v];
            tot[v] = s;
        }
    }
    __syncthreads();
}

// ------------------------------------------------------------ sweep kernels
// One launch per sweep (general path: any power-of-two n_x x n_y).
// Arrival ticket over the nblk CTAs of one mask: true in the last CTA to
// arrive (after a fence, so every other CTA's global writes are visible),
// which also re-arms the counter.
__device__ __forceinline__ bool cta_ticket(unsigned* ctr, int nblk) {
    __shared__ int s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned t = atomicAdd(ctr, 1u);
        s_last = (t == (unsigned)(nblk - 1));
        if (s_last) *ctr = 0u;
    }
    __syncthreads();
    if (s_last) __threadfence();
    return s_last;
}

template <typename T, int LG_L, int LG_R>
__global__ void __launch_bounds__(256) row_iter_kernel(RowArgs<T> a) {
    using F = FftShape<LG_L, LG_R>;
    extern __shared__ __align__(16) unsigned char smraw[];
    const int b = blockIdx.y;
    MaskState* st = a.st + b;
    if (st->stop | st->done) return;
    // RAAR: this sweep measures the gap of x_{it-1}; the last CTA decides it
    const int gi = a.it - 1;
    const bool dec = a.mode >= kRowRaar && gi >= 1 && st->decided < gi &&
                     (a.mode == kRowProbe || decision_needed(a.ctl, gi));
    const int G = blockDim.x / F::TG;
    const int g = threadIdx.x / F::TG, j = threadIdx.x % F::TG;
    row_task<T, LG_L, LG_R>(a, b, blockIdx.x * G + g, j, reinterpret_cast<cx<T>*>(smraw) + g * F::SM, a.twf,
                            nullptr, true, true, group_sync<F::TG>(g));
    if (dec && cta_ticket(a.ctr + b, a.nblk) && threadIdx.x < 32)
        decide_raar_warp(st, a.hist, a.hist_stride, a.ctl, b, gi, a.rpart + (size_t)b * a.ny * a.wpr * 2,
                         a.ny * a.wpr, nullptr, 0);
}

template <typename T, int LG_L, int LG_R>
__global__ void __launch_bounds__(256) row_final_kernel(FinalArgs<T> a, double* hist, int hist_stride,
                                                        unsigned* ctr, int nblk) {
    using F = FftShape<LG_L, LG_R>;
    extern __shared__ __align__(16) unsigned char smraw[];
    const int b = blockIdx.y;
    MaskState* st = a.st + b;
    if (st->done) return;
    const int K = a.ctl.max_iters;
    const bool dec = a.x && !st->stop && st->decided < K;
    const int G = blockDim.x / F::TG;
    const int g = threadIdx.x / F::TG, j = threadIdx.x % F::TG;
    final_task<T, LG_L, LG_R>(a, b, blockIdx.x * G + g, j, reinterpret_cast<cx<T>*>(smraw) + g * F::SM, a.tw,
                              true, group_sync<F::TG>(g));
    if (dec && cta_ticket(ctr + b, nblk) && threadIdx.x < 32)
        decide_raar_warp(st, hist, hist_stride, a.ctl, b, K, a.rpart + (size_t)b * a.ny * a.wpr * 2,
                         a.ny * a.wpr, nullptr, 0);
}

// Largest CTA a column kernel is launched with (see col_config in pm_capi.cu):
// 256 threads while a transform needs <= 64 threads or holds >= 32 points per
// thread (register budget), else 512.
__host__ __device__ constexpr int col_max_threads_for(int lgR, int TG) { return (TG <= 64 || lgR >= 5) ? 256 : 512; }
template <int LG_L, int LG_R>
constexpr int col_max_threads() { return col_max_threads_for(FftShape<LG_L, LG_R>::lgR, FftShape<LG_L, LG_R>::TG); }

template <typename T, int LG_L, int LG_R>
__global__ void __launch_bounds__(col_max_threads<LG_L, LG_R>()) col_iter_kernel(ColArgs<T> a) {
    using F = FftShape<LG_L, LG_R>;
    extern __shared__ __align__(16) unsigned char smraw[];
    const int b = blockIdx.y;
    MaskState* st = a.st + b;
    if (st->stop | st->done) return;
    const int C = blockDim.x / F::TG;
    double acc[3];
    col_task<T, LG_L, LG_R, 0>(a, b, blockIdx.x * C, C, reinterpret_cast<cx<T>*>(smraw), a.twf, nullptr, true,
                               acc);
    if (a.mode < 2 || a.u_iter < 1) return;
    if (!a.raar && !decision_needed(a.ctl, a.u_iter)) return;   // no metrics, no ticket
    double tot[3];
    if (a.raar) {
        // lit/dark of x_{u_iter}, kept for the decision the next row sweep takes
        if (recorded(a.ctl, a.u_iter) &&
            reduce_ticket<3>(acc, a.part + (size_t)b * a.nblk * 3, a.ctr + b, a.nblk, blockIdx.x, tot) &&
            threadIdx.x == 0) {
            st->pend_lit = tot[1];
            st->pend_dark = tot[2];
        }
        return;
    }
    if (reduce_ticket<3>(acc, a.part + (size_t)b * a.nblk * 3, a.ctr + b, a.nblk, blockIdx.x, tot)) {
        if (threadIdx.x == 0) {
            const int i = a.u_iter;
            decide(st, a.hist + ((size_t)b * a.hist_stride + (i - 1)) * 4, a.ctl, i,
                   (i - 1) % a.ctl.record_every == 0, tot);
        }
    }
}

// -------------------------------------------------------- persistent solve
// The whole solve in one cooperative launch: one CTA per SM, phases
// separated by a grid barrier instead of kernel boundaries (a kernel
// boundary costs several microseconds on B200, a barrier about one).
struct GridBar {
    unsigned count;   // arrivals, monotonic within a launch (zeroed before it)
    unsigned gen;     // released epoch
};

__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Grid barrier: every CTA releases one arrival (no returned atomic) and
// polls the monotonic arrival count until the whole grid has arrived at this
// epoch; `epoch` counts this launch's barriers (identical in all CTAs).
#ifndef PM_BAR_NS
#define PM_BAR_NS 32         // poll back-off (ns) of the grid barrier
#endif
__device__ __forceinline__ void grid_sync(GridBar* bar, unsigned& epoch) {
    __syncthreads();
    ++epoch;
    if (threadIdx.x == 0) {
        red_release_add(&bar->count, 1u);
        const unsigned target = epoch * gridDim.x;
        while (ld_acquire(&bar->count) < target) {
            if constexpr (PM_BAR_NS > 0) __nanosleep(PM_BAR_NS);
        }
    }
    __syncthreads();
}

template <typename T>
struct SolveArgs {
    RowArgs<T> row;
    ColArgs<T> col;
    FinalArgs<T> fin;
    GridBar* bar;
    int batch;
    int it_begin, it_end;      // iterations it_begin..it_end-1 (row it, col it)
    int do_init;               // run the initial-iterate phases first
    int do_final;              // finish with the best-approximation pair
    int init_mode;             // column init from real m (0) or complex field (1)
    int do_probe;              // RAAR: end with the gap / decision of the last iterate
    unsigned long long* stamps; // optional: globaltimer at every phase boundary (CTA 0)
    int res;                   // p and m may stay resident (one row and one column task per CTA)
    int tma;                   // the column phase's TMA maps below are valid
    CUtensorMap tm_in;         // column input w' ([batch][n_y][2 n_x] floats or doubles)
    CUtensorMap tm_m;          // m ([batch][n_y][n_x])
    int tma_out;               // the column phase stores z' by TMA (tm_out valid)
    CUtensorMap tm_out;        // z' ([batch][n_y][2 n_x])
};

// stamps[cta * kStampsPerCta + i] = %globaltimer at the i-th stamp point
// (PM_FINE builds: a longer row, slots 128.. hold the fine stamps).
constexpr int kStampsPerCta = PM_FINE ? 1024 : 256;
__device__ __forceinline__ void stamp(unsigned long long* s, int& i) {
    if (s && threadIdx.x == 0 && i < kStampsPerCta) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        s[blockIdx.x * kStampsPerCta + i] = t;
    }
    ++i;
}

__device__ __forceinline__ bool mask_live(const MaskState* st) {
    return !(__ldcg(&st->stop) | __ldcg(&st->done));
}

#ifndef PM_SOLVE_NT
#define PM_SOLVE_NT 512
#endif
constexpr int kSolveThreads = PM_SOLVE_NT;

// Shared-memory layout of solve_kernel: the FFT exchange buffers (the larger
// of the row phase's G transforms and the column phase's C interleaved ones),
// then, while they fit, the staged real grid of a task (p rows / m columns,
// PS) and copies of the twiddle tables (TS; L1 does not survive the grid
// barrier's acquire, so tables read through L1 would miss once per pass).
template <typename T, int LG, int LGR_R, int LGR_C, bool TV = false>
struct SolveSmem {
    using FR = FftShape<LG, LGR_R>;
    using FC = FftShape<LG, LGR_C>;
    static constexpr int G = kSolveThreads / FR::TG > 0 ? kSolveThreads / FR::TG : 1;
    static constexpr int C = kSolveThreads / FC::TG > 0 ? kSolveThreads / FC::TG : 1;
    static constexpr int rows = G * FR::SM;
    static constexpr int pad = 128 / (int)(sizeof(cx<T>) * C) > 0 ? 128 / (int)(sizeof(cx<T>) * C) : 1;
    static constexpr int cols = FC::SM ? C * (FC::SM + pad) : 0;
    static constexpr int up16(int x) { return (x + 15) / 16 * 16; }
    static constexpr int EX = up16((int)sizeof(cx<T>) * (rows > cols ? rows : cols));
    static constexpr int ST = up16((int)sizeof(T) * ((G > C ? G : C) << LG) +
                                   (int)sizeof(T) * C * MtStride<T, (1 << LG), C>::PAD);   // + transposed-m pad
    static constexpr bool F32 = sizeof(T) == 4;
    static constexpr bool SAME = LGR_R == LGR_C;
    static constexpr int NTAB = 1;                                // forward transforms only (conjugate storage)
    static constexpr int TWR = FR::TW * NTAB;                     // entries
    static constexpr int TWC = SAME ? 0 : FC::TW * NTAB;
    // compact (c, s) shared twiddles (fp32, 4096 points with TMA tiles: the
    // 65 KB table would not leave room for the column tile)
    static constexpr bool TW2 = F32 && TV && LG >= 12;
    static constexpr int TWB = up16((TWR + TWC) * (TW2 ? 8 : (int)sizeof(twe<T>)));
    static constexpr int TILE = up16((int)sizeof(cx<T>) * ((G > C ? G : C) << LG));   // one task's input
    static constexpr int LIMIT = 225 * 1024;
    // Cross-task prefetch (PM_PF=1) needs the staging, a tile and (measured:
    // without them the twiddle loads are hoisted into spills) the shared
    // twiddles. It is off by default: on B200 the sweeps are issue-bound, not
    // load-latency-bound, once p/m and twiddles are in shared memory (batch-32
    // 1024^2 +2%, 2048^2 -9%; scripts/sweep_perf.py). Without it: twiddles
    // first (they are on every pass), then staging.
#ifndef PM_PF
#define PM_PF 0
#endif
#ifndef PM_TMA
#define PM_TMA 1
#endif
    // TMA column tiles (column phase): the task's input [n_y][C] and its m
    // [n_y][MC] (a TMA box row is >= 16 bytes), plus two mbarriers. Placed
    // after every other region when they fit (A); else the shared twiddles
    // give way (B); else the tiles overlay the row phase's staging, which is
    // idle during the column phase (C).
    static constexpr int MC = C * (int)sizeof(T) >= 16 ? C : 16 / (int)sizeof(T);
    static constexpr int FTB = up16((int)sizeof(cx<T>) * (C << LG));
    static constexpr int MTB = up16((int)sizeof(T) * (MC << LG));
    static constexpr int TMAB = FTB + MTB + 16;
    static constexpr int XSB = up16((int)sizeof(cx<T>) * (G << LG));   // RAAR: the row's x staged with p
    static constexpr bool PF = PM_PF && EX + ST + TILE + TWB <= LIMIT;
    static constexpr bool TS0 = PF ? (EX + ST + TILE + TWB <= LIMIT) : (EX + TWB <= LIMIT);
    static constexpr bool PS0 = PF || (EX + (TS0 ? TWB : 0) + ST <= LIMIT);
    static constexpr int BASE0 = EX + (PS0 ? ST : 0) + (PF ? TILE : 0) + (TS0 ? TWB : 0);
    static constexpr bool WANT = TV && PM_TMA && LG >= 8 && !PF;
    static constexpr bool TMA_A = WANT && BASE0 + TMAB <= LIMIT;
    // (B / C drop the shared twiddles; measured: the hoisted global twiddle
    // loads then spill at 2048^2 / 4096^2, so only A is enabled)
    static constexpr bool TMA_B = false && WANT && !TMA_A && EX + ST + TMAB <= LIMIT;
    static constexpr bool TMA_C = false && WANT && !TMA_A && !TMA_B && EX + TMAB <= LIMIT;
    // F: the column tile only, when the m tile does not fit as well (2048^2,
    // 4096^2); m is then staged by cp.async from its transposed copy
#ifndef PM_TMA_F
#define PM_TMA_F 1
#endif
    static constexpr bool TMA_F = PM_TMA_F && WANT && !TMA_A && BASE0 + FTB + 16 + 128 <= LIMIT;
    static constexpr bool TMA = TMA_A || TMA_B || TMA_C || TMA_F;
    static constexpr bool TMA_M = TMA && !TMA_F;                 // m streamed by TMA too
    static constexpr int TS = ((TMA_B || TMA_C) ? false : TS0) ? (TW2 ? 2 : 1) : 0;
    static constexpr bool PS = (TMA_B || TMA_C) ? true : PS0;
    static constexpr int OFF_ST = EX;
    static constexpr int OFF_TILE = EX + (PS ? ST : 0);
    static constexpr int OFF_TW = OFF_TILE + (PF ? TILE : 0);
    static constexpr int BYTES = OFF_TW + (TS ? TWB : 0);
    static constexpr int up128(int x) { return (x + 127) / 128 * 128; }
    static constexpr int OFF_FT = TMA_C ? EX : up128(BYTES);
    static constexpr int OFF_MT = OFF_FT + FTB;
    static constexpr int OFF_BAR = OFF_MT + (TMA_M ? MTB : 0);
    // TMA builds also stream the row phase's rows through the column tile
    // (idle then), one bulk copy and one mbarrier per row group
#ifndef PM_ROW_TMA
#define PM_ROW_TMA 1
#endif
    static constexpr bool ROW_TMA = PM_ROW_TMA && TMA && FTB >= (int)sizeof(cx<T>) * (G << LG);
    static constexpr int NBAR = 2 + (ROW_TMA ? G : 0);
    static_assert(!ROW_TMA || G <= 16, "row_loads() holds 16 groups");
    static constexpr int TMA_END = TMA ? OFF_BAR + up16(8 * NBAR) : 0;
    static constexpr int BYTES_T = TMA_END > BYTES ? TMA_END : BYTES;
    static constexpr bool XS = PS && BYTES_T + XSB <= LIMIT;
    static constexpr int OFF_XS = BYTES_T;
    // Resident p and m (plain build, one row task and one column task per
    // CTA: a single mask): the CTA's p rows and m columns stay in shared
    // memory for the whole launch instead of being staged every phase.
#ifndef PM_RES
#define PM_RES 1
#endif
    static constexpr int XSE = XS ? XSB : 0;
    static constexpr bool RES_GS = PM_RES && PS && !TV && BYTES_T + 2 * ST <= LIMIT;
    static constexpr bool RES_RAAR = PM_RES && PS && !TV && BYTES_T + XSE + 2 * ST <= LIMIT;
    static constexpr int BYTES_ALL = BYTES_T + (RES_GS ? 2 * ST : 0);
    static constexpr int BYTES_ALL_RAAR = BYTES_T + XSE + (RES_RAAR ? 2 * ST : 0);
    static constexpr int CB = C * (int)sizeof(T);                 // bytes per m run of a column task
    static constexpr int CH = CB >= 16 ? 16 : CB;                 // cp.async size for it
};

template <typename T>
struct Tables {
    const twe<T>* rf;   // forward row / column tables
    const twe<T>* cf;
};

// The solve's twiddle tables: shared copies (made once per launch) or global.
template <typename T, int LG, int LGR_R, int LGR_C, bool TV = false>
__device__ __forceinline__ Tables<T> load_tables(const RowArgs<T>& r, const ColArgs<T>& c, unsigned char* smraw) {
    using L = SolveSmem<T, LG, LGR_R, LGR_C, TV>;
    if constexpr (!L::TS) {
        return Tables<T>{r.twf, c.twf};
    } else if constexpr (L::TS == 2) {
        float2* t = reinterpret_cast<float2*>(smraw + L::OFF_TW);
        constexpr int nr = L::FR::TW, nc = L::FC::TW;
        float2* rf = t;
        float2* cf = L::SAME ? rf : t + L::TWR;
        for (int i = threadIdx.x; i < nr; i += blockDim.x) rf[i] = make_float2(r.twf[i].x, r.twf[i].y);
        if constexpr (!L::SAME) {
            for (int i = threadIdx.x; i < nc; i += blockDim.x) cf[i] = make_float2(c.twf[i].x, c.twf[i].y);
        }
        __syncthreads();
        return Tables<T>{reinterpret_cast<const twe<T>*>(rf), reinterpret_cast<const twe<T>*>(cf)};
    } else {
        twe<T>* t = reinterpret_cast<twe<T>*>(smraw + L::OFF_TW);
        constexpr int nr = L::FR::TW, nc = L::FC::TW;
        twe<T>* rf = t;
        twe<T>* cf = L::SAME ? rf : t + L::TWR;
        for (int i = threadIdx.x; i < nr; i += blockDim.x) rf[i] = r.twf[i];
        if constexpr (!L::SAME) {
            for (int i = threadIdx.x; i < nc; i += blockDim.x) cf[i] = c.twf[i];
        }
        __syncthreads();
        return Tables<T>{rf, cf};
    }
}

// Contiguous share of `total` rows for this CTA: the first total % grid CTAs
// take one row more, so no CTA does more than ceil(total / grid).
__device__ __forceinline__ void row_share(int total, int& start, int& count) {
    const int q = total / (int)gridDim.x, rem = total % (int)gridDim.x;
    count = q + ((int)blockIdx.x < rem ? 1 : 0);
    start = (int)blockIdx.x * q + min((int)blockIdx.x, rem);
}

// Row phase: each CTA runs its contiguous share of the batch's rows, G at a
// time. The field loads of a task are issued before its mask state is known,
// so the state's L2 round trip overlaps them. Groups of whole warps with no
// row left skip the round (their barriers are their own).
// Launch-long residency of p and m (SolveSmem::RES_*): region offsets and
// whether this CTA has loaded them yet.
struct Resident {
    bool on;
    bool p_ok, m_ok;
    int off_p, off_m;
};

template <typename T, int LG, int LGR_R, int LGR_C, int ALG, bool TV = false>
__device__ __forceinline__ void row_phase(const RowArgs<T>& a, int batch, unsigned char* smraw,
                                          const Tables<T>& tw, Resident* rs = nullptr, bool tma = false) {
    using L = SolveSmem<T, LG, LGR_R, LGR_C, TV>;
    using F = FftShape<LG, LGR_R>;
    cx<T>* smem = reinterpret_cast<cx<T>*>(smraw);
    const int G = blockDim.x / F::TG;
    const int g = threadIdx.x / F::TG, j = threadIdx.x % F::TG;
    const bool res = rs && rs->on;
    T* ps = reinterpret_cast<T*>(smraw + (res ? rs->off_p : L::OFF_ST)) + ((size_t)g << LG);
    const bool stage_p = !(res && rs->p_ok);
    cx<T>* tile = reinterpret_cast<cx<T>*>(smraw + L::OFF_TILE) + ((size_t)g << LG);
    constexpr int NX = 1 << LG;
    int start, count;
    row_share(batch << LG, start, count);
    // prefetch the next round's row while this one computes (whole-warp
    // groups, more than one round in this CTA's share)
    const bool pf = L::PF && F::TG >= 32 && count > G;
    // row TMA (ROW_TMA builds with TMA active): every row of a group arrives in
    // its slice of the column tile by one bulk copy, issued a round ahead by
    // the group's first thread; the group's mbarrier completes it
    const bool rt = L::ROW_TMA && tma && F::TG >= 32;
    cx<T>* rtile = reinterpret_cast<cx<T>*>(smraw + L::OFF_FT) + ((size_t)g << LG);
    unsigned long long* rbar = reinterpret_cast<unsigned long long*>(smraw + L::OFF_BAR) + 2 + g;
    unsigned* s_rloads = row_loads();
    auto rissue = [&](int rr) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");     // earlier reads of the slice
        mbar_expect_tx(rbar, (unsigned)(sizeof(cx<T>) * NX));
        bulk_load(rtile, a.field + (size_t)(start + rr) * NX, (unsigned)(sizeof(cx<T>) * NX), rbar);
    };
    if (rt && j == 0 && g < count) rissue(g);
    for (int r0 = 0; r0 < count; r0 += G) {
        const bool inb = r0 + g < count;
        if (F::TG >= 32 && !inb) break;
        const int r = start + (inb ? r0 + g : 0);
        const int b = r >> LG;
        const bool live = inb && mask_live(a.st + b);
        const int rn = r0 + G + g;                 // this group's next row in the share
        const unsigned rpar = rt ? (s_rloads[g] & 1u) : 0u;
        auto prefetch = [&]() {
            if (rt) {
                if (j == 0) {
                    s_rloads[g] += 1;
                    if (rn < count) rissue(rn);
                }
            } else if (pf && rn < count) {
                stage_tile<cx<T>, 1, NX, F::TG>(tile, a.field + (size_t)(start + rn) * NX, 0, j);
            }
        };
        constexpr bool XS = ALG == 1 && L::XS;
        row_task<T, LG, LGR_R, decltype(group_sync<F::TG>(g)), ALG, L::TS, L::PS, decltype(prefetch), XS>(
            a, b, r & (NX - 1), j, smem + g * F::SM, tw.rf, ps, inb, live, group_sync<F::TG>(g),
            rt ? rtile : ((pf && r0 > 0) ? tile : nullptr), prefetch,
            XS ? reinterpret_cast<cx<T>*>(smraw + L::OFF_XS) + ((size_t)g << LG) : nullptr, stage_p,
            rt ? rbar : nullptr, rpar);
    }
    if (res && a.mode != kRowInit) rs->p_ok = true;
}

template <typename T, int LG, int LGR_R, int LGR_C, bool TV = false>
__device__ __forceinline__ void final_phase(const FinalArgs<T>& a, int batch, unsigned char* smraw,
                                            const Tables<T>& tw) {
    using L = SolveSmem<T, LG, LGR_R, LGR_C, TV>;
    using F = FftShape<LG, LGR_R>;
    cx<T>* smem = reinterpret_cast<cx<T>*>(smraw);
    const int G = blockDim.x / F::TG;
    const int g = threadIdx.x / F::TG, j = threadIdx.x % F::TG;
    int start, count;
    row_share(batch << LG, start, count);
    for (int r0 = 0; r0 < count; r0 += G) {
        const bool inb = r0 + g < count;
        if (F::TG >= 32 && !inb) break;
        const int r = start + (inb ? r0 + g : 0);
        const int b = r >> LG;
        const bool act = inb && !__ldcg(&a.st[b].done);
        final_task<T, LG, LGR_R, L::TS>(a, b, r & ((1 << LG) - 1), j, smem + g * F::SM, tw.rf, act,
                                        group_sync<F::TG>(g));
    }
}

// Column phase; with metrics, task t of mask b leaves its block sum in
// part[b][t] so the per-mask total is combined in task order (independent of
// which CTA ran which task, hence of batch size and grid size).
// TMA maps of the column phase: its input (w') and m, as [batch][n_y][2 n_x]
// / [batch][n_y][n_x] tensors in 256-row blocks, one box per task tile (null: no TMA).
struct ColTma {
    const CUtensorMap* in;
    const CUtensorMap* m;
    unsigned* count;              // tile loads completed by this CTA (mbarrier parity)
    const CUtensorMap* out;       // z' ([batch][n_y][2 n_x]) written by TMA stores (null: st.global)
};

template <typename T, int LG, int LGR_R, int LGR_C, bool TV = false>
__device__ __forceinline__ void col_phase(const ColArgs<T>& a, int batch, unsigned char* smraw,
                                          const Tables<T>& tw, ColTma ct = ColTma{nullptr, nullptr, nullptr},
                                          Resident* rs = nullptr) {
    using L = SolveSmem<T, LG, LGR_R, LGR_C, TV>;
    using F = FftShape<LG, LGR_C>;
    cx<T>* smem = reinterpret_cast<cx<T>*>(smraw);
    const bool res = rs && rs->on && a.mode == 2;
    T* ms = reinterpret_cast<T*>(smraw + (res ? rs->off_m : L::OFF_ST));
    const bool stage_m = !(res && rs->m_ok);
    cx<T>* tile = reinterpret_cast<cx<T>*>(smraw + L::OFF_TILE);
    constexpr int NX = 1 << LG;
    const int C = blockDim.x / F::TG;
    const int tpm = NX / C;                 // tasks per mask
    const int total = batch * tpm;
    // RAAR keeps only lit/dark (the gap comes from the row sweep), in a
    // parity-selected buffer: the decision on x_{it-1} reads it while this
    // phase of iteration it may already run
    const bool metr = a.mode == 2 && a.u_iter >= 1 &&
                      (a.raar ? recorded(a.ctl, a.u_iter) : gap_needed(a.ctl, a.u_iter));
    double* const part = a.part + ((a.raar && (a.u_iter & 1)) ? a.part_alt : 0);
    // prefetch the next task's columns while this one computes (iterate mode,
    // more than one task for this CTA)
    const bool pf = L::PF && a.mode == 2 && (int)blockIdx.x + (int)gridDim.x < total;
    if constexpr (L::TMA) {
        // CTAs with several tasks in this phase (batches, large grids); a
        // single task is faster with direct loads (measured: 1024^2, 1 mask)
        if (ct.in && a.mode == 2 && 2 * (int)gridDim.x <= total) {
            // TMA: tiles for task t are in flight before t starts; each task
            // issues its successor's copies once its own tiles are consumed
            static_assert(NX >= 256, "blocked TMA maps: whole 256-row blocks");
            cx<T>* ft = reinterpret_cast<cx<T>*>(smraw + L::OFF_FT);
            T* mt = reinterpret_cast<T*>(smraw + L::OFF_MT);
            unsigned long long* bars = reinterpret_cast<unsigned long long*>(smraw + L::OFF_BAR);
            auto issue_f = [&](int t) {
                const int bt = t / tpm, c0 = (t - bt * tpm) * C;
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // prior reads of the tile
                mbar_expect_tx(&bars[0], (unsigned)(sizeof(cx<T>) * C * NX));
                tma_load_3d(ft, ct.in, 2 * c0, 0, bt * (NX / 256), &bars[0]);
            };
            // a box must start on a 16-byte boundary: when a task is narrower
            // than 16 bytes of m, the box starts at the aligned column below
            // and the task reads from its offset inside the tile
            constexpr int MA = 16 / (int)sizeof(T);
            auto issue_m = [&](int t) {
                const int bt = t / tpm, c0 = (t - bt * tpm) * C;
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_expect_tx(&bars[1], (unsigned)(sizeof(T) * L::MC * NX));
                tma_load_3d(mt, ct.m, c0 & ~(MA - 1), 0, bt * (NX / 256), &bars[1]);
            };
            // (measured: claiming tasks from a global counter instead of this
            // static order was slower, 4096^2 275 -> 283 us per iteration:
            // concurrently running neighbours share sectors of the field)
            if (threadIdx.x == 0 && (int)blockIdx.x < total) {
                issue_f(blockIdx.x);
                if constexpr (L::TMA_M) issue_m(blockIdx.x);
            }
            for (int t = blockIdx.x; t < total; t += gridDim.x) {
                const int b = t / tpm, tt = t - b * tpm;
                const bool act = mask_live(a.st + b);
                const int tn = t + gridDim.x;
                auto next_f = [&]() { if (tn < total) issue_f(tn); };
                auto next_m = [&]() { if (L::TMA_M && tn < total) issue_m(tn); };
                TmaTask<T> tk{ft, L::TMA_M ? mt + ((tt * C) & (MA - 1)) : nullptr, bars, *ct.count & 1u, L::MC,
                              ct.out, 2 * tt * C, b};
                double acc[3];
                col_task<T, LG, LGR_C, NX, L::TS, L::PS, L::C, NoPrefetch, true, decltype(next_f), decltype(next_m)>(
                    a, b, tt * C, C, smem, tw.cf, ms, act, acc, nullptr, NoPrefetch{}, tk, next_f, next_m);
                *ct.count += 1;
                if (metr && act) {
                    double tot[3];
                    block_reduce<3>(acc, tot);
                    if (threadIdx.x == 0) {
                        double* q = part + ((size_t)b * tpm + tt) * 3;
                        q[0] = tot[0]; q[1] = tot[1]; q[2] = tot[2];
                    }
                }
            }
            if (ct.out && threadIdx.x == 0) bulk_wait_all();     // z' complete before the grid barrier
            return;
        }
    }
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
        const int b = t / tpm, tt = t - b * tpm;
        const bool act = mask_live(a.st + b);
        const int tn = t + gridDim.x;
        auto prefetch = [&]() {
            if (pf && tn < total) {
                const int bn = tn / tpm, cn = (tn - bn * tpm) * C;
                stage_tile<cx<T>, NX, L::C, kSolveThreads>(tile, a.in + (size_t)bn * NX * NX + cn, NX, threadIdx.x);
            }
        };
        double acc[3];
        col_task<T, LG, LGR_C, NX, L::TS, L::PS, L::C>(a, b, tt * C, C, smem, tw.cf, ms, act, acc,
                                                        (pf && t != (int)blockIdx.x) ? tile : nullptr, prefetch,
                                                        TmaTask<T>{}, NoPrefetch{}, NoPrefetch{}, stage_m);
        if (metr && act) {
            double tot[3];
            block_reduce<3>(acc, tot);
            if (threadIdx.x == 0) {
                double* q = part + ((size_t)b * tpm + tt) * 3;
                q[0] = tot[0]; q[1] = tot[1]; q[2] = tot[2];
            }
        }
    }
    if (res) rs->m_ok = true;
}

// Per-mask reduction of the column phase's task partials and the stop
// decision, by CTA (b mod grid).
template <typename T, int LG, int LGR_C>
__device__ __forceinline__ void decide_phase(const ColArgs<T>& a, int batch) {
    using F = FftShape<LG, LGR_C>;
    const int C = blockDim.x / F::TG;
    const int tpm = (1 << LG) / C;
    const int lane = threadIdx.x & 31;
    if (threadIdx.x >= 32) return;
    const bool metr = gap_needed(a.ctl, a.u_iter);
    // the last CTAs decide: the row share puts the fewest rows on them
    for (int b = gridDim.x - 1 - blockIdx.x; b < batch; b += gridDim.x) {
        MaskState* st = a.st + b;
        if (!mask_live(st)) continue;
        double tot[3] = {0.0, 0.0, 0.0};
        if (metr) {
#pragma unroll
            for (int v = 0; v < 3; ++v) {
                double x = 0.0;
                for (int i = lane; i < tpm; i += 32) x += __ldcg(&a.part[((size_t)b * tpm + i) * 3 + v]);
#pragma unroll
                for (int o = 16; o >= 1; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
                tot[v] = x;
            }
        }
        if (lane == 0) {
            const int i = a.u_iter;
            decide(st, a.hist + ((size_t)b * a.hist_stride + (i - 1)) * 4, a.ctl, i,
                   (i - 1) % a.ctl.record_every == 0, tot);
        }
    }
}

// RAAR decision on iterate i of every live mask, by CTA (b mod grid): gap
// from the row partials, lit/dark from the column partials of iteration i.
template <typename T>
__device__ __forceinline__ void decide_phase_raar(const RowArgs<T>& r, int batch, int i) {
    if (threadIdx.x >= 32 || i < 1) return;
    for (int b = gridDim.x - 1 - blockIdx.x; b < batch; b += gridDim.x) {
        MaskState* st = r.st + b;
        if (!mask_live(st)) continue;
        decide_raar_warp(st, r.hist, r.hist_stride, r.ctl, b, i, r.rpart + (size_t)b * r.ny * r.wpr * 2,
                         r.ny * r.wpr, r.cpart + ((i & 1) ? r.cpart_alt : 0) + (size_t)b * r.tpm * 3, r.tpm);
    }
}

template <typename T, int LG, int LGR_R, int LGR_C, int ALG, bool TV = false>
__global__ void __launch_bounds__(kSolveThreads, 1) solve_kernel(const __grid_constant__ SolveArgs<T> a) {
    // dynamic shared memory follows the static variables: realign it to 128
    // bytes (TMA destinations), for which the launch reserves 128 more bytes
    extern __shared__ __align__(128) unsigned char smraw_[];
    unsigned char* smraw = smraw_ + ((128u - (smem_u32(smraw_) & 127u)) & 127u);
    using L = SolveSmem<T, LG, LGR_R, LGR_C, TV>;
    const int B = a.batch;
    int si = 0;
    unsigned epoch = 0;
    stamp(a.stamps, si);
    fine_init(a.stamps);
    const Tables<T> tw = load_tables<T, LG, LGR_R, LGR_C, TV>(a.row, a.col, smraw);
    Resident rs{a.res != 0 && (ALG == 1 ? L::RES_RAAR : L::RES_GS), false, false,
                L::BYTES_T + (ALG == 1 ? L::XSE : 0), L::BYTES_T + (ALG == 1 ? L::XSE : 0) + L::ST};
    unsigned tma_count = 0;
    ColTma ct{nullptr, nullptr, &tma_count, nullptr};
    if constexpr (L::TMA) {
        if (a.tma) {
            ct.in = &a.tm_in;
            ct.m = &a.tm_m;
            if (a.tma_out) ct.out = &a.tm_out;
            if (threadIdx.x == 0) {
                unsigned long long* bars = reinterpret_cast<unsigned long long*>(smraw + L::OFF_BAR);
                for (int i = 0; i < L::NBAR; ++i) mbar_init(&bars[i], 1);
                for (int i = 0; i < 16; ++i) row_loads()[i] = 0;
                asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            }
            __syncthreads();
        }
    }
    if (a.do_init) {
        ColArgs<T> c = a.col;
        c.mode = a.init_mode;
        c.u_iter = 0;
        col_phase<T, LG, LGR_R, LGR_C, TV>(c, B, smraw, tw);          // u0 column half
        grid_sync(a.bar, epoch);
        RowArgs<T> r = a.row;
        r.mode = kRowInit;
        row_phase<T, LG, LGR_R, LGR_C, ALG, TV>(r, B, smraw, tw, &rs, a.tma != 0);     // u0 row half, w0 (RAAR: and x_0)
        grid_sync(a.bar, epoch);
        c.mode = 2;
        col_phase<T, LG, LGR_R, LGR_C, TV>(c, B, smraw, tw, ct, &rs);      // z1
        grid_sync(a.bar, epoch);
    }
    const bool early = a.col.ctl.early_tol >= 0.0;
    const bool lock = a.col.ctl.lockstep != 0;     // host verdicts (should_abort) every iteration
    if constexpr (ALG == 1) {
        // RAAR: the decision on x_{it-1} follows the row phase that measures its gap
        for (int it = a.it_begin; it < a.it_end; ++it) {
            RowArgs<T> r = a.row;
            r.mode = kRowRaar;
            r.it = it;
            row_phase<T, LG, LGR_R, LGR_C, ALG, TV>(r, B, smraw, tw, &rs, a.tma != 0);   // gap of x_{it-1}, x_it, w_it
            grid_sync(a.bar, epoch);
            decide_phase_raar<T>(r, B, it - 1);
            if (early || lock) grid_sync(a.bar, epoch);
            ColArgs<T> c = a.col;
            c.mode = 2;
            c.u_iter = it;
            col_phase<T, LG, LGR_R, LGR_C, TV>(c, B, smraw, tw, ct, &rs);    // lit/dark of x_it, z_{it+1}
            grid_sync(a.bar, epoch);
        }
        if (a.do_probe) {
            RowArgs<T> r = a.row;
            r.mode = kRowProbe;
            r.it = a.it_end;
            row_phase<T, LG, LGR_R, LGR_C, ALG, TV>(r, B, smraw, tw, &rs, a.tma != 0);   // gap of x_{it_end-1}
            grid_sync(a.bar, epoch);
            decide_phase_raar<T>(r, B, a.it_end - 1);
            grid_sync(a.bar, epoch);
        }
        if (a.do_final) {
            final_phase<T, LG, LGR_R, LGR_C, TV>(a.fin, B, smraw, tw);   // pair, mask, gap of x_K
            grid_sync(a.bar, epoch);
            decide_phase_raar<T>(a.row, B, a.fin.ctl.max_iters);
        }
    } else {
        for (int it = a.it_begin; it < a.it_end; ++it) {
            RowArgs<T> r = a.row;
            r.mode = kRowGS;
            r.it = it;
            fine_stamp(1);
            row_phase<T, LG, LGR_R, LGR_C, ALG, TV>(r, B, smraw, tw, &rs, a.tma != 0);   // u_it, w_it
            stamp(a.stamps, si);
            fine_stamp(2);
            grid_sync(a.bar, epoch);
            stamp(a.stamps, si);
            fine_stamp(3);
            ColArgs<T> c = a.col;
            c.mode = 2;
            c.u_iter = it;
            col_phase<T, LG, LGR_R, LGR_C, TV>(c, B, smraw, tw, ct, &rs);    // metrics of u_it, z_{it+1}
            stamp(a.stamps, si);
            fine_stamp(4);
            grid_sync(a.bar, epoch);
            stamp(a.stamps, si);
            fine_stamp(5);
            // decisions: records, early stop, max_iters, and the last iterate
            // of this launch (the stepping API reads state after every launch)
            if (gap_needed(c.ctl, it) || lock || it >= c.ctl.max_iters || it == a.it_end - 1)
                decide_phase<T, LG, LGR_C>(c, B);
            if (early || lock) grid_sync(a.bar, epoch);               // stop flags must be seen by every CTA
        }
        if (a.do_final) final_phase<T, LG, LGR_R, LGR_C, TV>(a.fin, B, smraw, tw);
    }
    stamp(a.stamps, si);
}

// ------------------------------------------------ standalone transform sweeps
// FftProvider.forward / inverse (src/transform.py:47-55): one axis per launch.
// `tw` is the table for `dir` (fp32) or the forward table (fp64).
template <typename T, int LG_L, int LG_R>
__global__ void __launch_bounds__(256) row_fft_kernel(const cx<T>* in, cx<T>* out, const twe<T>* tw,
                                                      int nx, int ny, T scale, int dir) {
    using F = FftShape<LG_L, LG_R>;
    using Sync = typename GroupSync<F::TG>::type;
    extern __shared__ __align__(16) unsigned char smraw[];
    const int G = blockDim.x / F::TG;
    const int g = threadIdx.x / F::TG, j = threadIdx.x % F::TG;
    const size_t o = (size_t)blockIdx.y * nx * ny + (size_t)(blockIdx.x * G + g) * nx + j;
    cx<T>* sm = reinterpret_cast<cx<T>*>(smraw) + g * F::SM;
    cx<T> v[F::R];
#pragma unroll
    for (int k = 0; k < F::R; ++k) v[k] = in[o + F::TG * k];
    if (dir < 0) fft1d<T, LG_L, LG_R, -1>(v, sm, tw, j, Sync{});
    else fft1d<T, LG_L, LG_R, +1>(v, sm, tw, j, Sync{});
#pragma unroll
    for (int k = 0; k < F::R; ++k) out[o + F::TG * k] = cscale(v[k], scale);
}

template <typename T, int LG_L, int LG_R>
__global__ void __launch_bounds__(col_max_threads<LG_L, LG_R>()) col_fft_kernel(const cx<T>* in, cx<T>* out,
                                                                              const twe<T>* tw, int nx, int ny,
                                                                              T scale, int dir) {
    using F = FftShape<LG_L, LG_R>;
    extern __shared__ __align__(16) unsigned char smraw[];
    const int C = blockDim.x / F::TG;
    const int c = threadIdx.x % C, j = threadIdx.x / C;
    const size_t o = (size_t)blockIdx.y * nx * ny + (size_t)j * nx + (size_t)(blockIdx.x * C + c);
    const size_t rs = (size_t)nx * F::TG;
    cx<T>* sm = reinterpret_cast<cx<T>*>(smraw) + c * col_stride<T, F::SM>(C);
    cx<T> v[F::R];
#pragma unroll
    for (int k = 0; k < F::R; ++k) v[k] = in[o + k * rs];
    if (dir < 0) fft1d<T, LG_L, LG_R, -1>(v, sm, tw, j, SyncBlock{});
    else fft1d<T, LG_L, LG_R, +1>(v, sm, tw, j, SyncBlock{});
#pragma unroll
    for (int k = 0; k < F::R; ++k) out[o + k * rs] = cscale(v[k], scale);
}

}  // namespace pm
