// Mixed-radix path for grids whose sides are not powers of two (prime factors
// 2, 3, 5, 7; n <= 4096), e.g. the paper's 800x600 SLM and
// the reference's acceptance grid (tests/test_acceptance.py:118-128,200-205).
//
// The power-of-two path runs a whole solve in one persistent launch; this
// path is two fused sweep kernels per iteration over a work buffer that
// holds RowFFT(u):
//   gen_col_sweep_kernel  a CTA stages TC columns, the twiddle table and its
//                         slice of m in shared memory (cp.async), runs the
//                         Stockham passes, replace_m with the metrics of the
//                         previous iterate (fixed-order fp64 partials; the
//                         last CTA of a mask decides record / early stop /
//                         max_iters / divergence), and the inverse passes;
//   gen_row_sweep_kernel  inverse row passes, P_S into the iterate
//                         (non-finite check), forward row passes;
//   gen_fft_kernel        one axis of a unitary 2-D DFT (start, finish and
//                         the stand-alone transform);
//   gen_final_kernel      u* = P_S v*, the float64 mask and uint8 levels.
// A pass is one radix of the plan: base radices 2, 3, 4, 5, 7, 8 and the
// register composites 9, 10, 12, 16 (internal twiddles as compile-time
// constants), so 800 = 16 x 10 x 5 and 600 = 12 x 10 x 5 take three passes.
// (Composites up to 32 ran slower: one long register DFT per thread leaves
// too few warps per SM, and every extra radix grows the kernels' code.)
// Semantics (threshold decisions, fixed-order fp64 sums, stop logic) are the
// fused path's: see pm_kernels.cuh.
#pragma once
#include <type_traits>

#include "pm_kernels.cuh"

namespace pm {

constexpr int kGenMaxPasses = 16;

struct GenPlan {
    int L;                       // transform length
    int np;                      // passes
    int radix[kGenMaxPasses];    // radix of pass s
    int ns[kGenMaxPasses];       // product of the radices before pass s
    int step[kGenMaxPasses];     // twiddle index step of pass s: L / (ns * radix)
    unsigned mg[kGenMaxPasses];  // multiply-high magic of ns (0 for ns = 1)
};

// cos / sin (2 pi k / r) for the small odd radices, fp64-accurate.
__host__ __device__ constexpr double gen_c(int r, int k) {
    return r == 3 ? (k == 0 ? 1.0 : -0.5)
         : r == 5 ? (k == 0 ? 1.0 : (k == 1 || k == 4) ? 0.30901699437494742410229341718282
                                                        : -0.80901699437494742410229341718282)
         : /* 7 */  (k == 0 ? 1.0 : (k == 1 || k == 6) ? 0.62348980185873353052500488400424
                   : (k == 2 || k == 5) ? -0.22252093395631440428890256449679
                                        : -0.90096886790241912623610231950745);
}
__host__ __device__ constexpr double gen_s(int r, int k) {
    return r == 3 ? (k == 0 ? 0.0 : k == 1 ? 0.86602540378443864676372317075294 : -0.86602540378443864676372317075294)
         : r == 5 ? (k == 0 ? 0.0 : k == 1 ? 0.95105651629515357211643933337938
                   : k == 2 ? 0.58778525229247312916870595463907 : k == 3 ? -0.58778525229247312916870595463907
                                                                        : -0.95105651629515357211643933337938)
         : (k == 0 ? 0.0 : k == 1 ? 0.78183148246802980870844452667406 : k == 2 ? 0.97492791218182360701813168299393
           : k == 3 ? 0.43388373911755812047576833284835 : k == 4 ? -0.43388373911755812047576833284835
           : k == 5 ? -0.97492791218182360701813168299393 : -0.78183148246802980870844452667406);
}

// cos / sin (2 pi m / R) as compile-time constants: the angle is reduced
// exactly on the integer numerator to [0, pi/4] (quadrant + reflection) and
// the Taylor series there is summed far below one fp64 ulp.
__host__ __device__ constexpr double gen_tsin(double x) {
    double t = x, s = x;
    for (int k = 1; k < 14; ++k) {
        t *= -x * x / ((2.0 * k) * (2.0 * k + 1.0));
        s += t;
    }
    return s;
}
__host__ __device__ constexpr double gen_tcos(double x) {
    double t = 1.0, s = 1.0;
    for (int k = 1; k < 14; ++k) {
        t *= -x * x / ((2.0 * k - 1.0) * (2.0 * k));
        s += t;
    }
    return s;
}
__host__ __device__ constexpr double gen_kc(int R, int m, bool want_sin) {
    const int mm = ((m % R) + R) % R;
    const int u = 4 * mm, q = u / R, r = u - q * R;              // angle = (q + r / R) pi / 2
    const double half_pi = 1.57079632679489661923132169163975;
    double c0 = 0.0, s0 = 0.0;
    if (2 * r <= R) {
        const double a = half_pi * r / R;
        c0 = gen_tcos(a);
        s0 = gen_tsin(a);
    } else {
        const double a = half_pi * (R - r) / R;
        c0 = gen_tsin(a);
        s0 = gen_tcos(a);
    }
    double c = c0, s = s0;
    if (q == 1) { c = -s0; s = c0; }
    else if (q == 2) { c = -c0; s = -s0; }
    else if (q == 3) { c = s0; s = -c0; }
    return want_sin ? s : c;
}

// Composite radices R = A * B, run in registers (Cooley-Tukey with
// n = b + B a, k = ka + A kb); A = 0 marks a base radix (2, 3, 4, 5, 7, 8).
// More splits (e.g. 25 = 5 x 5, 32 = 8 x 4) only need a line here, a case in
// gen_passes and an entry in gen_factor's list.
template <int R> struct GenSplit { static constexpr int A = 0, B = 0; };
#define PM_GEN_SPLIT(R_, A_, B_) \
    template <> struct GenSplit<R_> { static constexpr int A = A_, B = B_; };
PM_GEN_SPLIT(9, 3, 3)
PM_GEN_SPLIT(10, 5, 2)
PM_GEN_SPLIT(12, 4, 3)
PM_GEN_SPLIT(16, 4, 4)
#undef PM_GEN_SPLIT

// Compile-time loop: f(integral_constant<int, i>) for i in [I, N).
template <int I, int N>
struct GenFor {
    template <class F>
    __device__ __forceinline__ static void run(F&& f) {
        if constexpr (I < N) {
            f(std::integral_constant<int, I>{});
            GenFor<I + 1, N>::run(f);
        }
    }
};

template <typename T, int R, int DIR>
__device__ __forceinline__ void gen_dft(cx<T>* x);

template <typename T, int R, int DIR>
__device__ __forceinline__ void gen_dft_split(cx<T>* x) {
    constexpr int A = GenSplit<R>::A, B = GenSplit<R>::B;
    cx<T> y[R];
    GenFor<0, B>::run([&](auto bc) {
        constexpr int b = decltype(bc)::value;
        cx<T> s[A];
#pragma unroll
        for (int a = 0; a < A; ++a) s[a] = x[b + B * a];
        gen_dft<T, A, DIR>(s);
        GenFor<0, A>::run([&](auto kc) {
            constexpr int ka = decltype(kc)::value;
            if constexpr (b * ka == 0) {
                y[b * A + ka] = s[ka];
            } else {
                // W_R^{b ka} = exp(DIR 2 pi i b ka / R)
                constexpr double c = gen_kc(R, b * ka, false), sn = DIR * gen_kc(R, b * ka, true);
                y[b * A + ka] = cmul_cs(s[ka], T(c), T(sn));
            }
        });
    });
#pragma unroll
    for (int ka = 0; ka < A; ++ka) {
        cx<T> s[B];
#pragma unroll
        for (int b = 0; b < B; ++b) s[b] = y[b * A + ka];
        gen_dft<T, B, DIR>(s);
#pragma unroll
        for (int kb = 0; kb < B; ++kb) x[ka + A * kb] = s[kb];
    }
}

// r + c a with a real broadcast (one FFMA2 in fp32).
__device__ __forceinline__ float2 cfmas(float2 a, float c, float2 r) { return fma2(a, make_float2(c, c), r); }
__device__ __forceinline__ double2 cfmas(double2 a, double c, double2 r) {
    return make_double2(r.x + c * a.x, r.y + c * a.y);
}

// In-place DFT of R points, sign DIR (-1 forward), natural order; fp32 in
// packed f32x2 arithmetic (pm_fft.cuh helpers).
template <typename T, int R, int DIR>
__device__ __forceinline__ void gen_dft(cx<T>* x) {
    if constexpr (GenSplit<R>::A > 0) {
        gen_dft_split<T, R, DIR>(x);
    } else if constexpr (R == 2) {
        const cx<T> a = x[0], b = x[1];
        x[0] = cadd(a, b);
        x[1] = csub(a, b);
    } else if constexpr (R == 4) {
        const cx<T> s02 = cadd(x[0], x[2]), d02 = csub(x[0], x[2]);
        const cx<T> s13 = cadd(x[1], x[3]), d13 = csub(x[1], x[3]);
        x[0] = cadd(s02, s13);
        x[2] = csub(s02, s13);
        x[1] = add_rot<DIR>(d02, d13);          // d02 + DIR i d13
        x[3] = add_rot<-DIR>(d02, d13);
    } else if constexpr (R == 8) {
        // two radix-4 DFTs (even / odd samples) combined with W8^k
        cx<T> e[4] = {x[0], x[2], x[4], x[6]}, o[4] = {x[1], x[3], x[5], x[7]};
        gen_dft<T, 4, DIR>(e);
        gen_dft<T, 4, DIR>(o);
        const T h = T(0.70710678118654752440084436210485);
        const cx<T> o1 = cmul_cs(o[1], h, T(DIR) * h);       // W8^1 = h (1 + DIR i)
        const cx<T> o3 = cmul_cs(o[3], -h, T(DIR) * h);      // W8^3 = h (-1 + DIR i)
        x[0] = cadd(e[0], o[0]);
        x[4] = csub(e[0], o[0]);
        x[1] = cadd(e[1], o1);
        x[5] = csub(e[1], o1);
        x[2] = add_rot<DIR>(e[2], o[2]);                     // W8^2 = DIR i
        x[6] = add_rot<-DIR>(e[2], o[2]);
        x[3] = cadd(e[3], o3);
        x[7] = csub(e[3], o3);
    } else {
        // odd R: pair the samples n and R - n (a = sum, b = difference), so
        // y_j / y_{R-j} = x0 + sum_k c(jk) a_k  +/-  i DIR sum_k s(jk) b_k
        constexpr int H = (R - 1) / 2;
        cx<T> a[H], b[H];
#pragma unroll
        for (int k = 0; k < H; ++k) {
            a[k] = cadd(x[k + 1], x[R - 1 - k]);
            b[k] = csub(x[k + 1], x[R - 1 - k]);
        }
        const cx<T> x0 = x[0];
        cx<T> s0 = x0;
#pragma unroll
        for (int k = 0; k < H; ++k) s0 = cadd(s0, a[k]);
        x[0] = s0;
#pragma unroll
        for (int j = 1; j <= H; ++j) {
            cx<T> re = x0, im = mk<T>(T(0), T(0));
#pragma unroll
            for (int k = 0; k < H; ++k) {
                re = cfmas(a[k], T(gen_c(R, (j * (k + 1)) % R)), re);
                im = cfmas(b[k], T(DIR) * T(gen_s(R, (j * (k + 1)) % R)), im);
            }
            x[j] = add_rot<1>(re, im);          // re + i im
            x[R - j] = add_rot<-1>(re, im);
        }
    }
}

// x / d for 0 <= x, d <= 4096 by a multiply-high: mg = ceil(2^32 / d) is
// exact for x < 2^32 / d (d = 1 handled apart, its magic overflows;
// computed on the host, GenPlan::mg).
__device__ __forceinline__ int gen_div(int x, int d, unsigned mg) { return d == 1 ? x : (int)__umulhi((unsigned)x, mg); }

// One Stockham pass of radix R over the TC transforms held in `a`
// ([L][TC] layout, TC a power of two), into `b`. tw[k] = exp(-2 pi i k / L),
// resident in shared memory.
template <typename T, int R>
__device__ __forceinline__ void gen_pass(const cx<T>* a, cx<T>* b, const cx<T>* tw, int L, int Ns, int step,
                                         unsigned mg, int lgTC, int dir) {
    const int TC = 1 << lgTC;
    const int M = L / R;                        // q * k * step < L
    for (int idx = threadIdx.x; idx < M * TC; idx += blockDim.x) {
        const int t = idx & (TC - 1), jb = idx >> lgTC;
        const int g = gen_div(jb, Ns, mg), k = jb - g * Ns;
        cx<T> x[R];
#pragma unroll
        for (int q = 0; q < R; ++q) x[q] = a[(jb + q * M) * TC + t];
        if (k > 0) {
#pragma unroll
            for (int q = 1; q < R; ++q) {
                const cx<T> w = tw[q * k * step];
                x[q] = cmul_cs(x[q], w.x, dir < 0 ? w.y : -w.y);
            }
        }
        if (dir < 0) gen_dft<T, R, -1>(x);
        else gen_dft<T, R, +1>(x);
        const int o = g * Ns * R + k;
#pragma unroll
        for (int q = 0; q < R; ++q) b[(o + q * Ns) * TC + t] = x[q];
    }
}

// All Stockham passes of one direction over the [L][TC] tile in A (B is the
// ping-pong buffer); returns the buffer holding the result.
template <typename T>
__device__ __forceinline__ cx<T>* gen_passes(cx<T>* A, cx<T>* B, const cx<T>* tw, const GenPlan& gp, int lgTC,
                                            int dir) {
    for (int s = 0; s < gp.np; ++s) {
        const int L = gp.L, Ns = gp.ns[s], st = gp.step[s];
        const unsigned mg = gp.mg[s];
#define PM_GEN_CASE(R_) \
    case R_: gen_pass<T, R_>(A, B, tw, L, Ns, st, mg, lgTC, dir); break;
        switch (gp.radix[s]) {   // the radices gen_factor plans with (pm_capi.cu)
            PM_GEN_CASE(2) PM_GEN_CASE(3) PM_GEN_CASE(4) PM_GEN_CASE(5) PM_GEN_CASE(7) PM_GEN_CASE(8)
            PM_GEN_CASE(9) PM_GEN_CASE(10) PM_GEN_CASE(12) PM_GEN_CASE(16)
            default: __trap();
        }
#undef PM_GEN_CASE
        __syncthreads();
        cx<T>* tmp = A; A = B; B = tmp;
    }
    return A;
}

// Shared-memory layout of the mixed-radix kernels: two [L][TC] complex
// tiles, the length-L twiddle table and a [L][TC] real tile (p or m).
template <typename T>
struct GenSmem {
    cx<T>* A;
    cx<T>* B;
    cx<T>* tw;
    T* g;
    __device__ GenSmem(unsigned char* raw, int L, int TC) {
        A = reinterpret_cast<cx<T>*>(raw);
        B = A + (size_t)L * TC;
        tw = B + (size_t)L * TC;
        g = reinterpret_cast<T*>(tw + L);
    }
};
__host__ __device__ constexpr size_t gen_smem_bytes(int L, int TC, int csz) {
    return (2 * (size_t)L * TC + L) * csz + (size_t)L * TC * (csz / 2);
}

// Asynchronous copies into the tiles (cp.async; the caller commits / waits):
// the twiddle table, and TC transforms of length L starting at transform t0
// (element n of transform t at t*tstride + n*estride), complex or real.
template <typename T>
__device__ __forceinline__ void gen_load_tw(cx<T>* tw, const cx<T>* src, int L) {
    for (int i = threadIdx.x; i < L; i += blockDim.x) cp_async<sizeof(cx<T>)>(tw + i, src + i);
}
// Programmatic dependent launch: wait until this kernel's predecessor has
// completed and its writes are visible (a no-op without the launch
// attribute); the successor is released as this grid's CTAs exit.
#ifndef PM_PDL_EARLY
#define PM_PDL_EARLY 0   // trigger the successor at kernel start (measured slower: its waiting CTAs hold slots)
#endif
__device__ __forceinline__ void gen_pdl_wait() {
#if PM_PDL_EARLY
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

template <typename E>
__device__ __forceinline__ void gen_gather(E* A, const E* src, int L, int lgTC, int t0, int tc, long long tstride,
                                           long long estride, E zero) {
    const int TC = 1 << lgTC;
    if (estride == 1) {                           // rows: walk along n for coalescing
        for (int t = 0; t < TC; ++t)
            for (int n = threadIdx.x; n < L; n += blockDim.x) {
                if (t < tc) cp_async<sizeof(E)>(A + n * TC + t, src + (t0 + t) * tstride + n);
                else A[n * TC + t] = zero;
            }
    } else {                                      // columns: walk along t
        for (int idx = threadIdx.x; idx < L * TC; idx += blockDim.x) {
            const int n = idx >> lgTC, t = idx & (TC - 1);
            if (t < tc) cp_async<sizeof(E)>(A + idx, src + (t0 + t) * tstride + n * estride);
            else A[idx] = zero;
        }
    }
}
template <typename T>
__device__ __forceinline__ void gen_scatter(const cx<T>* A, cx<T>* dst, int L, int lgTC, int t0, int tc,
                                            long long tstride, long long estride, T scale) {
    const int TC = 1 << lgTC;
    if (estride == 1) {
        for (int t = 0; t < tc; ++t)
            for (int n = threadIdx.x; n < L; n += blockDim.x)
                dst[(t0 + t) * tstride + n] = cscale(A[n * TC + t], scale);
    } else {
        for (int idx = threadIdx.x; idx < L * TC; idx += blockDim.x) {
            const int n = idx >> lgTC, t = idx & (TC - 1);
            if (t < tc) dst[(t0 + t) * tstride + n * estride] = cscale(A[idx], scale);
        }
    }
}

// One axis of the unitary 2-D DFT for `ntrans` transforms of length gp.L per
// batch slice: element n of transform t at t*tstride + n*estride (+ slice *
// bstride). Skips masks that are stopped (unless all_masks) or diverged.
template <typename T>
__global__ void gen_fft_kernel(const cx<T>* in, cx<T>* out, const cx<T>* __restrict__ tw, GenPlan gp, int ntrans,
                               long long tstride, long long estride, long long bstride, int dir, T scale, int lgTC,
                               const MaskState* st, int all_masks) {
    extern __shared__ __align__(16) unsigned char smraw[];
    const int b = blockIdx.y;
    if (st && (st[b].done || (!all_masks && st[b].stop))) return;
    const int TC = 1 << lgTC, L = gp.L;
    const int t0 = blockIdx.x * TC, tc = min(TC, ntrans - t0);
    GenSmem<T> sm(smraw, L, TC);
    gen_load_tw<T>(sm.tw, tw, L);
    gen_gather<cx<T>>(sm.A, in + b * bstride, L, lgTC, t0, tc, tstride, estride, mk<T>(T(0), T(0)));
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();
    const cx<T>* R = gen_passes<T>(sm.A, sm.B, sm.tw, gp, lgTC, dir);
    gen_scatter<T>(R, out + b * bstride, L, lgTC, t0, tc, tstride, estride, scale);
}

struct GenSolveArgs;

struct GenSolveArgs {
    SolveCtl ctl;
    MaskState* st;
    double* hist;
    int hist_stride;
    double* part;         // [batch][nblk][3]
    unsigned* ctr;
    int nblk;
    long long n;          // pixels per mask
};

// Column sweep of the mixed-radix solve, fused: ColFFT -> replace_m (+ the
// metrics and decision of u_{u_iter}) -> ColIFFT on the work buffer `w`
// (rows already transformed), in place; metrics_only leaves `w` untouched.
template <typename T>
__global__ void gen_col_sweep_kernel(cx<T>* w, const T* m, const T* mT, const double* thr_m, const double* escale,
                                     const cx<T>* __restrict__ tw, GenPlan gp, int nx, int lgTC, GenSolveArgs g,
                                     int u_iter, int metrics_only, int all_masks, int raar, int need_dec) {
    extern __shared__ __align__(16) unsigned char smraw[];
    const int TC = 1 << lgTC, L = gp.L;
    GenSmem<T> sm(smraw, L, TC);
    gen_load_tw<T>(sm.tw, tw, L);                 // constant: before the predecessor completes
    gen_pdl_wait();
    const int b = blockIdx.y;
    MaskState* st = g.st + b;
    if (st->done || (!all_masks && st->stop)) return;
    // need_dec (host): a record, early stopping, a host verdict or max_iters wants
    // this iterate decided now; otherwise the sweep skips the metrics and the
    // per-mask ticket (a non-finite iterate's first iteration stays in `bad`
    // until the next decision)
    const bool dec = need_dec && u_iter >= 1 && st->decided < u_iter && !st->stop;
    const bool rec = dec && recorded(g.ctl, u_iter);
    // RAAR: only lit / dark here (kept in the mask state); the gap and the
    // decision come from the next row sweep, where x and P_M x meet
    const bool gneed = dec && !raar && gap_needed(g.ctl, u_iter);
    const int t0 = blockIdx.x * TC, tc = min(TC, nx - t0);
    const T sc = T(1.0 / sqrt((double)L));
    cx<T>* wb = w + b * g.n;
    gen_gather<cx<T>>(sm.A, wb, L, lgTC, t0, tc, 1, nx, mk<T>(T(0), T(0)));
    cp_async_commit();
    if (mT)   // m transposed per mask: each of the TC columns is one contiguous run
        gen_gather<T>(sm.g, mT + b * g.n, L, lgTC, t0, tc, L, 1, T(0));
    else
        gen_gather<T>(sm.g, m + b * g.n, L, lgTC, t0, tc, 1, nx, T(0));
    // (m stays in flight during the passes)
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    cx<T>* A = gen_passes<T>(sm.A, sm.B, sm.tw, gp, lgTC, -1);
    cx<T>* B = A == sm.A ? sm.B : sm.A;
    cp_async_wait<0>();
    __syncthreads();
    const ZThr<T> thr = zthr<T>(T(thr_m[b]));
    const double es = escale[b];
    double acc[3] = {0.0, 0.0, 0.0};
    cx<T> chk = mk<T>(T(0), T(0));
    for (int idx = threadIdx.x; idx < L * TC; idx += blockDim.x) {
        const int t = idx & (TC - 1);
        if (t >= tc) continue;
        const cx<T> u = cscale(A[idx], sc);                      // u^ = F(u)
        fold_finite(chk, u);                                     // Field check of iteration u_iter + 1
        const T mm = sm.g[idx];
        const cx<T> vh = replace_mod(u, mm, thr);
        if (gneed) acc[0] += norm_sq_d(csub(u, vh));
        if (rec) {
            const double inten = norm_sq_d(u) * es;
            const double m2 = (double)mm * (double)mm;
            if (!(inten <= 1.7976931348623157e308)) {
                acc[1] = __longlong_as_double(0x7ff8000000000000LL);       // RealGrid's check (src/grid.py:128-129)
            } else if (m2 > 0.0) {
                const double dev = fabs(m2 - inten);
                if (dev > g.ctl.t_lit * m2 && dev / m2 > g.ctl.t_lit)
                    acc[1] += g.ctl.t_dark * dev / (g.ctl.t_lit * m2) - g.ctl.t_dark;
            } else if (inten > g.ctl.t_dark) {
                acc[2] += inten - g.ctl.t_dark;
            }
        }
        A[idx] = vh;
    }
    if (!metrics_only && !all_finite(chk)) first_bad(&st->bad, u_iter + 1);
    __syncthreads();
    if (!metrics_only) {
        A = gen_passes<T>(A, B, sm.tw, gp, lgTC, +1);
        gen_scatter<T>(A, wb, L, lgTC, t0, tc, 1, nx, sc);
    }
    if (!dec) return;
    double tot[3];
    if (reduce_ticket<3>(acc, g.part + (size_t)b * g.nblk * 3, g.ctr + b, g.nblk, blockIdx.x, tot) &&
        threadIdx.x == 0) {
        if (raar) {
            st->pend_lit = tot[1];
            st->pend_dark = tot[2];
        } else {
            decide(st, g.hist + ((size_t)b * g.hist_stride + (u_iter - 1)) * 4, g.ctl, u_iter, rec, tot);
        }
    }
}

// Row sweep of the mixed-radix solve, fused: RowIFFT of the work buffer ->
// u = P_S v into the iterate (non-finite check) -> RowFFT(u) back into the
// work buffer for the next column sweep.
template <typename T>
__global__ void gen_row_sweep_kernel(cx<T>* w, cx<T>* u, const T* p, long long p_stride, const double* thr_p,
                                     const cx<T>* __restrict__ tw, GenPlan gp, int ny, int lgTC, MaskState* st,
                                     long long n, int it, int store_u) {
    extern __shared__ __align__(16) unsigned char smraw[];
    const int TC = 1 << lgTC, L = gp.L;
    GenSmem<T> sm(smraw, L, TC);
    gen_load_tw<T>(sm.tw, tw, L);                 // constant: before the predecessor completes
    gen_pdl_wait();
    const int b = blockIdx.y;
    if (st[b].done || st[b].stop) return;
    const int t0 = blockIdx.x * TC, tc = min(TC, ny - t0);
    const T sc = T(1.0 / sqrt((double)L));
    cx<T>* wb = w + b * n;
    cx<T>* ub = u + b * n;
    gen_gather<cx<T>>(sm.A, wb, L, lgTC, t0, tc, L, 1, mk<T>(T(0), T(0)));
    cp_async_commit();
    gen_gather<T>(sm.g, p + b * p_stride, L, lgTC, t0, tc, L, 1, T(0));  // p, in flight during the passes
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    cx<T>* A = gen_passes<T>(sm.A, sm.B, sm.tw, gp, lgTC, +1);
    cx<T>* B = A == sm.A ? sm.B : sm.A;
    cp_async_wait<0>();
    __syncthreads();
    const ZThr<T> thr = zthr<T>(T(thr_p[b]));
    cx<T> chk = mk<T>(T(0), T(0));
    for (int idx = threadIdx.x; idx < L * TC; idx += blockDim.x) {
        const int t = idx & (TC - 1);                        // element idx >> lgTC of row t0 + t
        if (t >= tc) continue;
        const cx<T> v = cscale(A[idx], sc);
        fold_finite(chk, v);                                 // v = F^-1 v^ (reference Field check)
        A[idx] = replace_mod(v, sm.g[idx], thr);
    }
    if (!all_finite(chk)) first_bad(&st[b].bad, it);
    __syncthreads();
    if (store_u) gen_scatter<T>(A, ub, L, lgTC, t0, tc, L, 1, T(1));   // the iterate (stepping sessions)
    A = gen_passes<T>(A, B, sm.tw, gp, lgTC, -1);
    gen_scatter<T>(A, wb, L, lgTC, t0, tc, L, 1, sc);
}

// RAAR row sweep of iteration `it`: RowIFFT of the work
// buffer gives v = P_M x_{it-1}; with x_{it-1} from `x_in`:
//   gap of x_{it-1} = ||P_S x_{it-1} - v|| (src/metrics.py:67-71), when needed;
//   x_it = beta x + beta P_S(2v - x) + (1 - 2 beta) v into `x_out` (upd), in
//   numpy's operation order, then RowFFT(x_it) back into the work buffer.
// The iterates alternate between two buffers so a mask that stops at
// x_{it-1} (decided here, after x_it is written) keeps it. The last CTA of a
// mask (ticket) sums the gap and |x_it|^2 partials in a fixed order, takes
// the record / early-stop decision of x_{it-1} with the column sweep's
// lit / dark, and leaves E / sum |x_it|^2 (the reconstructed-intensity scale of
// x_it) in `xsc` for the next column sweep. upd = 0: measure and decide only
// (the last iterate, the stepping API's probe).
template <typename T>
__global__ void gen_row_raar_kernel(cx<T>* w, const cx<T>* x_in, cx<T>* x_out, const T* p, long long p_stride,
                                    const double* thr_p, const cx<T>* __restrict__ tw, GenPlan gp, int ny, int lgTC,
                                    GenSolveArgs g, T beta, T c1, const double* energy, double* xsc, int it,
                                    int upd) {
    extern __shared__ __align__(16) unsigned char smraw[];
    const int TC = 1 << lgTC, L = gp.L;
    GenSmem<T> sm(smraw, L, TC);
    gen_load_tw<T>(sm.tw, tw, L);
    gen_pdl_wait();
    const int b = blockIdx.y;
    MaskState* st = g.st + b;
    if (st->done || st->stop) return;
    const int i = it - 1;                                     // the iterate measured here
    const bool dec = i >= 1 && st->decided < i;
    const bool rec = dec && recorded(g.ctl, i);
    const bool gneed = dec && gap_needed(g.ctl, i);
    const int t0 = blockIdx.x * TC, tc = min(TC, ny - t0);
    const T sc = T(1.0 / sqrt((double)L));
    cx<T>* wb = w + b * g.n;
    gen_gather<cx<T>>(sm.A, wb, L, lgTC, t0, tc, L, 1, mk<T>(T(0), T(0)));
    cp_async_commit();
    gen_gather<T>(sm.g, p + b * p_stride, L, lgTC, t0, tc, L, 1, T(0));
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    cx<T>* A = gen_passes<T>(sm.A, sm.B, sm.tw, gp, lgTC, +1);
    cx<T>* B = A == sm.A ? sm.B : sm.A;
    cp_async_wait<0>();
    __syncthreads();
    const ZThr<T> thr = zthr<T>(T(thr_p[b]));
    const cx<T>* xb = x_in + b * g.n;
    cx<T>* xo = x_out + b * g.n;
    double g2 = 0.0, e2 = 0.0;
    for (int idx = threadIdx.x; idx < L * TC; idx += blockDim.x) {
        const int k = idx >> lgTC, t = idx & (TC - 1);
        if (t >= tc) continue;
        const long long e = (long long)(t0 + t) * L + k;
        const cx<T> vv = cscale(A[idx], sc);                  // v = P_M x_{it-1}
        const cx<T> xx = xb[e];
        const T pk = sm.g[idx];
        if (gneed) g2 += norm_sq_d(csub_rn(replace_mod(xx, pk, thr), vv));
        if (upd) {
            const cx<T> py = replace_mod(csub_rn(cscale(vv, T(2)), xx), pk, thr);
            const cx<T> xn = cadd_rn(cadd_rn(cmul_rn(xx, beta), cmul_rn(py, beta)), cmul_rn(vv, c1));
            xo[e] = xn;
            e2 += norm_sq_d(xn);
            A[idx] = xn;
        }
    }
    if (upd && !isfinite(e2)) first_bad(&st->bad, it);
    double acc[2] = {g2, e2}, tot[2];
    const bool last = reduce_ticket<2>(acc, g.part + (size_t)b * g.nblk * 2, g.ctr + b, g.nblk, blockIdx.x, tot);
    if (last && threadIdx.x == 0) {
        if (upd) xsc[b] = energy[b] / tot[1];
        if (dec) {
            const double t3[3] = {tot[0], st->pend_lit, st->pend_dark};
            decide(st, g.hist + ((size_t)b * g.hist_stride + (i - 1)) * 4, g.ctl, i, rec, t3);
        }
    }
    if (!upd) return;
    __syncthreads();
    A = gen_passes<T>(A, B, sm.tw, gp, lgTC, -1);
    gen_scatter<T>(A, wb, L, lgTC, t0, tc, L, 1, sc);
}

// RAAR finish: the final iterate of mask b is x_j, j = iters_run (stopped)
// or `it` (aborted); odd j lives in the second buffer and is copied into the
// first, which the best-approximation pair then reads.
template <typename T>
__global__ void gen_pick_kernel(cx<T>* x0, const cx<T>* x1, const MaskState* st, long long n, int it) {
    const int b = blockIdx.y;
    if (st[b].done) return;
    const int j = st[b].stop ? st[b].iters_run : it;
    if (!(j & 1)) return;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        x0[b * n + i] = x1[b * n + i];
}

// Best-approximation pair and mask from v* (src/solver.py:201-206).
template <typename T>
__global__ void gen_final_kernel(const cx<T>* vs, const T* p, long long p_stride, const double* tol_p,
                                 const MaskState* st, long long n, cx<T>* v_star, cx<T>* u_star, double* phases,
                                 uint8_t* levels) {
    const int b = blockIdx.y;
    if (st[b].done) return;
    const T tol = T(tol_p[b]);
    cx<T> chk = mk<T>(T(0), T(0));
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const long long x = b * n + i;
        const cx<T> v = vs[x];
        fold_finite(chk, v);
        if (v_star) v_star[x] = v;
        const cx<T> us = replace_mod_exact<T>(v, p[b * p_stride + i], tol);
        if (u_star) u_star[x] = us;
        if (phases || levels) {
            double th = phase_of((double)us.x, (double)us.y);
            if (tol > T(0) && np_cabs(us) < tol) th = 0.0;        // np.abs(u*) < zero_tol
            if (phases) phases[x] = th;
            if (levels) levels[x] = level_of(th);
        }
    }
    if (!all_finite(chk)) const_cast<MaskState*>(st)[b].pair_bad = 1;
}

// Real m -> complex field (the initial iterate's Fourier-plane start).
template <typename T>
__global__ void gen_real_to_complex(const T* m, cx<T>* f, long long total) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x)
        f[i] = mk<T>(m[i], T(0));
}

}  // namespace pm
