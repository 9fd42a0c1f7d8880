// Mixed-radix path for grids whose sides are not powers of two (radices 2,
// 3, 4, 5, 7; n <= 4096), e.g. the paper's 800x600 SLM and
// the reference's acceptance grid (tests/test_acceptance.py:118-128,200-205).
//
// The power-of-two path fuses each half iteration into one register-resident
// sweep; this path is a plain sequence of kernels over a work buffer, which
// is enough for the sizes it serves:
//   gen_fft_kernel      one axis of a unitary 2-D DFT: a CTA gathers TC
//                       transforms into shared memory (coalesced along
//                       whichever axis is contiguous), runs the Stockham
//                       passes there and scatters the result;
//   gen_replace_kernel  replace_m in the Fourier plane + the metrics of the
//                       iterate (gap by Parseval, E_lit / E_dark) reduced
//                       per block in a fixed order; the last block decides
//                       (record / early stop / max_iters / divergence);
//   gen_slm_kernel      P_S back into the iterate + non-finite detection;
//   gen_final_kernel    u* = P_S v*, the float64 mask and uint8 levels.
// Semantics (threshold decisions, fixed-order fp64 sums, stop logic) are the
// fused path's: see pm_kernels.cuh.
#pragma once
#include "pm_kernels.cuh"

namespace pm {

constexpr int kGenMaxPasses = 16;

struct GenPlan {
    int L;                       // transform length
    int np;                      // passes
    int radix[kGenMaxPasses];    // radix of pass s
    int ns[kGenMaxPasses];       // product of the radices before pass s
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

// In-place DFT of R points, sign DIR (-1 forward), natural order.
template <typename T, int R, int DIR>
__device__ __forceinline__ void gen_dft(cx<T>* x) {
    if constexpr (R == 2) {
        const cx<T> a = x[0], b = x[1];
        x[0] = mk<T>(a.x + b.x, a.y + b.y);
        x[1] = mk<T>(a.x - b.x, a.y - b.y);
    } else if constexpr (R == 4) {
        const cx<T> s02 = mk<T>(x[0].x + x[2].x, x[0].y + x[2].y), d02 = mk<T>(x[0].x - x[2].x, x[0].y - x[2].y);
        const cx<T> s13 = mk<T>(x[1].x + x[3].x, x[1].y + x[3].y), d13 = mk<T>(x[1].x - x[3].x, x[1].y - x[3].y);
        // DIR * i * d13
        const cx<T> r13 = DIR < 0 ? mk<T>(d13.y, -d13.x) : mk<T>(-d13.y, d13.x);
        x[0] = mk<T>(s02.x + s13.x, s02.y + s13.y);
        x[2] = mk<T>(s02.x - s13.x, s02.y - s13.y);
        x[1] = mk<T>(d02.x + r13.x, d02.y + r13.y);
        x[3] = mk<T>(d02.x - r13.x, d02.y - r13.y);
    } else {
        cx<T> y[R];
#pragma unroll
        for (int k = 0; k < R; ++k) {
            T re = x[0].x, im = x[0].y;
#pragma unroll
            for (int n = 1; n < R; ++n) {
                const T c = T(gen_c(R, (n * k) % R)), s = T(DIR) * T(gen_s(R, (n * k) % R));
                re += x[n].x * c - x[n].y * s;
                im += x[n].x * s + x[n].y * c;
            }
            y[k] = mk<T>(re, im);
        }
#pragma unroll
        for (int k = 0; k < R; ++k) x[k] = y[k];
    }
}

// x / d for 0 <= x, d <= 2^20 without an integer division: the fp64
// product is within 1e-12 of the quotient, far inside 1/d of the next integer.
__device__ __forceinline__ int gen_div(int x, double inv_d) { return (int)((double)x * inv_d + 1e-9); }

// One Stockham pass of radix R over the TC transforms held in `a`
// ([L][TC] layout, TC a power of two), into `b`. tw[k] = exp(-2 pi i k / L).
template <typename T, int R>
__device__ __forceinline__ void gen_pass(const cx<T>* a, cx<T>* b, const cx<T>* __restrict__ tw, int L, int Ns,
                                         int lgTC, int dir) {
    const int TC = 1 << lgTC;
    const int M = L / R;
    const int step = L / (Ns * R);              // twiddle index step per (q * k); q * k * step < L
    const double inv_ns = 1.0 / Ns;
    for (int idx = threadIdx.x; idx < M * TC; idx += blockDim.x) {
        const int t = idx & (TC - 1), jb = idx >> lgTC;
        const int g = gen_div(jb, inv_ns), k = jb - g * Ns;
        cx<T> x[R];
#pragma unroll
        for (int q = 0; q < R; ++q) {
            cx<T> v = a[(jb + q * M) * TC + t];
            if (q > 0 && k > 0) {
                const cx<T> w = __ldg(tw + q * k * step);
                const T ws = dir < 0 ? w.y : -w.y;
                v = mk<T>(v.x * w.x - v.y * ws, v.x * ws + v.y * w.x);
            }
            x[q] = v;
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
__device__ __forceinline__ cx<T>* gen_passes(cx<T>* A, cx<T>* B, const cx<T>* __restrict__ tw, const GenPlan& gp,
                                            int lgTC, int dir) {
    for (int s = 0; s < gp.np; ++s) {
        switch (gp.radix[s]) {
            case 2: gen_pass<T, 2>(A, B, tw, gp.L, gp.ns[s], lgTC, dir); break;
            case 3: gen_pass<T, 3>(A, B, tw, gp.L, gp.ns[s], lgTC, dir); break;
            case 4: gen_pass<T, 4>(A, B, tw, gp.L, gp.ns[s], lgTC, dir); break;
            case 5: gen_pass<T, 5>(A, B, tw, gp.L, gp.ns[s], lgTC, dir); break;
            default: gen_pass<T, 7>(A, B, tw, gp.L, gp.ns[s], lgTC, dir); break;
        }
        __syncthreads();
        cx<T>* tmp = A; A = B; B = tmp;
    }
    return A;
}

// Tile <-> global for TC transforms of length L starting at transform t0
// (element n of transform t at t*tstride + n*estride).
template <typename T>
__device__ __forceinline__ void gen_gather(cx<T>* A, const cx<T>* src, int L, int lgTC, int t0, int tc,
                                           long long tstride, long long estride) {
    const int TC = 1 << lgTC;
    const double inv_l = 1.0 / L;
    for (int idx = threadIdx.x; idx < L * TC; idx += blockDim.x) {
        int n, t;
        if (estride == 1) { t = gen_div(idx, inv_l); n = idx - t * L; }
        else { n = idx >> lgTC; t = idx & (TC - 1); }
        A[n * TC + t] = t < tc ? src[(t0 + t) * tstride + n * estride] : mk<T>(T(0), T(0));
    }
    __syncthreads();
}
template <typename T>
__device__ __forceinline__ void gen_scatter(const cx<T>* A, cx<T>* dst, int L, int lgTC, int t0, int tc,
                                            long long tstride, long long estride, T scale) {
    const int TC = 1 << lgTC;
    const double inv_l = 1.0 / L;
    for (int idx = threadIdx.x; idx < L * TC; idx += blockDim.x) {
        int n, t;
        if (estride == 1) { t = gen_div(idx, inv_l); n = idx - t * L; }
        else { n = idx >> lgTC; t = idx & (TC - 1); }
        if (t < tc) dst[(t0 + t) * tstride + n * estride] = cscale(A[n * TC + t], scale);
    }
}

// One axis of the unitary 2-D DFT for `ntrans` transforms of length gp.L per
// batch slice: element n of transform t at t*tstride + n*estride (+ slice *
// bstride). Skips masks that are stopped (unless all_masks) or diverged.
template <typename T>
__global__ void gen_fft_kernel(const cx<T>* in, cx<T>* out, const cx<T>* __restrict__ tw, GenPlan gp, int ntrans,
                               long long tstride, long long estride, long long bstride, int dir, T scale, int lgTC,
                               const MaskState* st, int all_masks) {
    const int TC = 1 << lgTC;
    extern __shared__ __align__(16) unsigned char smraw[];
    const int b = blockIdx.y;
    if (st && (st[b].done || (!all_masks && st[b].stop))) return;
    const int L = gp.L;
    const int t0 = blockIdx.x * TC;
    const int tc = min(TC, ntrans - t0);
    cx<T>* A = reinterpret_cast<cx<T>*>(smraw);
    cx<T>* B = A + (size_t)L * TC;
    const cx<T>* src = in + b * bstride;
    cx<T>* dst = out + b * bstride;
    const bool contig_e = estride == 1;          // rows: walk along n; columns: walk along t
    const double inv_l = 1.0 / L;
    for (int idx = threadIdx.x; idx < L * TC; idx += blockDim.x) {
        int n, t;
        if (contig_e) { t = gen_div(idx, inv_l); n = idx - t * L; }
        else { n = idx >> lgTC; t = idx & (TC - 1); }
        A[n * TC + t] = t < tc ? src[(t0 + t) * tstride + n * estride] : mk<T>(T(0), T(0));
    }
    __syncthreads();
    for (int s = 0; s < gp.np; ++s) {
        switch (gp.radix[s]) {
            case 2: gen_pass<T, 2>(A, B, tw, L, gp.ns[s], lgTC, dir); break;
            case 3: gen_pass<T, 3>(A, B, tw, L, gp.ns[s], lgTC, dir); break;
            case 4: gen_pass<T, 4>(A, B, tw, L, gp.ns[s], lgTC, dir); break;
            case 5: gen_pass<T, 5>(A, B, tw, L, gp.ns[s], lgTC, dir); break;
            default: gen_pass<T, 7>(A, B, tw, L, gp.ns[s], lgTC, dir); break;
        }
        __syncthreads();
        cx<T>* tmp = A; A = B; B = tmp;
    }
    for (int idx = threadIdx.x; idx < L * TC; idx += blockDim.x) {
        int n, t;
        if (contig_e) { t = gen_div(idx, inv_l); n = idx - t * L; }
        else { n = idx >> lgTC; t = idx & (TC - 1); }
        if (t < tc) dst[(t0 + t) * tstride + n * estride] = cscale(A[n * TC + t], scale);
    }
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

// v^ = replace_m(u^) in place (unless metrics_only), with the metrics of the
// iterate u_{u_iter} when it is decided here: gap^2 = sum |u^ - v^|^2
// (Parseval, GS), E_lit / E_dark of the reconstruction (src/metrics.py:67-112).
template <typename T>
__global__ void gen_replace_kernel(cx<T>* f, const T* m, const double* thr_m, const double* escale, GenSolveArgs g,
                                   int u_iter, int metrics_only, int all_masks) {
    const int b = blockIdx.y;
    MaskState* st = g.st + b;
    if (st->done || (!all_masks && st->stop)) return;
    const bool dec = u_iter >= 1 && st->decided < u_iter && !st->stop;
    const bool rec = dec && recorded(g.ctl, u_iter);
    const bool gneed = dec && gap_needed(g.ctl, u_iter);
    const T thr = T(thr_m[b]);
    const double sc = escale[b];
    cx<T>* fb = f + b * g.n;
    const T* mb = m + b * g.n;
    double acc[3] = {0.0, 0.0, 0.0};
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < g.n;
         i += (long long)gridDim.x * blockDim.x) {
        const cx<T> u = fb[i];
        const T mm = mb[i];
        const cx<T> vh = replace_mod(u, mm, thr);
        if (gneed) acc[0] += norm_sq_d(csub(u, vh));
        if (rec) {
            const double inten = norm_sq_d(u) * sc;
            const double m2 = (double)mm * (double)mm;
            if (m2 > 0.0) {
                const double dev = fabs(m2 - inten);
                if (dev > g.ctl.t_lit * m2 && dev / m2 > g.ctl.t_lit)
                    acc[1] += g.ctl.t_dark * dev / (g.ctl.t_lit * m2) - g.ctl.t_dark;
            } else if (inten > g.ctl.t_dark) {
                acc[2] += inten - g.ctl.t_dark;
            }
        }
        if (!metrics_only) fb[i] = vh;
    }
    if (!dec) return;
    double tot[3];
    if (reduce_ticket<3>(acc, g.part + (size_t)b * g.nblk * 3, g.ctr + b, g.nblk, blockIdx.x, tot) &&
        threadIdx.x == 0)
        decide(st, g.hist + ((size_t)b * g.hist_stride + (u_iter - 1)) * 4, g.ctl, u_iter, rec, tot);
}

// Column sweep of the mixed-radix solve, fused: ColFFT -> replace_m (+ the
// metrics and decision of u_{u_iter}) -> ColIFFT on the work buffer `w`
// (rows already transformed), in place; metrics_only leaves `w` untouched.
template <typename T>
__global__ void gen_col_sweep_kernel(cx<T>* w, const T* m, const double* thr_m, const double* escale,
                                     const cx<T>* __restrict__ tw, GenPlan gp, int nx, int lgTC, GenSolveArgs g,
                                     int u_iter, int metrics_only, int all_masks) {
    extern __shared__ __align__(16) unsigned char smraw[];
    const int b = blockIdx.y;
    MaskState* st = g.st + b;
    if (st->done || (!all_masks && st->stop)) return;
    const bool dec = u_iter >= 1 && st->decided < u_iter && !st->stop;
    const bool rec = dec && recorded(g.ctl, u_iter);
    const bool gneed = dec && gap_needed(g.ctl, u_iter);
    const int TC = 1 << lgTC, L = gp.L;
    const int t0 = blockIdx.x * TC, tc = min(TC, nx - t0);
    const T sc = T(1.0 / sqrt((double)L));
    cx<T>* A = reinterpret_cast<cx<T>*>(smraw);
    cx<T>* B = A + (size_t)L * TC;
    cx<T>* wb = w + b * g.n;
    const T* mb = m + b * g.n;
    gen_gather<T>(A, wb, L, lgTC, t0, tc, 1, nx);
    A = gen_passes<T>(A, B, tw, gp, lgTC, -1);
    B = A == reinterpret_cast<cx<T>*>(smraw) ? A + (size_t)L * TC : reinterpret_cast<cx<T>*>(smraw);
    const T thr = T(thr_m[b]);
    const double es = escale[b];
    double acc[3] = {0.0, 0.0, 0.0};
    for (int idx = threadIdx.x; idx < L * TC; idx += blockDim.x) {
        const int n = idx >> lgTC, t = idx & (TC - 1);
        if (t >= tc) continue;
        const cx<T> u = cscale(A[idx], sc);                      // u^ = F(u)
        const T mm = mb[(long long)n * nx + t0 + t];
        const cx<T> vh = replace_mod(u, mm, thr);
        if (gneed) acc[0] += norm_sq_d(csub(u, vh));
        if (rec) {
            const double inten = norm_sq_d(u) * es;
            const double m2 = (double)mm * (double)mm;
            if (m2 > 0.0) {
                const double dev = fabs(m2 - inten);
                if (dev > g.ctl.t_lit * m2 && dev / m2 > g.ctl.t_lit)
                    acc[1] += g.ctl.t_dark * dev / (g.ctl.t_lit * m2) - g.ctl.t_dark;
            } else if (inten > g.ctl.t_dark) {
                acc[2] += inten - g.ctl.t_dark;
            }
        }
        A[idx] = vh;
    }
    __syncthreads();
    if (!metrics_only) {
        A = gen_passes<T>(A, B, tw, gp, lgTC, +1);
        gen_scatter<T>(A, wb, L, lgTC, t0, tc, 1, nx, sc);
    }
    if (!dec) return;
    double tot[3];
    if (reduce_ticket<3>(acc, g.part + (size_t)b * g.nblk * 3, g.ctr + b, g.nblk, blockIdx.x, tot) &&
        threadIdx.x == 0)
        decide(st, g.hist + ((size_t)b * g.hist_stride + (u_iter - 1)) * 4, g.ctl, u_iter, rec, tot);
}

// Row sweep of the mixed-radix solve, fused: RowIFFT of the work buffer ->
// u = P_S v into the iterate (non-finite check) -> RowFFT(u) back into the
// work buffer for the next column sweep.
template <typename T>
__global__ void gen_row_sweep_kernel(cx<T>* w, cx<T>* u, const T* p, long long p_stride, const double* thr_p,
                                     const cx<T>* __restrict__ tw, GenPlan gp, int ny, int lgTC, MaskState* st,
                                     long long n, int it) {
    extern __shared__ __align__(16) unsigned char smraw[];
    const int b = blockIdx.y;
    if (st[b].done || st[b].stop) return;
    const int TC = 1 << lgTC, L = gp.L;
    const int t0 = blockIdx.x * TC, tc = min(TC, ny - t0);
    const T sc = T(1.0 / sqrt((double)L));
    cx<T>* A = reinterpret_cast<cx<T>*>(smraw);
    cx<T>* B = A + (size_t)L * TC;
    cx<T>* wb = w + b * n;
    cx<T>* ub = u + b * n;
    const T* pb = p + b * p_stride;
    gen_gather<T>(A, wb, L, lgTC, t0, tc, L, 1);
    A = gen_passes<T>(A, B, tw, gp, lgTC, +1);
    B = A == reinterpret_cast<cx<T>*>(smraw) ? A + (size_t)L * TC : reinterpret_cast<cx<T>*>(smraw);
    const T thr = T(thr_p[b]);
    T chk = T(0);
    for (int idx = threadIdx.x; idx < L * TC; idx += blockDim.x) {
        const int k = idx >> lgTC, t = idx & (TC - 1);      // element k of row t0 + t
        if (t >= tc) continue;
        const long long x = (long long)(t0 + t) * L + k;
        T s2;
        const cx<T> uu = replace_mod(cscale(A[idx], sc), pb[x], thr, s2);
        chk += s2;
        ub[x] = uu;
        A[idx] = uu;
    }
    if (!isfinite(chk)) first_bad(&st[b].bad, it);
    __syncthreads();
    A = gen_passes<T>(A, B, tw, gp, lgTC, -1);
    gen_scatter<T>(A, wb, L, lgTC, t0, tc, L, 1, sc);
}

// u = P_S v from the work buffer back into the iterate, non-finite check.
template <typename T>
__global__ void gen_slm_kernel(const cx<T>* v, cx<T>* u, const T* p, long long p_stride, const double* thr_p,
                               MaskState* st, long long n, int it) {
    const int b = blockIdx.y;
    if (st[b].done || st[b].stop) return;
    const T thr = T(thr_p[b]);
    const cx<T>* vb = v + b * n;
    cx<T>* ub = u + b * n;
    const T* pb = p + b * p_stride;
    T chk = T(0);
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        T s2;
        ub[i] = replace_mod(vb[i], pb[i], thr, s2);
        chk += s2;
    }
    if (!isfinite(chk)) first_bad(&st[b].bad, it);
}

// Best-approximation pair and mask from v* (src/solver.py:201-206).
template <typename T>
__global__ void gen_final_kernel(const cx<T>* vs, const T* p, long long p_stride, const double* tol_p,
                                 const MaskState* st, long long n, cx<T>* v_star, cx<T>* u_star, double* phases,
                                 uint8_t* levels) {
    const int b = blockIdx.y;
    if (st[b].done) return;
    const T tol = T(tol_p[b]);
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const long long x = b * n + i;
        const cx<T> v = vs[x];
        if (v_star) v_star[x] = v;
        const cx<T> us = replace_mod_exact<T>(v, p[b * p_stride + i], tol);
        if (u_star) u_star[x] = us;
        if (phases || levels) {
            double th = phase_of((double)us.x, (double)us.y);
            const T mag = sqrt(us.x * us.x + us.y * us.y);
            if (tol > T(0) && mag < tol) th = 0.0;
            if (phases) phases[x] = th;
            if (levels) levels[x] = level_of(th);
        }
    }
}

// Real m -> complex field (the initial iterate's Fourier-plane start).
template <typename T>
__global__ void gen_real_to_complex(const T* m, cx<T>* f, long long total) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x)
        f[i] = mk<T>(m[i], T(0));
}

}  // namespace pm
