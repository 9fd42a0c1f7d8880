// The solver's kernels.
//
// One Gerchberg–Saxton iteration u <- P_S F^-1 replace_m F u
// (reference src/solver.py:150-170) is executed as TWO fused sweeps over the
// field, which lives in HBM/L2 as interleaved complex (n_y, n_x) row-major:
//
//   column sweep  (col_iter_kernel):  w -> column FFT -> [metrics of u] ->
//                 replace modulus with m -> column IFFT -> z
//   row sweep     (row_iter_kernel):  z -> row IFFT -> P_S with p ->
//                 row FFT -> w   (or, on the last iterate: v*, u*, mask)
//
// Between sweeps the field is held "row-transformed" (w = RowFFT(u)), so the
// column sweep completes F(u) and the row sweep completes F^-1(v^). Each
// sweep reads and writes the field once and reads one real grid: 40 B/pixel
// per iteration in fp32, 80 B in fp64.
//
// Convergence metrics (gap, err_lit, err_dark; src/metrics.py:67-112) are
// reduced on the device with a fixed-order tree (per-CTA partials + the last
// CTA of each mask combining them in index order), so they are bitwise
// reproducible run to run and independent of batch size. The last CTA of a
// column sweep also takes the stop decision (max_iters, early stop, host
// abort, non-finite), so a whole solve runs without host round trips.
#pragma once
#include "pm_fft.cuh"

namespace pm {

constexpr double kTwoPi = 6.283185307179586;   // float64(2*np.pi)
constexpr int kColPad = 2;                      // extra elements per column buffer (bank spread)

struct MaskState {
    int stop;        // the current iterate is the last one: next row sweep finalises
    int done;        // final pair written; all later launches exit immediately
    int iters_run;   // SolveResult.iters_run
    int diverged;    // iteration whose iterate went non-finite (0 = never)
    int aborted;     // host requested stop (should_abort)
    int have_prev;   // early stop: a previous gap exists
    int n_records;
    int pad_;
    double prev_gap;
    double energy;   // sum |u|^2 of the latest SLM-plane iterate (fp64)
};

struct SolveCtl {
    int max_iters;
    int record_every;
    double early_tol;   // < 0: early stopping off
    double t_lit, t_dark;
};

template <typename T>
struct RowArgs {
    cx<T>* field;
    const T* p;
    long long p_stride;       // elements between masks' p (0: shared)
    const cx<T>* tw;
    int nx, ny;
    T scale;                  // 1/sqrt(nx)
    const double* tol_p;      // [batch]
    int mode;                 // 0: no projection (initial iterate), 1: iterate, 2: final
    int it;                   // index of the iterate this sweep produces
    MaskState* st;
    double* part;             // [batch][nblk][2]
    unsigned* ctr;            // [batch]
    int nblk;
    cx<T>* v_star;            // final outputs, nullable
    cx<T>* u_star;
    double* phases;
    uint8_t* levels;
};

template <typename T>
struct ColArgs {
    cx<T>* field;
    const T* m;
    long long m_stride;
    const cx<T>* tw;
    int nx, ny;
    T scale;                  // 1/sqrt(ny)
    const double* tol_m;      // [batch]
    const double* energy_target;  // [batch] sum m^2 (fp64)
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

__device__ __forceinline__ bool finite2(float2 a) { return isfinite(a.x) && isfinite(a.y); }
__device__ __forceinline__ bool finite2(double2 a) { return isfinite(a.x) && isfinite(a.y); }

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
        double x = acc[v];
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
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
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            double x = 0.0;
            for (int i = lane; i < nblk; i += 32) x += __ldcg(&part[i * NV + v]);
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
            if (lane == 0) tot[v] = x;
        }
    }
    if (threadIdx.x == 0) *ctr = 0u;
    return true;
}

// Phase of the complex128-cast value, np.mod(., 2pi) semantics, >= 2pi -> 0
// (src/grid.py:168-176).
__device__ __forceinline__ double phase_of(double re, double im) {
    double th = atan2(im, re);
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

// ----------------------------------------------------------------- row sweep
template <typename T, int LG_L, int LG_R>
__global__ void __launch_bounds__(256) row_iter_kernel(RowArgs<T> a) {
    using F = FftShape<LG_L, LG_R>;
    extern __shared__ __align__(16) unsigned char smraw[];
    const int b = blockIdx.y;
    MaskState* st = a.st + b;
    if (st->done) return;
    const bool fin = a.mode == 2 || st->stop;
    const int G = blockDim.x / F::TG;
    const int g = threadIdx.x / F::TG, j = threadIdx.x % F::TG;
    const int row = blockIdx.x * G + g;
    const size_t N = (size_t)a.nx * a.ny;
    cx<T>* sm = reinterpret_cast<cx<T>*>(smraw) + g * F::SM;
    cx<T>* f = a.field + b * N + (size_t)row * a.nx;
    const T* p = a.p + b * a.p_stride + (size_t)row * a.nx;

    cx<T> v[F::R];
#pragma unroll
    for (int k = 0; k < F::R; ++k) v[k] = f[j + F::TG * k];

    double acc[2] = {0.0, 0.0};   // energy sum |u|^2, non-finite count
    if constexpr (F::TG <= 32) {
        fft1d<T, LG_L, LG_R, +1>(v, sm, a.tw, j, SyncWarp{});
    } else {
        fft1d<T, LG_L, LG_R, +1>(v, sm, a.tw, j, SyncBlock{});
    }
    const T tol = T(a.tol_p[b]);
#pragma unroll
    for (int k = 0; k < F::R; ++k) { v[k].x *= a.scale; v[k].y *= a.scale; }

    if (fin) {
        // Best-approximation pair: v* = P_M u_K (this row's IFFT), u* = P_S v*,
        // mask = phases_of(u*, tol_p)  (src/solver.py:201-206).
        const size_t o = b * N + (size_t)row * a.nx;
#pragma unroll
        for (int k = 0; k < F::R; ++k) {
            const int x = j + F::TG * k;
            const cx<T> vs = v[k];
            if (!finite2(vs)) acc[1] += 1.0;
            if (a.v_star) a.v_star[o + x] = vs;
            const cx<T> us = replace_mod(vs, p[x], tol);
            if (a.u_star) a.u_star[o + x] = us;
            double th = phase_of((double)us.x, (double)us.y);
            const T mag = sqrt(us.x * us.x + us.y * us.y);
            if (tol > T(0) && mag < tol) th = 0.0;
            if (a.phases) a.phases[o + x] = th;
            if (a.levels) a.levels[o + x] = level_of(th);
        }
    } else {
        if (a.mode == 1) {
#pragma unroll
            for (int k = 0; k < F::R; ++k) {
                if (!finite2(v[k])) acc[1] += 1.0;
                v[k] = replace_mod(v[k], p[j + F::TG * k], tol);
                acc[0] += (double)v[k].x * (double)v[k].x + (double)v[k].y * (double)v[k].y;
            }
        }
        if constexpr (F::TG <= 32) {
            fft1d<T, LG_L, LG_R, -1>(v, sm, a.tw, j, SyncWarp{});
        } else {
            fft1d<T, LG_L, LG_R, -1>(v, sm, a.tw, j, SyncBlock{});
        }
#pragma unroll
        for (int k = 0; k < F::R; ++k) {
            v[k].x *= a.scale; v[k].y *= a.scale;
            f[j + F::TG * k] = v[k];
        }
        if (a.mode == 0) return;   // initial iterate: nothing to reduce
    }

    double tot[2];
    if (reduce_ticket<2>(acc, a.part + (size_t)b * a.nblk * 2, a.ctr + b, a.nblk, blockIdx.x, tot)) {
        if (threadIdx.x == 0) {
            if (fin) {
                if (tot[1] != 0.0 && st->diverged == 0) st->diverged = st->iters_run > 0 ? st->iters_run : 1;
                st->done = 1;
            } else {
                st->energy = tot[0];
                if (tot[1] != 0.0 || !isfinite(tot[0])) {
                    st->diverged = a.it;
                    st->iters_run = a.it;
                    st->stop = 1;
                    st->done = 1;
                }
            }
        }
    }
}

// -------------------------------------------------------------- column sweep
// Largest CTA a column kernel is launched with (see col_config in pm_capi.cu):
// 256 threads while a transform needs <= 64 threads, else 512.
template <int LG_L, int LG_R>
constexpr int col_max_threads() { return FftShape<LG_L, LG_R>::TG <= 64 ? 256 : 512; }

template <typename T, int LG_L, int LG_R>
__global__ void __launch_bounds__(col_max_threads<LG_L, LG_R>()) col_iter_kernel(ColArgs<T> a) {
    using F = FftShape<LG_L, LG_R>;
    extern __shared__ __align__(16) unsigned char smraw[];
    const int b = blockIdx.y;
    MaskState* st = a.st + b;
    if (st->done) return;
    const int C = blockDim.x / F::TG;
    const int c = threadIdx.x % C, j = threadIdx.x / C;
    const int col = blockIdx.x * C + c;
    const size_t N = (size_t)a.nx * a.ny;
    const size_t nx = a.nx;
    cx<T>* sm = reinterpret_cast<cx<T>*>(smraw) + c * (F::SM + kColPad);
    cx<T>* f = a.field + b * N + col;
    const T* m = a.m + b * a.m_stride + col;

    cx<T> v[F::R];
    if (a.mode == 0) {
#pragma unroll
        for (int k = 0; k < F::R; ++k) v[k] = mk<T>(m[(j + F::TG * k) * nx], T(0));
    } else {
#pragma unroll
        for (int k = 0; k < F::R; ++k) v[k] = f[(j + F::TG * k) * nx];
    }
    if (a.mode < 2) {
        // initial iterate u0 = F^-1(m e^{i0}), column half (src/solver.py:93-108)
        fft1d<T, LG_L, LG_R, +1>(v, sm, a.tw, j, SyncBlock{});
#pragma unroll
        for (int k = 0; k < F::R; ++k) {
            v[k].x *= a.scale; v[k].y *= a.scale;
            f[(j + F::TG * k) * nx] = v[k];
        }
        return;
    }
    fft1d<T, LG_L, LG_R, -1>(v, sm, a.tw, j, SyncBlock{});

    const bool metr = a.u_iter >= 1;
    const bool rec = metr && ((a.u_iter - 1) % a.ctl.record_every == 0);
    const T tol = T(a.tol_m[b]);
    const double s = rec ? a.energy_target[b] / st->energy : 0.0;
    double acc[3] = {0.0, 0.0, 0.0};   // gap^2, err_lit, err_dark
#pragma unroll
    for (int k = 0; k < F::R; ++k) {
        const T mm = m[(j + F::TG * k) * nx];
        cx<T> u = v[k];
        u.x *= a.scale; u.y *= a.scale;                    // u^ = F(u)
        const cx<T> vh = replace_mod(u, mm, tol);          // v^ = replace_m(u^)
        if (metr) {
            // G(u) = ||P_S u - P_M u|| = ||u^ - v^|| (Parseval; u is on S)
            const double dx = (double)(u.x - vh.x), dy = (double)(u.y - vh.y);
            acc[0] += dx * dx + dy * dy;
            if (rec) {
                // reconstructed intensity and physical error (src/metrics.py:74-112)
                const double inten = ((double)u.x * (double)u.x + (double)u.y * (double)u.y) * s;
                const double m2 = (double)mm * (double)mm;
                if (m2 > 0.0) {
                    const double dev = fabs(m2 - inten);
                    if (dev / m2 > a.ctl.t_lit)
                        acc[1] += a.ctl.t_dark * dev / (a.ctl.t_lit * m2) - a.ctl.t_dark;
                } else if (inten > a.ctl.t_dark) {
                    acc[2] += inten - a.ctl.t_dark;
                }
            }
        }
        v[k] = vh;
    }
    fft1d<T, LG_L, LG_R, +1>(v, sm, a.tw, j, SyncBlock{});
#pragma unroll
    for (int k = 0; k < F::R; ++k) {
        v[k].x *= a.scale; v[k].y *= a.scale;
        f[(j + F::TG * k) * nx] = v[k];
    }
    if (!metr) return;

    double tot[3];
    if (reduce_ticket<3>(acc, a.part + (size_t)b * a.nblk * 3, a.ctr + b, a.nblk, blockIdx.x, tot)) {
        if (threadIdx.x == 0) {
            // record / early-stop / abort logic of src/solver.py:173-199 for u_i
            const int i = a.u_iter;
            const double g = sqrt(tot[0]);
            double* h = a.hist + ((size_t)b * a.hist_stride + (i - 1)) * 4;
            int stop = 0;
            if (!isfinite(tot[0])) {
                st->diverged = i;
                stop = 1;
            }
            if (rec) {
                h[0] = g; h[1] = tot[1]; h[2] = tot[2]; h[3] = 1.0;
                st->n_records += 1;
            }
            if (a.ctl.early_tol >= 0.0) {
                if (st->have_prev && g > 0.0 && fabs(g - st->prev_gap) <= a.ctl.early_tol * g) stop = 1;
                st->prev_gap = g;
                st->have_prev = 1;
            }
            if (i >= a.ctl.max_iters) stop = 1;
            if (stop) {
                st->stop = 1;
                st->iters_run = i;
                if (st->diverged) st->done = 1;
            }
        }
    }
}

// ------------------------------------------------ standalone transform sweeps
// FftProvider.forward / inverse (src/transform.py:47-55): one axis per launch.
template <typename T, int LG_L, int LG_R>
__global__ void __launch_bounds__(256) row_fft_kernel(const cx<T>* in, cx<T>* out, const cx<T>* tw,
                                                      int nx, int ny, T scale, int dir) {
    using F = FftShape<LG_L, LG_R>;
    extern __shared__ __align__(16) unsigned char smraw[];
    const int G = blockDim.x / F::TG;
    const int g = threadIdx.x / F::TG, j = threadIdx.x % F::TG;
    const size_t o = (size_t)blockIdx.y * nx * ny + (size_t)(blockIdx.x * G + g) * nx;
    cx<T>* sm = reinterpret_cast<cx<T>*>(smraw) + g * F::SM;
    cx<T> v[F::R];
#pragma unroll
    for (int k = 0; k < F::R; ++k) v[k] = in[o + j + F::TG * k];
    if constexpr (F::TG <= 32) {
        if (dir < 0) fft1d<T, LG_L, LG_R, -1>(v, sm, tw, j, SyncWarp{});
        else fft1d<T, LG_L, LG_R, +1>(v, sm, tw, j, SyncWarp{});
    } else {
        if (dir < 0) fft1d<T, LG_L, LG_R, -1>(v, sm, tw, j, SyncBlock{});
        else fft1d<T, LG_L, LG_R, +1>(v, sm, tw, j, SyncBlock{});
    }
#pragma unroll
    for (int k = 0; k < F::R; ++k) {
        v[k].x *= scale; v[k].y *= scale;
        out[o + j + F::TG * k] = v[k];
    }
}

template <typename T, int LG_L, int LG_R>
__global__ void __launch_bounds__(col_max_threads<LG_L, LG_R>()) col_fft_kernel(const cx<T>* in, cx<T>* out, const cx<T>* tw,
                                                       int nx, int ny, T scale, int dir) {
    using F = FftShape<LG_L, LG_R>;
    extern __shared__ __align__(16) unsigned char smraw[];
    const int C = blockDim.x / F::TG;
    const int c = threadIdx.x % C, j = threadIdx.x / C;
    const size_t o = (size_t)blockIdx.y * nx * ny + (size_t)(blockIdx.x * C + c);
    cx<T>* sm = reinterpret_cast<cx<T>*>(smraw) + c * (F::SM + kColPad);
    cx<T> v[F::R];
#pragma unroll
    for (int k = 0; k < F::R; ++k) v[k] = in[o + (size_t)(j + F::TG * k) * nx];
    if (dir < 0) fft1d<T, LG_L, LG_R, -1>(v, sm, tw, j, SyncBlock{});
    else fft1d<T, LG_L, LG_R, +1>(v, sm, tw, j, SyncBlock{});
#pragma unroll
    for (int k = 0; k < F::R; ++k) {
        v[k].x *= scale; v[k].y *= scale;
        out[o + (size_t)(j + F::TG * k) * nx] = v[k];
    }
}

}  // namespace pm
