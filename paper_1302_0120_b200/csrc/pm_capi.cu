// C ABI of libphasemask_b200 (declared in include/phasemask_b200.h):
// plans, launch configuration, the solve orchestration (a CUDA graph of
// 2K+4 sweep launches per solve, no host round trip per iteration), the
// stand-alone transform / projection / reduction entry points and the
// measurement helpers used by bench.py.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>   // header-only NVTX ranges (ncu --nvtx / nsys)
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <atomic>
#include <chrono>
#include <cstddef>
#include <set>
#include <string>
#include <vector>

#include "phasemask_b200.h"
#include "pm_generic.cuh"
#include "pm_rng.cuh"
#include "pm_kernels.cuh"
#include "pm_table.h"

using namespace pm;

// ------------------------------------------------------------------ errors
namespace {
thread_local std::string g_err;

int set_err(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

int cuda_err(cudaError_t e, const char* what) {
    cudaGetLastError();  // clear sticky-free errors
    const int code = (e == cudaErrorMemoryAllocation) ? PM_ERR_NOMEM : PM_ERR_CUDA;
    return set_err(code, std::string(what) + ": " + cudaGetErrorString(e));
}
}  // namespace

#define CK(call)                                                  \
    do {                                                          \
        cudaError_t e_ = (call);                                  \
        if (e_ != cudaSuccess) return cuda_err(e_, #call);        \
    } while (0)
#define CKR(call)                                                 \
    do {                                                          \
        int r_ = (call);                                          \
        if (r_ != PM_OK) return r_;                               \
    } while (0)

// ------------------------------------------------------- elementwise kernels
namespace pm {

// src/projections.py:46-66 as a stand-alone per-pixel kernel, through the
// solve's own register-array projection (project_regs: fast pass, exact
// re-decision inside the band) four pixels per thread, so the projection
// KATs exercise the hot path's decision code.
template <typename T>
__global__ void replace_kernel(const cx<T>* in, const T* target, long long tstride, T tol_,
                               cx<T>* out, long long n) {
    const long long b = blockIdx.y;
    const ZThr<T> z = zthr<T>(tol_);
    const cx<T>* ib = in + b * n;
    const T* tb = target + b * tstride;
    cx<T>* ob = out + b * n;
    auto keep = [](int, cx<T>, cx<T> o) { return o; };
    for (long long i = (blockIdx.x * (long long)blockDim.x + threadIdx.x) * 4; i < n;
         i += (long long)gridDim.x * blockDim.x * 4) {
        if (i + 4 <= n) {
            cx<T> v[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) v[k] = ib[i + k];
            auto t_of = [&](int k) -> T { return tb[i + k]; };
            project_regs<false>(v, z, t_of, keep);
#pragma unroll
            for (int k = 0; k < 4; ++k) ob[i + k] = v[k];
        } else {
            for (long long j = i; j < n; ++j) ob[j] = replace_mod(ib[j], tb[j], z);
        }
    }
}

// Fixed partition: block i reduces [i*chunk, (i+1)*chunk) with a fixed
// per-thread stride and a fixed tree; partials combined in index order.
__device__ __forceinline__ double block_sum(double x) {
    __shared__ double ws[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0) ws[warp] = x;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0)
        for (int w = 0; w < (int)((blockDim.x + 31) >> 5); ++w) s += ws[w];
    return s;
}

__device__ __forceinline__ double block_max(double x) {
    __shared__ double wm[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
    if (lane == 0) wm[warp] = x;
    __syncthreads();
    double m = 0.0;
    if (threadIdx.x == 0)
        for (int w = 0; w < (int)((blockDim.x + 31) >> 5); ++w) m = fmax(m, wm[w]);
    return m;
}

template <typename TIn>
__device__ __forceinline__ double sq_mag(const TIn* d, long long i);
template <> __device__ __forceinline__ double sq_mag<float>(const float* d, long long i) {
    const double a = (double)fabsf(d[i]);
    return a * a;
}
template <> __device__ __forceinline__ double sq_mag<double>(const double* d, long long i) {
    const double a = fabs(d[i]);
    return a * a;
}
template <> __device__ __forceinline__ double sq_mag<float2>(const float2* d, long long i) {
    const float2 u = d[i];
    const double a = (double)np_cabs(u);                    // np.abs in field precision
    return a * a;
}
template <> __device__ __forceinline__ double sq_mag<double2>(const double2* d, long long i) {
    const double a = np_cabs(d[i]);
    return a * a;
}

template <typename TIn>
__global__ void norm_partial_kernel(const TIn* d, long long n, long long chunk, double* part) {
    const long long lo = blockIdx.x * chunk, hi = min(n, lo + chunk);
    double acc = 0.0;
    for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) acc += sq_mag<TIn>(d, i);
    const double s = block_sum(acc);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void sum_partial_kernel(const double* d, long long n, long long chunk, double* part) {
    const long long lo = blockIdx.x * chunk, hi = min(n, lo + chunk);
    double acc = 0.0;
    for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) acc += d[i];
    const double s = block_sum(acc);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// |P_S u - w|^2 partials for metrics.gap (src/metrics.py:67-71).
template <typename T>
__global__ void gap_partial_kernel(const cx<T>* u, const cx<T>* pm_u, const T* p, T tol_,
                                   long long n, long long chunk, double* part) {
    const long long lo = blockIdx.x * chunk, hi = min(n, lo + chunk);
    const ZThr<T> tol = zthr<T>(tol_);
    double acc = 0.0;
    for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        const cx<T> ps = replace_mod(u[i], p[i], tol);
        const double a = (double)np_cabs(mk<T>(ps.x - pm_u[i].x, ps.y - pm_u[i].y));   // np.abs in field precision
        acc += a * a;
    }
    const double s = block_sum(acc);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void final_sum_kernel(const double* part, int nb, double* out, int take_sqrt) {
    double x = 0.0;
    for (int i = threadIdx.x; i < nb; i += 32) x += part[i];
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (threadIdx.x == 0) *out = take_sqrt ? sqrt(x) : x;
}

template <typename T>
__global__ void phases_kernel(const cx<T>* u, long long n, T tol, double* out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const cx<T> v = u[i];
        double th = phase_of((double)v.x, (double)v.y);
        if (tol > T(0) && np_cabs(v) < tol) th = 0.0;        // np.abs(u) < zero_tol
        out[i] = th;
    }
}

// The reference's correctness oracle naive_dft (src/transform.py:56-81) on
// the device: out = W_rows X W_cols^T with W[k][j] = exp(sign 2 pi i k j / n)
// / sqrt(n), in fp64. One thread per output pixel, the double sum in a fixed
// order; the phase of each term is reduced exactly (k j mod n) before sincospi.
__global__ void naive_dft_kernel(const double2* x, int nx, int ny, double sign, double2* out) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= nx * ny) return;
    const int r = idx / nx, c = idx % nx;
    double re = 0.0, im = 0.0;
    for (int a = 0; a < ny; ++a) {
        const double fa = (double)((long long)r * a % ny) / ny;
        double ta = 0.0, tb = 0.0;                        // (W_rows X)[r][b] W_cols[c][b] summed over b
        for (int b = 0; b < nx; ++b) {
            const double f = fa + (double)((long long)c * b % nx) / nx;
            double sn, cs;
            sincospi(2.0 * sign * f, &sn, &cs);
            const double2 v = x[(size_t)a * nx + b];
            ta += v.x * cs - v.y * sn;
            tb += v.x * sn + v.y * cs;
        }
        re += ta;
        im += tb;
    }
    const double s = 1.0 / (sqrt((double)nx) * sqrt((double)ny));
    out[idx] = make_double2(re * s, im * s);
}

// Reconstructed intensity |F u|^2 (src/metrics.py:74-87): per mask (blockIdx.y)
// fixed-partition partial sums and maxima of (double)|F u|^2, |.| taken in
// the field precision and squared in fp64 as the reference does.
template <typename T>
__device__ __forceinline__ double recon_i(cx<T> f) {
    const double a = (double)sqrt(f.x * f.x + f.y * f.y);
    return a * a;
}
template <typename T>
__global__ void recon_partial_kernel(const cx<T>* F, long long n, long long chunk, double* part, int nb) {
    const cx<T>* f = F + blockIdx.y * n;
    const long long lo = blockIdx.x * chunk, hi = min(n, lo + chunk);
    double acc = 0.0, mx = 0.0;
    for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        const double v = recon_i<T>(f[i]);
        acc += v;
        mx = fmax(mx, v);
    }
    const double s = block_sum(acc);
    __syncthreads();
    const double m = block_max(mx);
    if (threadIdx.x == 0) {
        part[(size_t)blockIdx.y * 2 * nb + blockIdx.x] = s;
        part[(size_t)blockIdx.y * 2 * nb + nb + blockIdx.x] = m;
    }
}
// scale = E / sum (1 without E) and the peak of the scaled intensity, per mask
// (max commutes with the monotone rounded scaling: max(I s) = max(I) s).
__global__ void recon_final_kernel(const double* part, int nb, const double* energy, double* out) {
    const int b = blockIdx.x;
    const double* q = part + (size_t)b * 2 * nb;
    double x = 0.0, m = 0.0;
    for (int i = threadIdx.x; i < nb; i += 32) {
        x += q[i];
        m = fmax(m, q[nb + i]);
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        x += __shfl_xor_sync(0xffffffffu, x, o);
        m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    }
    if (threadIdx.x == 0) {
        const double sc = energy ? (x == 0.0 ? 0.0 : energy[b] / x) : 1.0;
        out[2 * b] = sc;
        out[2 * b + 1] = m * sc;
    }
}
// The scaled intensity in DFT order and its log-scale 8-bit image in
// centred order (to_centered_order + service._log_scale_u8,
// src/service.py:91-95): v = I / peak (0 if peak == 0),
// round(255 (log10(max(v, floor)) - lf) / -lf), lf = log10(floor).
template <typename T>
__global__ void recon_image_kernel(const cx<T>* F, int nx, int ny, const double* sp, double floor_, double lf,
                                   double* inten, uint8_t* img) {
    const long long n = (long long)nx * ny;
    const int b = blockIdx.y;
    const double sc = sp[2 * b], peak = sp[2 * b + 1];
    const cx<T>* f = F + b * n;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const double v = recon_i<T>(f[i]) * sc;
        if (inten) inten[b * n + i] = v;
        if (img) {
            const double d = peak > 0.0 ? v / peak : 0.0;
            const double l = (log10(fmax(d, floor_)) - lf) / (-lf);
            const int y = (int)(i / nx), x = (int)(i - (long long)y * nx);
            const int yc = (y + ny / 2) % ny, xc = (x + nx / 2) % nx;     // fftshift
            img[b * n + (long long)yc * nx + xc] = (uint8_t)rint(l * 255.0);
        }
    }
}

// out[b][x][y] = in[b][y][x] for [batch][ny][nx] grids (32 x 32 tiles).
template <typename T>
__global__ void transpose_kernel(const T* __restrict__ in, T* __restrict__ out, int nx, int ny) {
    __shared__ T tile[32][33];
    const size_t off = (size_t)blockIdx.z * nx * ny;
    const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int y = y0 + r, x = x0 + threadIdx.x;
        if (y < ny && x < nx) tile[r][threadIdx.x] = in[off + (size_t)y * nx + x];
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int x = x0 + r, y = y0 + threadIdx.x;
        if (x < nx && y < ny) out[off + (size_t)x * ny + y] = tile[threadIdx.x][r];
    }
}

// L2 roof: `passes` sweeps over an L2-resident buffer inside ONE launch (mode
// 0: reads only, 1: copy a -> b), L1 bypassed, 4 independent 16-byte
// accesses in flight per thread.
__global__ void __launch_bounds__(512) l2_kernel(const float4* __restrict__ a, float4* __restrict__ b, long long n,
                                                  int passes, int mode, float* sink) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    float acc = 0.f;
    for (int pass = 0; pass < passes; ++pass) {
        for (long long i = t; i < n; i += 4 * stride) {
            float4 v[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) v[k] = i + k * stride < n ? __ldcg(a + i + k * stride) : make_float4(0, 0, 0, 0);
            if (mode) {
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (i + k * stride < n) __stcg(b + i + k * stride, v[k]);
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k) acc += v[k].x + v[k].y + v[k].z + v[k].w;
            }
        }
    }
    if (acc == 1.2345e-30f) *sink = acc;
}

__global__ void copy_kernel(const float4* __restrict__ a, float4* __restrict__ b, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        b[i] = a[i];
}

// Decision tolerances of one mask (host and device): the reference's zero_tol
// as the precision's float (src/projections.py:49-53 compares float32 mag with
// the Python-float tolerance in float32, NEP 50). Every projection decides on
// normalised values (pm_kernels.cuh, scaling convention), so the tolerances
// are used as they are: thrp / thrx for P_S, thrm for the Fourier replace.
__host__ __device__ inline void zero_thresholds(double tp, double tm, bool single, double* thrp, double* thrm,
                                                double* thrx) {
    const double qp = single ? (double)(float)tp : tp;
    *thrp = qp;
    *thrm = single ? (double)(float)tm : tm;
    *thrx = qp;
}

// The per-solve prologue in ONE launch (it was eight stream operations: two
// memsets, the tolerance maxima and their combine, sum p^2, sum m^2, the
// escale combine, S p): block (x, b) covers [x*chunk, (x+1)*chunk) of mask b,
// a fixed partition of the grid (independent of batch), and leaves
// {max p, max m, sum p^2, sum m^2} of its chunk in part[b][x]; with a shared
// p only mask 0's blocks read it. The last block to finish (ticket) clears
// the mask states and combines the partials in index order: the zero
// tolerances 1024 eps max(.) and their thresholds (src/projections.py:41-43,
// src/grid.py:21,33-34) when they are reduced on the device (an identically
// zero p or all-dark m marks the mask done, reported as the reference's
// ValueError), the energy sum m^2 when not given, and the reconstructed-
// intensity scale escale = sum m^2 / sum p^2 (sum |u|^2 = sum p^2 on S).
// S p is the P_S target of the GS row sweeps (they write S u). Every block
// helps clear the histories.
struct ProArgs {
    const void* p;
    const void* m;
    void* ps;                 // S p (GS sweeps), or null
    double S;
    long long n, chunk;
    int nb, batch, per_mask, single;
    int do_tol, do_msum;
    double* part;             // [batch][nb][4]
    MaskState* st;
    double* hist;
    long long hist_n;         // doubles to clear
    double *tolp, *thrp, *thrm, *thrx, *energy, *escale;
    unsigned* ticket;
};

template <typename T>
__global__ void __launch_bounds__(256) prologue_kernel(ProArgs a) {
    const int b = blockIdx.y, x = blockIdx.x;
    const bool do_p = a.per_mask || b == 0;
    const T* pb = static_cast<const T*>(a.p) + (a.per_mask ? (long long)b * a.n : 0);
    const T* mb = static_cast<const T*>(a.m) + (long long)b * a.n;
    T* psb = a.ps ? static_cast<T*>(a.ps) + (a.per_mask ? (long long)b * a.n : 0) : nullptr;
    const long long lo = x * a.chunk, hi = min(a.n, lo + a.chunk);
    const bool do_m = a.do_tol || a.do_msum;
    T pmx = T(0), mmx = T(0);
    double p2 = 0.0, m2 = 0.0;
    // eight loads in flight per thread (amplitudes are >= 0: the zero padding
    // past the chunk changes neither the maxima nor the sums)
    constexpr int U = 8;
    for (long long base = lo + threadIdx.x; base < hi; base += U * blockDim.x) {
        T v[U], w[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const long long i = base + (long long)k * blockDim.x;
            v[k] = (do_p && i < hi) ? pb[i] : T(0);
            w[k] = (do_m && i < hi) ? mb[i] : T(0);
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const long long i = base + (long long)k * blockDim.x;
            pmx = max(pmx, v[k]);
            p2 += (double)v[k] * (double)v[k];
            mmx = max(mmx, w[k]);
            m2 += (double)w[k] * (double)w[k];
            if (psb && do_p && i < hi) psb[i] = v[k] * T(a.S);
        }
    }
    // fixed-order block reduction of the four values
    __shared__ double red[4][8];
    __shared__ int last;
    double v4[4] = {(double)pmx, (double)mmx, p2, m2};
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        v4[0] = fmax(v4[0], __shfl_xor_sync(0xffffffffu, v4[0], o));
        v4[1] = fmax(v4[1], __shfl_xor_sync(0xffffffffu, v4[1], o));
        v4[2] += __shfl_xor_sync(0xffffffffu, v4[2], o);
        v4[3] += __shfl_xor_sync(0xffffffffu, v4[3], o);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0)
        for (int k = 0; k < 4; ++k) red[k][warp] = v4[k];
    // the histories: cleared by every block, grid-stride
    const long long nblk = (long long)gridDim.x * gridDim.y, bid = (long long)b * gridDim.x + x;
    for (long long i = bid * blockDim.x + threadIdx.x; i < a.hist_n; i += nblk * blockDim.x) a.hist[i] = 0.0;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t[4] = {red[0][0], red[1][0], red[2][0], red[3][0]};
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
            t[0] = fmax(t[0], red[0][w]);
            t[1] = fmax(t[1], red[1][w]);
            t[2] += red[2][w];
            t[3] += red[3][w];
        }
        double* q = a.part + ((size_t)b * a.nb + x) * 4;
        for (int k = 0; k < 4; ++k) q[k] = t[k];
        __threadfence();
        last = atomicAdd(a.ticket, 1u) == (unsigned)(nblk - 1);
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    // mask states cleared before the zero flags are set
    unsigned* sw = reinterpret_cast<unsigned*>(a.st);
    const int words = a.batch * (int)(sizeof(MaskState) / sizeof(unsigned));
    for (int i = threadIdx.x; i < words; i += blockDim.x) sw[i] = 0u;
    __syncthreads();
    // one warp per mask: each lane folds the partials lane, lane + 32, ... in
    // order, then a fixed xor tree (deterministic; one round of loads in flight
    // instead of nb dependent ones)
    for (int k = warp; k < a.batch; k += (int)(blockDim.x >> 5)) {
        const double* qp = a.part + (size_t)(a.per_mask ? k : 0) * a.nb * 4;
        const double* qm = a.part + (size_t)k * a.nb * 4;
        double pmax = 0.0, mmax = 0.0, sp = 0.0, sm = 0.0;
#pragma unroll 5
        for (int i = lane; i < a.nb; i += 32) {
            pmax = fmax(pmax, __ldcg(qp + 4 * i + 0));
            mmax = fmax(mmax, __ldcg(qm + 4 * i + 1));
            sp += __ldcg(qp + 4 * i + 2);
            sm += __ldcg(qm + 4 * i + 3);
        }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
            pmax = fmax(pmax, __shfl_xor_sync(0xffffffffu, pmax, o));
            mmax = fmax(mmax, __shfl_xor_sync(0xffffffffu, mmax, o));
            sp += __shfl_xor_sync(0xffffffffu, sp, o);
            sm += __shfl_xor_sync(0xffffffffu, sm, o);
        }
        if (lane != 0) continue;
        if (a.do_tol) {
            const double eps = a.single ? 1.1920928955078125e-07 : 2.220446049250313e-16;
            const double tp = 1024.0 * eps * pmax, tm = 1024.0 * eps * mmax;
            a.tolp[k] = tp;
            zero_thresholds(tp, tm, a.single, a.thrp + k, a.thrm + k, a.thrx + k);
            const int z = (pmax == 0.0 ? 1 : 0) | (mmax == 0.0 ? 2 : 0);
            if (z) {
                a.st[k].zero = z;
                a.st[k].done = 1;
            }
        }
        if (a.do_msum) a.energy[k] = sm;
        a.escale[k] = a.energy[k] / sp;
    }
    if (threadIdx.x == 0) *a.ticket = 0u;        // ready for the next launch (graph replays too)
}

// Host abort (should_abort -> True): the current iterate becomes the last.
__global__ void force_stop_kernel(MaskState* st, int batch, int it) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b < batch && !st[b].stop && !st[b].done) {
        st[b].stop = 1;
        st[b].iters_run = it;
        st[b].aborted = 1;
    }
}

}  // namespace pm

// ---------------------------------------------------------------- plan
namespace {

int lg2_exact(int n) {
    if (n < 1 || (n & (n - 1))) return -1;
    int l = 0;
    while ((1 << l) < n) ++l;
    return l;
}

const KernelSet& kset(int prec, int lg) { return prec == PM_SINGLE ? kernels_f32(lg) : kernels_f64(lg); }

// Twiddles of the Stockham passes, [pass][r-1][k] (see FftShape), as
// (cos, sin) of the angle DIR * 2 pi r k / (Ns Rs) in long double.
std::vector<std::pair<double, double>> twiddle_angles(int lg, int lgR_max, int dir) {
    const int lgR = std::min(lg, lgR_max);
    const int NP = lgR == 0 ? 0 : (lg + lgR - 1) / lgR;
    std::vector<std::pair<double, double>> out;
    const long double pi = 3.141592653589793238462643383279502884L;
    for (int s = 1; s < NP; ++s) {
        const int lgRs = (s < NP - 1) ? lgR : lg - (NP - 1) * lgR;
        const long long Rs = 1LL << lgRs, Ns = 1LL << (s * lgR), M = Ns * Rs;
        for (long long r = 1; r < Rs; ++r)
            for (long long k = 0; k < Ns; ++k) {
                const long double ang = 2.0L * pi * (long double)((r * k) % M) / (long double)M;
                out.emplace_back((double)cosl(ang), (double)(dir * sinl(ang)));
            }
    }
    return out;
}

// Device twiddle tables for one axis: fp32 forward/inverse float4 entries
// (c, s, -s, c) so a twiddle multiply is FMUL2 + FFMA2; fp64 one (c, s) table.
int upload_twiddles(int prec, int lg, int lgR, int TW, void** fwd, void** inv) {
    *fwd = *inv = nullptr;
    if (prec == PM_SINGLE) {
        for (int d = 0; d < 2; ++d) {
            const int dir = d == 0 ? -1 : +1;
            std::vector<float4> t;
            for (auto& w : twiddle_angles(lg, lgR, dir))
                t.push_back(make_float4((float)w.first, (float)w.second, -(float)w.second, (float)w.first));
            if ((int)t.size() != TW) return set_err(PM_ERR_CUDA, "twiddle table size mismatch");
            void** dst = d == 0 ? fwd : inv;
            CK(cudaMalloc(dst, std::max<size_t>(1, t.size()) * sizeof(float4)));
            if (!t.empty()) CK(cudaMemcpy(*dst, t.data(), t.size() * sizeof(float4), cudaMemcpyHostToDevice));
        }
    } else {
        std::vector<double2> t;
        for (auto& w : twiddle_angles(lg, lgR, -1)) t.push_back(make_double2(w.first, w.second));
        if ((int)t.size() != TW) return set_err(PM_ERR_CUDA, "twiddle table size mismatch");
        CK(cudaMalloc(fwd, std::max<size_t>(1, t.size()) * sizeof(double2)));
        if (!t.empty()) CK(cudaMemcpy(*fwd, t.data(), t.size() * sizeof(double2), cudaMemcpyHostToDevice));
        *inv = *fwd;
    }
    return PM_OK;
}

std::map<const void*, size_t>& smem_configured() {
    static std::map<const void*, size_t> s;
    return s;
}
std::mutex g_attr_mu;

// Opt a kernel into `bytes` of dynamic shared memory (> 48 KB needs it).
cudaError_t allow_smem(const void* fn, size_t bytes) {
    if (bytes <= 48 * 1024) return cudaSuccess;
    std::lock_guard<std::mutex> lk(g_attr_mu);
    auto it = smem_configured().find(fn);
    if (it != smem_configured().end() && it->second >= bytes) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) smem_configured()[fn] = bytes;
    return e;
}

struct RowCfg { int G, threads, nblk; size_t smem; };
struct ColCfg { int C, threads, nblk; size_t smem; };

}  // namespace

struct pm_plan {
    int device = 0, nx = 0, ny = 0, prec = 0, lgx = 0, lgy = 0;
    size_t N = 0, csz = 0, rsz = 0;   // pixels, complex and real element sizes
    int cap = 0;                      // batch capacity
    int hist_cap = 0;                 // max_iters capacity of the history buffer
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    void* tw_row = nullptr;           // forward twiddles, row axis
    void* tw_row_i = nullptr;         // inverse (fp32; == tw_row for fp64)
    void* tw_col = nullptr;
    void* tw_col_i = nullptr;
    void* field = nullptr;            // cap * N complex
    void* tmp = nullptr;              // cap * N complex (scratch)
    void* pbuf = nullptr;             // cap * N real
    void* mbuf = nullptr;             // cap * N real
    double* phases = nullptr;         // cap * N
    uint8_t* levels = nullptr;        // cap * N
    void* ustar = nullptr;            // cap * N complex
    void* vstar = nullptr;
    void* field2 = nullptr;           // RAAR: cap * N complex, second field buffer (w')
    void* mT = nullptr;               // persistent column phase: m transposed per mask
    size_t mT_bytes = 0;
    void* ps = nullptr;               // GS sessions: S p, the row sweeps' P_S target
    size_t ps_bytes = 0;
    void* xbuf = nullptr;             // RAAR: cap * N complex, the iterate x
    double* rpart = nullptr;          // RAAR: cap * ny * wpr * 2 row partials
    double* thrx = nullptr;           // cap P_S thresholds on true-scale values (RAAR, mixed-radix path)
    int raar_cap = 0;
    // mixed-radix path (a side that is not a power of two; pm_generic.cuh)
    bool generic = false;
    GenPlan gx{}, gy{};               // row (n_x) and column (n_y) transforms
    void* gtwx = nullptr;             // exp(-2 pi i k / n_x), k < n_x, plan precision
    void* gtwy = nullptr;
    int gtc_r = 1, gtc_c = 1;         // transforms per CTA
    int gnt_r = 256, gnt_c = 256;     // threads per CTA of the row / column kernels
    size_t gsm_r = 0, gsm_c = 0;      // their shared memory
    // TMA maps of the persistent column phase (pm_kernels.cuh col_phase)
    CUtensorMap tm_field{}, tm_field2{}, tm_m{};
    bool tm_field_ok = false, tm_field2_ok = false, tm_m_ok = false;
    MaskState* st = nullptr;          // cap
    double* hist = nullptr;           // cap * hist_cap * 4
    double* part = nullptr;           // column partial sums, 2 (parity) * cap * nb * 3
    unsigned* ctr = nullptr;          // 2 * cap counters
    double* tolp = nullptr;           // cap: reference zero_tol of p
    double* thrp = nullptr;           // cap: decision thresholds (fp32: on |u|^2)
    double* thrm = nullptr;
    double* thrms = nullptr;          // cap: column thresholds on the unscaled transform
    double* escale = nullptr;         // cap: sum m^2 / sum p^2
    double* energy = nullptr;         // cap: sum m^2 (host-provided)
    double* psum = nullptr;           // (unused since the fused prologue)
    double* red = nullptr;            // reduction scratch
    int red_cap = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    long long launches = 0;
    GridBar* bar = nullptr;           // grid barrier of the persistent kernel
    unsigned long long* stamps = nullptr;  // optional phase timestamps (pm_debug_phase_stamps)
    // streamed decisions of a callback solve (pm_solve_async): host-mapped
    RingSlot* ring_h = nullptr;       // [ring_cap] host view
    RingSlot* ring_d = nullptr;       // device view
    int* hostw_h = nullptr;           // {acknowledged iteration, abort request} host view
    int* hostw_d = nullptr;
    int ring_cap = 0;
    // page-locked staging of the small per-solve transfers (energies, thresholds,
    // mask states, histories): pageable cudaMemcpyAsync would synchronise the stream
    unsigned char* hst = nullptr;
    size_t hst_bytes = 0;
    int solve_grid = 0;               // CTAs of the persistent kernel (0: not available)
    int solve_grid_tma = 0;           // CTAs of its TMA variant (0: not available)
    int path = 0;                     // 0 auto, 1 persistent, 2 sweep graph
    RowCfg rc{};
    ColCfg cc{};
    std::map<std::string, cudaGraphExec_t> graphs;
    std::mutex mu;

    // current solve session
    struct Session {
        bool active = false;
        bool stepping = false;        // pm_solve_begin/step/finish (vs one enqueued solve)
        int batch = 0, it = 0;
        pm_params prm{};
        const void* p = nullptr;
        const void* m = nullptr;
        const void* mT = nullptr;     // transposed m of this session (null: column tasks stage from m)
        const void* ps = nullptr;     // S p (GS; the p grids of the session scaled on the device)
        long long p_stride = 0;
        void* phases = nullptr;
        void* levels = nullptr;
        void* ustar = nullptr;
        void* vstar = nullptr;
        bool energy_on_device = false;
        bool tol_on_device = false;
        bool ring = false;            // decisions streamed to ring_h (pm_solve_async)
        bool lockstep = false;        // and each one waits for the host's verdict
    } s;
};

namespace {

// NVTX range of one entry point (scope-bound).
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangPop_(); }
    static void nvtxRangPop_() { nvtxRangePop(); }
};

// PM_TRACE=1: host wall-clock stamps of the solve's stages on stderr (diagnostics).
inline void trace(const char* what) {
    static const bool on = getenv("PM_TRACE") != nullptr;
    if (!on) return;
    static thread_local auto t0 = std::chrono::steady_clock::now();
    const auto t = std::chrono::steady_clock::now();
    fprintf(stderr, "[pm] %8.1f us  %s\n", std::chrono::duration<double, std::micro>(t - t0).count(), what);
    t0 = t;
}

// Run control of the session: the reference's loop parameters plus the
// record ring of a callback solve (pm_solve_async).
SolveCtl make_ctl(const pm_plan* pl) {
    const pm_params& prm = pl->s.prm;
    SolveCtl c;
    c.max_iters = prm.max_iters;
    c.record_every = prm.record_every;
    c.early_tol = prm.early_stop_tol;
    c.t_lit = prm.t_lit;
    c.t_dark = prm.t_dark;
    c.ring = pl->s.ring ? pl->ring_d : nullptr;
    c.host = pl->s.ring ? (volatile int*)pl->hostw_d : nullptr;
    c.lockstep = (pl->s.ring && pl->s.lockstep) ? 1 : 0;
    c.decide_all = pl->s.stepping ? 1 : 0;
    return c;
}

// The plan's page-locked staging area, at least `bytes` (grows; the stream is
// idle when it is replaced: callers stage only between solves).
int host_stage(pm_plan* pl, size_t bytes, unsigned char** out) {
    if (pl->hst_bytes < bytes) {
        CK(cudaStreamSynchronize(pl->stream));
        if (pl->hst) cudaFreeHost(pl->hst);
        pl->hst = nullptr;
        pl->hst_bytes = 0;
        const size_t nb = std::max<size_t>(bytes, 64 << 10);
        CK(cudaHostAlloc((void**)&pl->hst, nb, cudaHostAllocDefault));
        pl->hst_bytes = nb;
    }
    *out = pl->hst;
    return PM_OK;
}

RowCfg row_config(const pm_plan* pl) {
    const AxisShape& k = kset(pl->prec, pl->lgx).row;
    RowCfg c;
    c.G = std::max(1, 128 / k.TG);
    c.G = std::min(c.G, pl->ny);
    c.threads = c.G * k.TG;
    c.nblk = pl->ny / c.G;
    c.smem = (size_t)c.G * k.SM * pl->csz;
    return c;
}

ColCfg col_config(const pm_plan* pl) {
    const AxisShape& k = kset(pl->prec, pl->lgy).col;
    ColCfg c;
    const int maxt = col_max_threads_for(k.lgR, k.TG);
    c.C = std::max(1, maxt / k.TG);
    c.C = std::min(c.C, pl->nx);
    c.threads = c.C * k.TG;
    c.nblk = pl->nx / c.C;
    const int pad = std::max(1, (int)(128 / (pl->csz * c.C)));
    c.smem = k.SM ? (size_t)c.C * (k.SM + pad) * pl->csz : 0;
    return c;
}

void free_buffers(pm_plan* pl) {
    void* bufs[] = {pl->field, pl->tmp, pl->pbuf, pl->mbuf, pl->phases, pl->levels, pl->ustar,
                    pl->vstar, pl->st, pl->hist, pl->part, pl->ctr, pl->escale, pl->energy, pl->psum};
    for (void* b : bufs)
        if (b) cudaFree(b);
    void* rbufs[] = {pl->field2, pl->xbuf, pl->rpart, pl->mT, pl->ps};
    for (void* b : rbufs)
        if (b) cudaFree(b);
    pl->field2 = pl->xbuf = pl->mT = pl->ps = nullptr;
    pl->mT_bytes = pl->ps_bytes = 0;
    pl->rpart = pl->thrx = nullptr;
    pl->raar_cap = 0;
    pl->field = pl->tmp = pl->pbuf = pl->mbuf = pl->ustar = pl->vstar = nullptr;
    pl->phases = nullptr;
    pl->levels = nullptr;
    pl->st = nullptr;
    pl->hist = pl->part = pl->tolp = pl->thrp = pl->thrm = pl->thrms = pl->escale = pl->energy = pl->psum = nullptr;
    pl->ctr = nullptr;
    pl->cap = 0;
    pl->hist_cap = 0;
}

void drop_graphs(pm_plan* pl) {
    for (auto& kv : pl->graphs) cudaGraphExecDestroy(kv.second);
    pl->graphs.clear();
}

// ------------------------------------------------------------ TMA maps
PFN_cuTensorMapEncodeTiled_v12000 tma_encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = []() -> PFN_cuTensorMapEncodeTiled_v12000 {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        return (PFN_cuTensorMapEncodeTiled_v12000)f;
    }();
    return fn;
}

// Columns per task of the persistent kernel (its CTA over the column transform).
int solve_cols(const pm_plan* pl) {
    const KernelSet& k = kset(pl->prec, pl->lgy);
    return std::max(1, k.solve_threads / std::max(1, k.col.TG));
}

// [depth][n_y][width] elements of `esize` bytes viewed as 256-row blocks, boxes [n_y/256][256][box_w].
bool tma_encode(CUtensorMap* map, void* base, int single, long long width, int n_y, int depth, int box_w) {
    auto fn = tma_encode_fn();
    if (!fn || !base || ((uintptr_t)base & 15)) return false;
    const size_t esz = single ? 4 : 8;
    // rows in blocks of 256: [mask * n_y/256 + block][row][width], so one box
    // {box_w, 256, n_y/256} is a task's whole [n_y][box_w] tile (one copy
    // instruction per tile instead of n_y/256)
    if (n_y % 256 != 0 || n_y / 256 > 256) return false;
    cuuint64_t dims[3] = {(cuuint64_t)width, 256, (cuuint64_t)(n_y / 256) * std::max(depth, 1)};
    cuuint64_t strides[2] = {(cuuint64_t)(width * esz), (cuuint64_t)(width * esz * 256)};
    cuuint32_t box[3] = {(cuuint32_t)box_w, 256, (cuuint32_t)(n_y / 256)};
    cuuint32_t estr[3] = {1, 1, 1};
    if ((box_w * esz) % 16 != 0 || box_w > 256 || strides[0] % 16 != 0) return false;
    CUresult r = fn(map, single ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims,
                    strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// m box width: the columns of a task, at least 16 bytes.
int tma_m_box(const pm_plan* pl) { return std::max(solve_cols(pl), (int)(16 / pl->rsz)); }

int ensure_capacity(pm_plan* pl, int batch, int max_iters) {
    if (batch <= pl->cap && max_iters <= pl->hist_cap) return PM_OK;
    const int cap = std::max(batch, pl->cap);
    const int hcap = std::max(max_iters, std::max(pl->hist_cap, 1));
    CK(cudaStreamSynchronize(pl->stream));
    drop_graphs(pl);
    free_buffers(pl);
    const size_t N = pl->N;
    const int nb = std::max(std::max(pl->cc.nblk, pl->nx), 148);   // >= tasks / blocks per mask of any path
    CK(cudaMalloc(&pl->field, cap * N * pl->csz));
    CK(cudaMalloc(&pl->tmp, cap * N * pl->csz));
    CK(cudaMalloc(&pl->pbuf, cap * N * pl->rsz));
    CK(cudaMalloc(&pl->mbuf, cap * N * pl->rsz));
    CK(cudaMalloc((void**)&pl->st, cap * sizeof(MaskState)));
    CK(cudaMalloc((void**)&pl->hist, (size_t)cap * hcap * 4 * sizeof(double)));
    CK(cudaMalloc((void**)&pl->part, (size_t)2 * cap * nb * 3 * sizeof(double)));
    CK(cudaMalloc((void**)&pl->ctr, ((size_t)cap + 1) * sizeof(unsigned)));   // + the prologue's ticket
    // the per-mask scalars in one block, [energy][tolp][thrp][thrm][thrms][thrx] (cap
    // each): a solve with host tolerances uploads them in one copy (session_setup)
    CK(cudaMalloc((void**)&pl->energy, 6 * (size_t)cap * sizeof(double)));
    pl->tolp = pl->energy + cap;
    pl->thrp = pl->tolp + cap;
    pl->thrm = pl->thrp + cap;
    pl->thrms = pl->thrm + cap;
    pl->thrx = pl->thrms + cap;
    CK(cudaMalloc((void**)&pl->escale, cap * sizeof(double)));
    CK(cudaMalloc((void**)&pl->psum, (size_t)2 * cap * 32 * sizeof(double)));
    CK(cudaMemsetAsync(pl->ctr, 0, ((size_t)cap + 1) * sizeof(unsigned), pl->stream));
    CK(cudaMemsetAsync(pl->st, 0, cap * sizeof(MaskState), pl->stream));
    pl->cap = cap;
    pl->hist_cap = hcap;
    pl->tm_field_ok = !pl->generic && tma_encode(&pl->tm_field, pl->field, pl->prec == PM_SINGLE, 2LL * pl->nx,
                                                 pl->ny, cap, 2 * solve_cols(pl));
    pl->tm_field2_ok = false;
    return PM_OK;
}

// Partial slots per row of the row sweep (one per warp of a row group).
int row_wpr(const pm_plan* pl) { return std::max(1, kset(pl->prec, pl->lgx).row.TG / 32); }

// Elements of one parity half of `part`.
size_t part_half(const pm_plan* pl) { return (size_t)pl->cap * std::max(std::max(pl->cc.nblk, pl->nx), 148) * 3; }

// Column tasks per mask of the persistent kernel.
int solve_tpm(const pm_plan* pl) {
    const KernelSet& k = kset(pl->prec, pl->lgy);
    const int C = std::max(1, k.solve_threads / std::max(1, k.col.TG));
    return std::max(1, pl->nx / C);
}

// RAAR buffers (allocated on first use, sized to the batch capacity).
int ensure_raar(pm_plan* pl) {
    if (pl->raar_cap >= pl->cap) return PM_OK;
    for (void* b : {pl->field2, pl->xbuf, (void*)pl->rpart})
        if (b) cudaFree(b);
    pl->field2 = pl->xbuf = nullptr;
    pl->rpart = nullptr;
    pl->raar_cap = 0;
    const size_t n = (size_t)pl->cap * pl->N;
    CK(cudaMalloc(&pl->field2, n * pl->csz));
    if (pl->generic) {                     // mixed radix: the second iterate buffer only
        pl->raar_cap = pl->cap;
        return PM_OK;
    }
    CK(cudaMalloc(&pl->xbuf, n * pl->csz));
    CK(cudaMalloc((void**)&pl->rpart, (size_t)pl->cap * pl->ny * row_wpr(pl) * 2 * sizeof(double)));
    pl->raar_cap = pl->cap;
    pl->tm_field2_ok = tma_encode(&pl->tm_field2, pl->field2, pl->prec == PM_SINGLE, 2LL * pl->nx, pl->ny, pl->cap,
                                  2 * solve_cols(pl));
    return PM_OK;
}

int ensure_outputs(pm_plan* pl, bool phases, bool levels, bool ustar, bool vstar) {
    const size_t n = (size_t)pl->cap * pl->N;
    if (phases && !pl->phases) CK(cudaMalloc((void**)&pl->phases, n * sizeof(double)));
    if (levels && !pl->levels) CK(cudaMalloc((void**)&pl->levels, n));
    if (ustar && !pl->ustar) CK(cudaMalloc(&pl->ustar, n * pl->csz));
    if (vstar && !pl->vstar) CK(cudaMalloc(&pl->vstar, n * pl->csz));
    return PM_OK;
}

// --------------------------------------------------------------- launches
template <typename T>
RowArgs<T> row_args(pm_plan* pl, int mode, int it) {
    const pm_params& prm = pl->s.prm;
    const bool raar = prm.algorithm == PM_ALGO_RAAR;
    RowArgs<T> a;
    a.field = (cx<T>*)pl->field;
    a.out = raar ? (cx<T>*)pl->field2 : a.field;
    a.p = (const T*)(raar ? pl->s.p : pl->s.ps);   // GS: S p (see prologue_kernel); RAAR: p
    a.p_stride = pl->s.p_stride;
    a.twf = (const twe<T>*)pl->tw_row;
    a.twi = (const twe<T>*)pl->tw_row_i;
    a.nx = pl->nx;
    a.ny = pl->ny;
    a.scale = (T)(1.0 / std::sqrt((double)pl->N));
    a.thr_p = pl->thrp;
    a.mode = mode;
    a.it = it;
    a.st = pl->st;
    a.x = raar ? (cx<T>*)pl->xbuf : nullptr;
    a.beta = (T)prm.beta;
    a.c1 = (T)(1.0 - 2.0 * prm.beta);
    a.thr_x = pl->thrx;
    a.rpart = pl->rpart;
    a.wpr = row_wpr(pl);
    a.ctl = make_ctl(pl);
    a.hist = pl->hist;
    a.hist_stride = pl->hist_cap;
    a.cpart = pl->part;
    a.cpart_alt = (long long)part_half(pl);
    a.tpm = solve_tpm(pl);
    a.ctr = pl->ctr;
    a.nblk = pl->rc.nblk;
    return a;
}

template <typename T>
FinalArgs<T> final_args(pm_plan* pl) {
    FinalArgs<T> a;
    a.field = (const cx<T>*)pl->field;
    a.p = (const T*)pl->s.p;
    a.p_stride = pl->s.p_stride;
    a.tw = (const twe<T>*)pl->tw_row;
    a.nx = pl->nx;
    a.ny = pl->ny;
    a.scale = (T)(1.0 / std::sqrt((double)pl->N));
    a.tol_p = pl->tolp;
    a.st = pl->st;
    a.v_star = (cx<T>*)pl->s.vstar;
    a.u_star = (cx<T>*)pl->s.ustar;
    a.phases = (double*)pl->s.phases;
    a.levels = (uint8_t*)pl->s.levels;
    const pm_params& prm = pl->s.prm;
    const bool raar = prm.algorithm == PM_ALGO_RAAR;
    a.x = raar ? (const cx<T>*)pl->xbuf : nullptr;
    a.thr_x = pl->thrx;
    a.rpart = pl->rpart;
    a.wpr = row_wpr(pl);
    a.ctl = make_ctl(pl);
    return a;
}

template <typename T>
ColArgs<T> col_args(pm_plan* pl, int mode, int u_iter) {
    const pm_params& prm = pl->s.prm;
    const bool raar = prm.algorithm == PM_ALGO_RAAR;
    ColArgs<T> a;
    a.field = (cx<T>*)pl->field;
    a.in = raar ? (const cx<T>*)pl->field2 : a.field;
    a.raar = raar ? 1 : 0;
    a.xpart = pl->rpart;
    a.xparts = pl->ny * row_wpr(pl);
    a.energy = pl->energy;
    a.part_alt = (long long)part_half(pl);
    a.m = (const T*)pl->s.m;
    a.m_stride = (long long)pl->N;
    a.mT = (const T*)pl->s.mT;
    a.twf = (const twe<T>*)pl->tw_col;
    a.twi = (const twe<T>*)pl->tw_col_i;
    a.nx = pl->nx;
    a.ny = pl->ny;
    a.scale = (T)(1.0 / std::sqrt((double)pl->N));
    a.thr_m = pl->thrm;
    a.escale = pl->escale;
    a.mode = mode;
    a.u_iter = u_iter;
    a.ctl = make_ctl(pl);
    a.st = pl->st;
    a.hist = pl->hist;
    a.hist_stride = pl->hist_cap;
    a.part = pl->part;
    a.ctr = pl->ctr;
    a.nblk = pl->cc.nblk;
    return a;
}

template <typename T>
int launch_row(pm_plan* pl, int batch, int mode, int it) {
    RowArgs<T> a = row_args<T>(pl, mode, it);
    void* args[] = {&a};
    CK(cudaLaunchKernel(kset(pl->prec, pl->lgx).row_iter, dim3(pl->rc.nblk, batch), dim3(pl->rc.threads),
                        args, pl->rc.smem, pl->stream));
    pl->launches++;
    return PM_OK;
}

template <typename T>
int launch_final(pm_plan* pl, int batch) {
    FinalArgs<T> a = final_args<T>(pl);
    double* hist = pl->hist;
    int hs = pl->hist_cap;
    unsigned* ctr = pl->ctr;
    int nblk = pl->rc.nblk;
    void* args[] = {&a, &hist, &hs, &ctr, &nblk};
    CK(cudaLaunchKernel(kset(pl->prec, pl->lgx).row_final, dim3(pl->rc.nblk, batch), dim3(pl->rc.threads),
                        args, pl->rc.smem, pl->stream));
    pl->launches++;
    return PM_OK;
}

template <typename T>
int launch_col(pm_plan* pl, int batch, int mode, int u_iter) {
    ColArgs<T> a = col_args<T>(pl, mode, u_iter);
    void* args[] = {&a};
    CK(cudaLaunchKernel(kset(pl->prec, pl->lgy).col_iter, dim3(pl->cc.nblk, batch), dim3(pl->cc.threads),
                        args, pl->cc.smem, pl->stream));
    pl->launches++;
    return PM_OK;
}

// One cooperative launch of the persistent solve kernel: optional initial
// iterate, iterations [it_begin, it_end), optional final pair.
// The TMA variant when CTAs get several column tasks per phase (batches):
// its tiles stream the next task in while one computes.
bool tma_wanted(const pm_plan* pl) {
    const long long col_tasks = (long long)pl->s.batch * (pl->nx / solve_cols(pl));
    return pl->solve_grid_tma > 0 && col_tasks >= 2LL * pl->solve_grid_tma;
}

template <typename T>
int launch_solve(pm_plan* pl, int do_init, int it_begin, int it_end, int do_final, int do_probe) {
    const KernelSet& k = kset(pl->prec, pl->lgx);
    SolveArgs<T> a;
    a.row = row_args<T>(pl, 1, 0);
    a.col = col_args<T>(pl, 2, 0);
    a.fin = final_args<T>(pl);
    a.bar = pl->bar;
    a.batch = pl->s.batch;
    a.it_begin = it_begin;
    a.it_end = it_end;
    a.do_init = do_init;
    a.do_final = do_final;
    a.init_mode = pl->s.prm.init_complex ? 1 : 0;
    a.do_probe = do_probe;
    a.stamps = pl->stamps;
    {
        static const bool off = getenv("PM_NO_TMA") != nullptr;
        const bool raar = pl->s.prm.algorithm == PM_ALGO_RAAR;
        const bool in_ok = raar ? pl->tm_field2_ok : pl->tm_field_ok;
        a.tma = (!off && in_ok && pl->tm_m_ok) ? 1 : 0;
        a.tm_in = raar ? pl->tm_field2 : pl->tm_field;
        a.tm_m = pl->tm_m;
    }
    const bool raar = pl->s.prm.algorithm == PM_ALGO_RAAR;
    const bool use_tma = a.tma && tma_wanted(pl);
    {   // p and m resident in shared memory when every CTA has one row and one column task
        static const bool off = getenv("PM_NO_RES") != nullptr;
        const long long grid = pl->solve_grid, nx = pl->nx;
        const int G = std::max(1, k.solve_threads / std::max(1, k.row.TG));
        const long long rows_per_cta = ((long long)pl->s.batch * nx + grid - 1) / std::max(1LL, grid);
        const long long col_tasks = (long long)pl->s.batch * (nx / solve_cols(pl));
        a.res = (!off && !use_tma && rows_per_cta <= G && col_tasks <= grid) ? 1 : 0;
    }
    a.tma = use_tma ? 1 : 0;
    {   // z' written back by TMA stores from the exchange buffer (PM_NO_TMA_STORE: st.global)
        static const bool off = getenv("PM_NO_TMA_STORE") != nullptr;
        a.tma_out = (use_tma && !off && pl->tm_field_ok) ? 1 : 0;
        a.tm_out = pl->tm_field;
    }
    const void* fn = use_tma ? (raar ? k.solve_raar_tma : k.solve_tma) : (raar ? k.solve_raar : k.solve);
    void* args[] = {&a};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(use_tma ? pl->solve_grid_tma : pl->solve_grid);
    cfg.blockDim = dim3(k.solve_threads);
    cfg.dynamicSmemBytes = (size_t)(use_tma ? (raar ? k.solve_smem_raar_tma : k.solve_smem_tma)
                                            : (raar ? k.solve_smem_raar : k.solve_smem));
    cfg.stream = pl->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CK(cudaMemsetAsync(pl->bar, 0, sizeof(GridBar), pl->stream));
    CK(cudaLaunchKernelExC(&cfg, fn, args));
    pl->launches++;
    return PM_OK;
}

int solve_launch(pm_plan* pl, int do_init, int it_begin, int it_end, int do_final, int do_probe = 0) {
    return pl->prec == PM_SINGLE ? launch_solve<float>(pl, do_init, it_begin, it_end, do_final, do_probe)
                                 : launch_solve<double>(pl, do_init, it_begin, it_end, do_final, do_probe);
}

int row(pm_plan* pl, int batch, int mode, int it) {
    return pl->prec == PM_SINGLE ? launch_row<float>(pl, batch, mode, it)
                                 : launch_row<double>(pl, batch, mode, it);
}
int final_pair(pm_plan* pl, int batch) {
    return pl->prec == PM_SINGLE ? launch_final<float>(pl, batch) : launch_final<double>(pl, batch);
}
int col(pm_plan* pl, int batch, int mode, int u_iter) {
    return pl->prec == PM_SINGLE ? launch_col<float>(pl, batch, mode, u_iter)
                                 : launch_col<double>(pl, batch, mode, u_iter);
}

// Stand-alone 2-D transform: rows (in -> out) then columns (out -> out).
template <typename T>
int launch_fft2(pm_plan* pl, const void* in, void* out, int dir, int batch) {
    const KernelSet& kr = kset(pl->prec, pl->lgx);
    const KernelSet& kc = kset(pl->prec, pl->lgy);
    const cx<T>* src = (const cx<T>*)in;
    cx<T>* dst = (cx<T>*)out;
    const twe<T>* twr = (const twe<T>*)(dir < 0 ? pl->tw_row : pl->tw_row_i);
    const twe<T>* twc = (const twe<T>*)(dir < 0 ? pl->tw_col : pl->tw_col_i);
    int nx = pl->nx, ny = pl->ny;
    T sx = (T)(1.0 / std::sqrt((double)nx)), sy = (T)(1.0 / std::sqrt((double)ny));
    {
        void* args[] = {&src, &dst, &twr, &nx, &ny, &sx, &dir};
        CK(cudaLaunchKernel(kr.row_fft, dim3(pl->rc.nblk, batch), dim3(pl->rc.threads), args,
                            pl->rc.smem, pl->stream));
    }
    {
        const cx<T>* src2 = dst;
        void* args[] = {&src2, &dst, &twc, &nx, &ny, &sy, &dir};
        CK(cudaLaunchKernel(kc.col_fft, dim3(pl->cc.nblk, batch), dim3(pl->cc.threads), args,
                            pl->cc.smem, pl->stream));
    }
    pl->launches += 2;
    return PM_OK;
}

// ------------------------------------------------------- mixed-radix path
// Factor n into passes of radix 4, 2, 3, 5, 7 (fails for other primes).
int env_int(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return v && *v ? std::atoi(v) : dflt;
}

// Pass plan of a length-n transform: the fewest passes over the radices
// the kernels instantiate (base 2, 3, 4, 5, 7, 8 and the register
// composites 9, 10, 12, 16 of pm_generic.cuh, up to rmax), ties broken
// towards the larger smallest radix.
bool gen_factor(int n, GenPlan* g, int rmax) {
    if (n < 1 || n > (1 << kMaxLg)) return false;
    static const int radices[] = {16, 12, 10, 9, 8, 7, 5, 4, 3, 2};
    // best[k] for every divisor k of n: (passes, -smallest radix, first radix)
    std::map<int, std::pair<std::pair<int, int>, int>> best;
    std::vector<int> divs;
    for (int d = 1; d <= n; ++d)
        if (n % d == 0) divs.push_back(d);
    best[1] = {{0, -1000}, 0};
    for (int k : divs) {
        if (k == 1) continue;
        std::pair<std::pair<int, int>, int> b{{1 << 20, 0}, 0};
        for (int r : radices) {
            if (r > rmax || k % r != 0) continue;
            auto it = best.find(k / r);
            if (it == best.end() || it->second.first.first >= (1 << 20)) continue;
            const std::pair<int, int> cand{it->second.first.first + 1, std::max(it->second.first.second, -r)};
            if (cand < b.first) b = {cand, r};
        }
        best[k] = b;
    }
    if (best[n].first.first >= (1 << 20) || best[n].first.first > kGenMaxPasses) return false;
    std::vector<int> rs;
    for (int rest = n; rest > 1; rest /= best[rest].second) rs.push_back(best[rest].second);
    // pass order: 1 = descending radix (default; 800x600 fp32: 0.82 vs
    // 0.87 ms with 0 = powers of two first, then the rest ascending); 2 = ascending
    const int order = env_int("PM_GEN_ORDER", 1);
    auto pow2 = [](int r) { return (r & (r - 1)) == 0; };
    std::sort(rs.begin(), rs.end(), [&](int a, int b) {
        if (order == 1) return a > b;
        if (order == 2) return a < b;
        if (pow2(a) != pow2(b)) return pow2(a);
        return pow2(a) ? a > b : a < b;
    });
    g->L = n;
    g->np = 0;
    int ns = 1;
    for (int r : rs) {
        g->radix[g->np] = r;
        g->ns[g->np] = ns;
        g->step[g->np] = n / (ns * r);
        g->mg[g->np] = ns == 1 ? 0u : 0xFFFFFFFFu / (unsigned)ns + 1u;
        ++g->np;
        ns *= r;
    }
    return true;
}

// exp(-2 pi i k / n) in the plan precision, long-double accurate.
int gen_twiddles(int prec, int n, void** out) {
    const long double pi = 3.141592653589793238462643383279502884L;
    if (prec == PM_SINGLE) {
        std::vector<float2> t(n);
        for (int k = 0; k < n; ++k) {
            const long double a = 2.0L * pi * (long double)k / (long double)n;
            t[k] = make_float2((float)cosl(a), (float)-sinl(a));
        }
        CK(cudaMalloc(out, n * sizeof(float2)));
        CK(cudaMemcpy(*out, t.data(), n * sizeof(float2), cudaMemcpyHostToDevice));
    } else {
        std::vector<double2> t(n);
        for (int k = 0; k < n; ++k) {
            const long double a = 2.0L * pi * (long double)k / (long double)n;
            t[k] = make_double2((double)cosl(a), (double)-sinl(a));
        }
        CK(cudaMalloc(out, n * sizeof(double2)));
        CK(cudaMemcpy(*out, t.data(), n * sizeof(double2), cudaMemcpyHostToDevice));
    }
    return PM_OK;
}

constexpr size_t kGenSmem = 100 * 1024;  // preferred tile bytes per CTA (TC is halved down to 1 above it)


int gen_setup(pm_plan* pl) {
    CKR(gen_twiddles(pl->prec, pl->nx, &pl->gtwx));
    CKR(gen_twiddles(pl->prec, pl->ny, &pl->gtwy));
    // transforms per CTA: a power of two, enough CTAs to cover the SMs,
    // columns wide enough for >= 32-byte segments
    // transforms per CTA (TC): 2, halved while the grid would not cover the
    // SMs or the tiles would not fit; 256 threads (measured on the paper's
    // 800x600 fp32: TC 1-8 x 64-256 threads, scripts/gen_tune_rmax.sh)
    auto shape_for = [&](const GenPlan& g, int ntrans, const char* etc, const char* ent, int& tc, int& nt) {
        tc = env_int(etc, 2);
        while (tc > 1 && (gen_smem_bytes(g.L, tc, pl->csz) > kGenSmem || (ntrans + tc - 1) / tc < 148)) tc >>= 1;
        nt = env_int(ent, 256);
    };
    shape_for(pl->gx, pl->ny, "PM_GEN_TCR", "PM_GEN_NTR", pl->gtc_r, pl->gnt_r);
    shape_for(pl->gy, pl->nx, "PM_GEN_TCC", "PM_GEN_NTC", pl->gtc_c, pl->gnt_c);
    {   // the register budget bounds the CTA size
        cudaFuncAttributes fa[4];
        const bool f32 = pl->prec == PM_SINGLE;
        CK(cudaFuncGetAttributes(&fa[0], f32 ? (const void*)&gen_fft_kernel<float> : (const void*)&gen_fft_kernel<double>));
        CK(cudaFuncGetAttributes(&fa[1], f32 ? (const void*)&gen_col_sweep_kernel<float>
                                             : (const void*)&gen_col_sweep_kernel<double>));
        CK(cudaFuncGetAttributes(&fa[2], f32 ? (const void*)&gen_row_sweep_kernel<float>
                                             : (const void*)&gen_row_sweep_kernel<double>));
        CK(cudaFuncGetAttributes(&fa[3], f32 ? (const void*)&gen_row_raar_kernel<float>
                                             : (const void*)&gen_row_raar_kernel<double>));
        const int cap = std::min({fa[0].maxThreadsPerBlock, fa[1].maxThreadsPerBlock, fa[2].maxThreadsPerBlock,
                                  fa[3].maxThreadsPerBlock}) / 32 * 32;
        pl->gnt_r = std::min(pl->gnt_r, cap);
        pl->gnt_c = std::min(pl->gnt_c, cap);
    }
    pl->gsm_r = gen_smem_bytes(pl->nx, pl->gtc_r, pl->csz);
    pl->gsm_c = gen_smem_bytes(pl->ny, pl->gtc_c, pl->csz);
    const size_t mx = std::max(pl->gsm_r, pl->gsm_c);
    cudaError_t e;
    if (pl->prec == PM_SINGLE) {
        e = allow_smem((const void*)&gen_fft_kernel<float>, mx);
        if (e == cudaSuccess) e = allow_smem((const void*)&gen_col_sweep_kernel<float>, mx);
        if (e == cudaSuccess) e = allow_smem((const void*)&gen_row_sweep_kernel<float>, mx);
        if (e == cudaSuccess) e = allow_smem((const void*)&gen_row_raar_kernel<float>, mx);
    } else {
        e = allow_smem((const void*)&gen_fft_kernel<double>, mx);
        if (e == cudaSuccess) e = allow_smem((const void*)&gen_col_sweep_kernel<double>, mx);
        if (e == cudaSuccess) e = allow_smem((const void*)&gen_row_sweep_kernel<double>, mx);
        if (e == cudaSuccess) e = allow_smem((const void*)&gen_row_raar_kernel<double>, mx);
    }
    if (e != cudaSuccess) return cuda_err(e, "cudaFuncSetAttribute(gen kernels)");
    return PM_OK;
}

// One axis (rows: axis 0, columns: axis 1) of the unitary 2-D DFT,
// in -> out, for `batch` masks; masks that stopped are skipped unless
// all_masks (st null: no mask state, stand-alone transform).
template <typename T>
int gen_axis(pm_plan* pl, const void* in, void* out, int axis, int dir, int batch, const MaskState* st,
             int all_masks) {
    const bool rows = axis == 0;
    const GenPlan& g = rows ? pl->gx : pl->gy;
    const int TC = rows ? pl->gtc_r : pl->gtc_c;
    const int ntrans = rows ? pl->ny : pl->nx;
    const long long tstride = rows ? pl->nx : 1, estride = rows ? 1 : pl->nx;
    const T scale = (T)(1.0 / std::sqrt((double)g.L));
    const dim3 grid((ntrans + TC - 1) / TC, batch);
    int lgTC = 0;
    while ((1 << lgTC) < TC) ++lgTC;
    gen_fft_kernel<T><<<grid, rows ? pl->gnt_r : pl->gnt_c, rows ? pl->gsm_r : pl->gsm_c, pl->stream>>>(
        (const cx<T>*)in, (cx<T>*)out, (const cx<T>*)(rows ? pl->gtwx : pl->gtwy), g, ntrans, tstride, estride,
        (long long)pl->N, dir, scale, lgTC, st, all_masks);
    CK(cudaGetLastError());
    pl->launches++;
    return PM_OK;
}

int gen_fft2(pm_plan* pl, const void* in, void* out, int dir, int batch, const MaskState* st = nullptr,
             int all_masks = 1) {
    if (pl->prec == PM_SINGLE) {
        CKR(gen_axis<float>(pl, in, out, 0, dir, batch, st, all_masks));
        return gen_axis<float>(pl, out, out, 1, dir, batch, st, all_masks);
    }
    CKR(gen_axis<double>(pl, in, out, 0, dir, batch, st, all_masks));
    return gen_axis<double>(pl, out, out, 1, dir, batch, st, all_masks);
}

int gen_elem_blocks(const pm_plan* pl) {
    return (int)std::max<long long>(1, std::min<long long>(((long long)pl->N + 1023) / 1024, 148));
}

GenSolveArgs gen_args(pm_plan* pl) {
    GenSolveArgs g;
    g.ctl = make_ctl(pl);
    g.st = pl->st;
    g.hist = pl->hist;
    g.hist_stride = pl->hist_cap;
    g.part = pl->part;
    g.ctr = pl->ctr;
    g.nblk = gen_elem_blocks(pl);
    g.n = (long long)pl->N;
    return g;
}

// w = RowFFT(u): the iterates (field) into the work buffer.
int gen_rows_fwd(pm_plan* pl, int all_masks) {
    return pl->prec == PM_SINGLE ? gen_axis<float>(pl, pl->field, pl->tmp, 0, PM_FORWARD, pl->s.batch, pl->st, all_masks)
                                 : gen_axis<double>(pl, pl->field, pl->tmp, 0, PM_FORWARD, pl->s.batch, pl->st,
                                                    all_masks);
}

// Launch configuration with programmatic dependent launch: the sweep kernel
// may be scheduled while its predecessor drains; it prefetches its twiddles
// and then waits (griddepcontrol.wait) before touching the predecessor's data.
struct PdlConfig {
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[1];
    const cudaLaunchConfig_t* get() {
        cfg.attrs = attr;
        return &cfg;
    }
};
PdlConfig pdl_config(dim3 grid, int threads, size_t smem, cudaStream_t stream) {
    static const bool off = getenv("PM_NO_PDL") != nullptr;
    PdlConfig c;
    c.cfg.gridDim = grid;
    c.cfg.blockDim = dim3(threads);
    c.cfg.dynamicSmemBytes = smem;
    c.cfg.stream = stream;
    c.attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    c.attr[0].val.programmaticStreamSerializationAllowed = off ? 0 : 1;
    c.cfg.numAttrs = 1;
    return c;
}

int lg_of(int tc) {
    int l = 0;
    while ((1 << l) < tc) ++l;
    return l;
}

// Fused column sweep on the work buffer (ColFFT, replace_m + metrics of
// u_{u_iter}, ColIFFT).
template <typename T>
int gen_col_sweep(pm_plan* pl, int u_iter, int metrics_only, int all_masks) {
    const int TC = pl->gtc_c;
    const dim3 grid((pl->nx + TC - 1) / TC, pl->s.batch);
    GenSolveArgs g = gen_args(pl);
    g.nblk = (int)grid.x;
    // does iterate u_iter need its decision in this sweep (see gen_col_sweep_kernel)
    const pm_params& prm = pl->s.prm;
    const bool raar = prm.algorithm == PM_ALGO_RAAR;
    const bool rec = u_iter >= 1 && (u_iter - 1) % prm.record_every == 0;
    const int need_dec = (metrics_only || all_masks ||
                          (raar ? rec
                                : (rec || prm.early_stop_tol >= 0.0 || pl->s.lockstep || u_iter >= prm.max_iters)))
                             ? 1 : 0;
    CK(cudaLaunchKernelEx(pdl_config(grid, pl->gnt_c, pl->gsm_c, pl->stream).get(), gen_col_sweep_kernel<T>,
                          (cx<T>*)pl->tmp, (const T*)pl->s.m, (const T*)pl->s.mT, (const double*)pl->thrm,
                          (const double*)pl->escale, (const cx<T>*)pl->gtwy, pl->gy, pl->nx, lg_of(TC), g, u_iter,
                          metrics_only, all_masks, raar ? 1 : 0, need_dec));
    pl->launches++;
    return PM_OK;
}

// Fused row sweep (RowIFFT, P_S into the iterate, RowFFT into the work buffer).
template <typename T>
int gen_row_sweep(pm_plan* pl, int it) {
    const int TC = pl->gtc_r;
    const dim3 grid((pl->ny + TC - 1) / TC, pl->s.batch);
    CK(cudaLaunchKernelEx(pdl_config(grid, pl->gnt_r, pl->gsm_r, pl->stream).get(), gen_row_sweep_kernel<T>,
                          (cx<T>*)pl->tmp, (cx<T>*)pl->field, (const T*)pl->s.p, (long long)pl->s.p_stride,
                          (const double*)pl->thrx, (const cx<T>*)pl->gtwx, pl->gx, pl->ny, lg_of(TC), pl->st,
                          (long long)pl->N, it, pl->s.stepping ? 1 : 0));
    pl->launches++;
    return PM_OK;
}

int ensure_mT(pm_plan* pl);
int ensure_ps(pm_plan* pl, int grids);
int launch_transpose_m(pm_plan* pl);

int gen_begin(pm_plan* pl) {
    auto& s = pl->s;
    const long long total = (long long)s.batch * pl->N;
    if (!s.prm.init_complex) {
        const int blocks = (int)std::min<long long>((total + 255) / 256, 4096);
        if (pl->prec == PM_SINGLE)
            gen_real_to_complex<float><<<blocks, 256, 0, pl->stream>>>((const float*)s.m, (float2*)pl->field, total);
        else
            gen_real_to_complex<double><<<blocks, 256, 0, pl->stream>>>((const double*)s.m, (double2*)pl->field,
                                                                         total);
        CK(cudaGetLastError());
        pl->launches++;
    }
    CKR(gen_fft2(pl, pl->field, pl->field, PM_INVERSE, s.batch, pl->st, 0));   // u0 = F^-1(m e^{i phi})
    // m transposed per mask, so a column task's m is TC contiguous runs (buffer
    // sized in session_setup, outside any capture)
    s.mT = nullptr;
    if (pl->mT_bytes >= (size_t)s.batch * pl->N * pl->rsz) CKR(launch_transpose_m(pl));
    return gen_rows_fwd(pl, 0);                                                  // w = RowFFT(u0)
}

// RAAR row sweep of iteration `it` (x_{it-1} from the buffer of its parity,
// x_it into the other; upd = 0: gap + decision of x_{it-1} only).
template <typename T>
int gen_row_raar(pm_plan* pl, int it, int upd) {
    const int TC = pl->gtc_r;
    const dim3 grid((pl->ny + TC - 1) / TC, pl->s.batch);
    GenSolveArgs g = gen_args(pl);
    g.nblk = (int)grid.x;
    cx<T>* xs[2] = {(cx<T>*)pl->field, (cx<T>*)pl->field2};
    const auto& prm = pl->s.prm;
    CK(cudaLaunchKernelEx(pdl_config(grid, pl->gnt_r, pl->gsm_r, pl->stream).get(), gen_row_raar_kernel<T>,
                          (cx<T>*)pl->tmp, (const cx<T>*)xs[(it - 1) & 1], xs[it & 1], (const T*)pl->s.p,
                          (long long)pl->s.p_stride, (const double*)pl->thrx, (const cx<T>*)pl->gtwx, pl->gx, pl->ny,
                          lg_of(TC), g, (T)prm.beta, (T)(1.0 - 2.0 * prm.beta), (const double*)pl->energy,
                          pl->escale, it, upd));
    pl->launches++;
    return PM_OK;
}

// RAAR: gap + decision of the current iterate x_{s.it} now (the stepping
// API's probe, and the last iterate before the pair). The column sweep
// leaves RowFFT(P_M x) in the work buffer for the row probe; `restore`
// puts RowFFT(x) back for further steps.
int gen_raar_probe(pm_plan* pl, bool restore) {
    const bool f32 = pl->prec == PM_SINGLE;
    const int it = pl->s.it;
    CKR(f32 ? gen_col_sweep<float>(pl, it, 0, 0) : gen_col_sweep<double>(pl, it, 0, 0));   // lit / dark, P_M
    CKR(f32 ? gen_row_raar<float>(pl, it + 1, 0) : gen_row_raar<double>(pl, it + 1, 0));   // gap, decision
    if (!restore) return PM_OK;
    const void* x = (it & 1) ? pl->field2 : pl->field;
    return f32 ? gen_axis<float>(pl, x, pl->tmp, 0, PM_FORWARD, pl->s.batch, pl->st, 0)
               : gen_axis<double>(pl, x, pl->tmp, 0, PM_FORWARD, pl->s.batch, pl->st, 0);
}

// Two fused sweeps per iteration over the work buffer, which holds
// RowFFT(u_{it-1}) on entry and RowFFT(u_it) on exit.
int gen_steps(pm_plan* pl, int n, bool probe) {
    auto& s = pl->s;
    const bool f32 = pl->prec == PM_SINGLE;
    bool any = false;
    if (s.prm.algorithm == PM_ALGO_RAAR) {
        for (int i = 0; i < n && s.it < s.prm.max_iters; ++i) {
            s.it += 1;
            any = true;
            // lit / dark of x_{it-1}; then its gap + decision and x_it
            CKR(f32 ? gen_col_sweep<float>(pl, s.it - 1, 0, 0) : gen_col_sweep<double>(pl, s.it - 1, 0, 0));
            CKR(f32 ? gen_row_raar<float>(pl, s.it, 1) : gen_row_raar<double>(pl, s.it, 1));
        }
        if (any && probe) CKR(gen_raar_probe(pl, true));
        return PM_OK;
    }
    for (int i = 0; i < n && s.it < s.prm.max_iters; ++i) {
        s.it += 1;
        any = true;
        CKR(f32 ? gen_col_sweep<float>(pl, s.it - 1, 0, 0) : gen_col_sweep<double>(pl, s.it - 1, 0, 0));
        CKR(f32 ? gen_row_sweep<float>(pl, s.it) : gen_row_sweep<double>(pl, s.it));
    }
    if (any && probe)                                                       // gap + decision of u_it now
        CKR(f32 ? gen_col_sweep<float>(pl, s.it, 1, 0) : gen_col_sweep<double>(pl, s.it, 1, 0));
    return PM_OK;
}

template <typename T>
int gen_final_t(pm_plan* pl) {
    auto& s = pl->s;
    const dim3 grid(gen_elem_blocks(pl), s.batch);
    gen_final_kernel<T><<<grid, 256, 0, pl->stream>>>((const cx<T>*)pl->tmp, (const T*)s.p, s.p_stride, pl->tolp,
                                                      pl->st, (long long)pl->N, (cx<T>*)s.vstar, (cx<T>*)s.ustar,
                                                      (double*)s.phases, (uint8_t*)s.levels);
    CK(cudaGetLastError());
    pl->launches++;
    return PM_OK;
}

// v* = P_M u (every mask, decision of the last iterate if still pending),
// then u*, the mask and the levels.
int gen_finish(pm_plan* pl) {
    const bool f32 = pl->prec == PM_SINGLE;
    int u_iter = pl->s.it;
    if (pl->s.prm.algorithm == PM_ALGO_RAAR) {
        CKR(gen_raar_probe(pl, false));    // the last iterate's gap and decision (no-op where taken)
        const dim3 grid(gen_elem_blocks(pl), pl->s.batch);
        if (f32)
            gen_pick_kernel<float><<<grid, 256, 0, pl->stream>>>((float2*)pl->field, (const float2*)pl->field2, pl->st,
                                                                 (long long)pl->N, pl->s.it);
        else
            gen_pick_kernel<double><<<grid, 256, 0, pl->stream>>>((double2*)pl->field, (const double2*)pl->field2,
                                                                  pl->st, (long long)pl->N, pl->s.it);
        CK(cudaGetLastError());
        pl->launches++;
        u_iter = 0;                        // every decision is taken
    }
    if (pl->s.prm.algorithm != PM_ALGO_RAAR && !pl->s.stepping) {
        // GS in one enqueued solve: the work buffer of a mask that stopped at
        // u_j already holds ColIFFT(replace_m(ColFFT(RowFFT u_j))), the row
        // pre-image of v* = P_M u_j (its row sweeps were skipped); the rest
        // hold RowFFT(u_K) and get that column sweep now (with u_K's decision).
        // The iterate itself is never stored.
        CKR(f32 ? gen_col_sweep<float>(pl, u_iter, 0, 0) : gen_col_sweep<double>(pl, u_iter, 0, 0));
    } else {
        CKR(gen_rows_fwd(pl, 1));          // every mask from its last iterate (stopped ones included)
        CKR(f32 ? gen_col_sweep<float>(pl, u_iter, 0, 1) : gen_col_sweep<double>(pl, u_iter, 0, 1));
    }
    CKR(f32 ? gen_axis<float>(pl, pl->tmp, pl->tmp, 0, PM_INVERSE, pl->s.batch, pl->st, 1)
            : gen_axis<double>(pl, pl->tmp, pl->tmp, 0, PM_INVERSE, pl->s.batch, pl->st, 1));
    return f32 ? gen_final_t<float>(pl) : gen_final_t<double>(pl);
}

int fft2_dev(pm_plan* pl, const void* in, void* out, int dir, int batch) {
    if (pl->generic) return gen_fft2(pl, in, out, dir, batch);
    return pl->prec == PM_SINGLE ? launch_fft2<float>(pl, in, out, dir, batch)
                                 : launch_fft2<double>(pl, in, out, dir, batch);
}

int check_plan(pm_plan* pl) {
    if (!pl) return set_err(PM_ERR_ARG, "null plan");
    CK(cudaSetDevice(pl->device));
    return PM_OK;
}

// -------------------------------------------------------------- solve
// m e^{i phi} starts for `batch` masks of n pixels from the PCG64 state.
int enqueue_random_start(int prec, const void* d_m, void* d_out, long long n, int batch,
                         const unsigned long long rng[4], cudaStream_t stream) {
    const int threads = 256;
    const int blocks = (int)std::max<long long>(1, std::min<long long>((n + threads - 1) / threads, 148 * 8));
    const u128 inc = u128_of(rng[2], rng[3]);
    const PcgJump j = pcg_jump(inc, (unsigned long long)blocks * threads);
    const auto hi = [](u128 v) { return (unsigned long long)(v >> 64); };
    const auto lo = [](u128 v) { return (unsigned long long)v; };
    if (prec == PM_SINGLE)
        random_start_kernel<float><<<blocks, threads, 0, stream>>>(
            (const float*)d_m, (float2*)d_out, n, batch, rng[0], rng[1], rng[2], rng[3], hi(j.mult), lo(j.mult),
            hi(j.plus), lo(j.plus));
    else
        random_start_kernel<double><<<blocks, threads, 0, stream>>>(
            (const double*)d_m, (double2*)d_out, n, batch, rng[0], rng[1], rng[2], rng[3], hi(j.mult), lo(j.mult),
            hi(j.plus), lo(j.plus));
    CK(cudaGetLastError());
    return PM_OK;
}

int validate_params(const pm_params* prm, int batch) {
    if (!prm) return set_err(PM_ERR_ARG, "null params");
    if (batch < 1) return set_err(PM_ERR_ARG, "batch must be >= 1");
    if (prm->max_iters < 1) return set_err(PM_ERR_ARG, "max_iters must be >= 1");
    if (prm->record_every < 1) return set_err(PM_ERR_ARG, "record_every must be >= 1");
    if (prm->algorithm != PM_ALGO_GS && prm->algorithm != PM_ALGO_RAAR)
        return set_err(PM_ERR_ARG, "algorithm must be 0 (GS) or 1 (RAAR)");
    if (prm->algorithm == PM_ALGO_RAAR && !std::isfinite(prm->beta))
        return set_err(PM_ERR_ARG, "RAAR beta must be finite");
    if (prm->init_complex && prm->init_random)
        return set_err(PM_ERR_ARG, "init_complex and init_random are exclusive");
    return PM_OK;
}

// The Fourier-plane start of the session's masks into the field: the
// caller's complex starts (init_complex) or the seeded random phases
// generated on the device (init_random); the solve then runs its complex
// start path for both.
int stage_start(pm_plan* pl, const void* init, cudaMemcpyKind kind) {
    auto& s = pl->s;
    if (s.prm.init_complex) {
        if (!init) return set_err(PM_ERR_ARG, "init_complex set but m_init is NULL");
        CK(cudaMemcpyAsync(pl->field, init, (size_t)s.batch * pl->N * pl->csz, kind, pl->stream));
    } else if (s.prm.init_random) {
        CKR(enqueue_random_start(pl->prec, s.m, pl->field, (long long)pl->N, s.batch, s.prm.rng, pl->stream));
        pl->launches++;
        s.prm.init_complex = 1;
    }
    return PM_OK;
}

int ensure_red(pm_plan* pl, int nb) {
    if (nb + 1 <= pl->red_cap) return PM_OK;
    CK(cudaStreamSynchronize(pl->stream));
    drop_graphs(pl);                  // captured graphs hold the old pointer
    if (pl->red) cudaFree(pl->red);
    pl->red = nullptr;
    CK(cudaMalloc((void**)&pl->red, (nb + 1) * sizeof(double)));
    pl->red_cap = nb + 1;
    return PM_OK;
}
// Blocks per mask of the prologue: a fixed function of the grid size.
// (8192 elements per block, up to 8 blocks per SM: enough loads in flight for
// HBM-resident grids; the last block combines them one warp per mask)
int prologue_blocks(long long n) { return (int)std::max<long long>(1, std::min<long long>(8 * 148, (n + 8191) / 8192)); }


// Upload per-mask scalars and reset state; point the session at p/m.
int session_setup(pm_plan* pl, const void* d_p, const void* d_m, int batch, const pm_params* prm,
                  const double* tol_p, const double* tol_m, const double* energy) {
    CKR(validate_params(prm, batch));
    CKR(ensure_capacity(pl, batch, prm->max_iters));
    if (prm->algorithm == PM_ALGO_RAAR) CKR(ensure_raar(pl));
    if (pl->generic && getenv("PM_NO_MT") == nullptr) {
        pl->s.batch = batch;                // ensure_mT sizes for this batch
        CKR(ensure_mT(pl));
    }
    auto& s = pl->s;
    s = pm_plan::Session();
    s.active = true;
    s.batch = batch;
    s.prm = *prm;
    s.p = d_p;
    s.m = d_m;
    s.p_stride = prm->p_per_mask ? (long long)pl->N : 0;
    if (!pl->generic && prm->algorithm == PM_ALGO_GS) {
        CKR(ensure_ps(pl, prm->p_per_mask ? batch : 1));
        s.ps = pl->ps;
    }
    // (m's tensor map only where the TMA build can run: several column tasks per CTA)
    pl->tm_m_ok = !pl->generic && tma_wanted(pl) &&
                  tma_encode(&pl->tm_m, const_cast<void*>(d_m), pl->prec == PM_SINGLE, pl->nx, pl->ny, batch,
                             tma_m_box(pl));
    // pinned-free small uploads: stage in the session's host vectors, which
    // must outlive the async copies -> keep them in the plan
    // page-locked uploads mirroring the device block [energy][tolp][thrp][thrm][thrms][thrx]
    // (cap doubles each): one copy (each small copy costs several microseconds of stream time)
    const size_t cap = (size_t)pl->cap;
    unsigned char* stage = nullptr;
    CKR(host_stage(pl, 6 * cap * sizeof(double), &stage));
    double* h_en = reinterpret_cast<double*>(stage);
    for (int b = 0; b < batch; ++b) h_en[b] = energy ? energy[b] : 0.0;
    s.energy_on_device = energy == nullptr;
    CKR(ensure_red(pl, 4 * prologue_blocks((long long)pl->N) * batch));   // the prologue's partials
    if (!tol_p) {
        CK(cudaMemcpyAsync(pl->energy, h_en, batch * sizeof(double), cudaMemcpyHostToDevice, pl->stream));
        // tolerances from the device-resident p and m (no host pass over them);
        // their partial maxima live in `red` (sized here, outside any capture)
        s.tol_on_device = true;
        return PM_OK;
    }
    double* h_tolp = h_en + cap;
    double* h_thrp = h_tolp + cap;
    double* h_thrm = h_thrp + cap;
    double* h_thrms = h_thrm + cap;
    double* h_thrx = h_thrms + cap;
    for (int b = 0; b < batch; ++b) {
        const double tp = tol_p[prm->p_per_mask ? b : 0];
        h_tolp[b] = tp;
        zero_thresholds(tp, tol_m[b], pl->prec == PM_SINGLE, &h_thrp[b], &h_thrm[b], &h_thrx[b]);
        h_thrms[b] = 0.0;
    }
    CK(cudaMemcpyAsync(pl->energy, h_en, 6 * cap * sizeof(double), cudaMemcpyHostToDevice, pl->stream));
    return PM_OK;
}

bool persistent(const pm_plan* pl) {
    static const bool off = getenv("PM_NO_PERSISTENT") != nullptr;
    if (pl->path == 2) return false;
    return pl->solve_grid > 0 && (pl->path == 1 || !off);
}

// m transposed per mask for the persistent column phase (one contiguous run
// of m per column task instead of n_y runs shorter than a 32-byte sector):
// 4096^2 fp32 335 -> 300 us per iteration, 2048^2 67.3 -> 65.6; neutral or
// slightly worse where the runs are already >= 32 bytes (1024^2 fp32, fp64),
// so only below that. Not when the TMA variant streams m boxes itself (its
// field-only form, 2048^2 / 4096^2, stages m from this copy).
// The transposed-m buffer for the session's batch (outside any capture;
// captured graphs hold the old pointer, so they go when it is reallocated).
// The S p buffer for `grids` amplitude grids (outside any capture; captured
// graphs hold the old pointer, so they go when it is reallocated).
int ensure_ps(pm_plan* pl, int grids) {
    const size_t bytes = (size_t)grids * pl->N * pl->rsz;
    if (bytes <= pl->ps_bytes) return PM_OK;
    CK(cudaStreamSynchronize(pl->stream));
    drop_graphs(pl);
    if (pl->ps) cudaFree(pl->ps);
    pl->ps = nullptr;
    pl->ps_bytes = 0;
    CK(cudaMalloc(&pl->ps, bytes));
    pl->ps_bytes = bytes;
    return PM_OK;
}

int ensure_mT(pm_plan* pl) {
    const size_t bytes = (size_t)pl->s.batch * pl->N * pl->rsz;
    if (bytes <= pl->mT_bytes) return PM_OK;
    CK(cudaStreamSynchronize(pl->stream));
    drop_graphs(pl);
    if (pl->mT) cudaFree(pl->mT);
    pl->mT = nullptr;
    pl->mT_bytes = 0;
    CK(cudaMalloc(&pl->mT, bytes));
    pl->mT_bytes = bytes;
    return PM_OK;
}

int launch_transpose_m(pm_plan* pl) {
    auto& s = pl->s;
    const dim3 grid((pl->nx + 31) / 32, (pl->ny + 31) / 32, s.batch), block(32, 8);
    if (pl->prec == PM_SINGLE)
        transpose_kernel<float><<<grid, block, 0, pl->stream>>>((const float*)s.m, (float*)pl->mT, pl->nx, pl->ny);
    else
        transpose_kernel<double><<<grid, block, 0, pl->stream>>>((const double*)s.m, (double*)pl->mT, pl->nx,
                                                                 pl->ny);
    CK(cudaGetLastError());
    pl->launches++;
    s.mT = pl->mT;
    return PM_OK;
}

int enqueue_mT(pm_plan* pl) {
    static const bool off = getenv("PM_NO_MT") != nullptr;
    pl->s.mT = nullptr;
    const bool tma_streams_m = tma_wanted(pl) && kset(pl->prec, pl->lgx).solve_tma_m;
    if (off || !persistent(pl) || tma_streams_m || (size_t)solve_cols(pl) * pl->rsz >= 32) return PM_OK;
    CKR(ensure_mT(pl));
    return launch_transpose_m(pl);
}

int enqueue_prologue(pm_plan* pl) {
    auto& s = pl->s;
    const long long n = (long long)pl->N;
    ProArgs a{};
    a.p = s.p;
    a.m = s.m;
    a.ps = const_cast<void*>(s.ps);
    a.S = 1.0 / std::sqrt((double)pl->N);
    a.n = n;
    a.nb = prologue_blocks(n);
    a.chunk = (n + a.nb - 1) / a.nb;
    a.batch = s.batch;
    a.per_mask = s.prm.p_per_mask ? 1 : 0;
    a.single = pl->prec == PM_SINGLE;
    a.do_tol = s.tol_on_device ? 1 : 0;
    a.do_msum = s.energy_on_device ? 1 : 0;
    a.part = pl->red;
    a.st = pl->st;
    a.hist = pl->hist;
    a.hist_n = (long long)s.batch * pl->hist_cap * 4;
    a.tolp = pl->tolp;
    a.thrp = pl->thrp;
    a.thrm = pl->thrm;
    a.thrx = pl->thrx;
    a.energy = pl->energy;
    a.escale = pl->escale;
    a.ticket = pl->ctr + pl->cap;
    const dim3 grid(a.nb, s.batch);
    if (a.single)
        prologue_kernel<float><<<grid, 256, 0, pl->stream>>>(a);
    else
        prologue_kernel<double><<<grid, 256, 0, pl->stream>>>(a);
    CK(cudaGetLastError());
    pl->launches++;
    return PM_OK;
}

int enqueue_begin(pm_plan* pl) {
    auto& s = pl->s;
    CKR(enqueue_prologue(pl));
    if (pl->generic) return gen_begin(pl);
    if (persistent(pl)) {
        CKR(enqueue_mT(pl));
        return solve_launch(pl, 1, 1, 1, 0);
    }
    CKR(col(pl, s.batch, s.prm.init_complex ? 1 : 0, 0));   // u0 column half
    CKR(row(pl, s.batch, kRowInit, 0));                     // u0 row half, w0 = RowFFT(u0)
    CKR(col(pl, s.batch, 2, 0));                            // z1 = ColIFFT replace F u0
    return PM_OK;
}

// Iterations s.it+1 .. s.it+n. With `probe` (the stepping API), a RAAR solve
// also measures and decides the last iterate now instead of in the next
// sweep, so its record is readable when the call returns.
int enqueue_steps(pm_plan* pl, int n, bool probe = false) {
    auto& s = pl->s;
    if (pl->generic) return gen_steps(pl, n, probe);
    const bool raar = s.prm.algorithm == PM_ALGO_RAAR;
    if (persistent(pl)) {
        const int first = s.it + 1, last = std::min(s.it + n, s.prm.max_iters);
        if (last < first) return PM_OK;
        s.it = last;
        return solve_launch(pl, 0, first, last + 1, 0, probe && raar);
    }
    bool any = false;
    for (int i = 0; i < n && s.it < s.prm.max_iters; ++i) {
        s.it += 1;
        any = true;
        CKR(row(pl, s.batch, raar ? kRowRaar : kRowGS, s.it));   // u_it (x_it), w_it
        CKR(col(pl, s.batch, 2, s.it));        // metrics of u_it, stop decision, z_{it+1}
    }
    if (any && probe && raar) CKR(row(pl, s.batch, kRowProbe, s.it + 1));   // gap + decision of x_it
    return PM_OK;
}

int enqueue_finish(pm_plan* pl) {
    if (pl->generic) return gen_finish(pl);
    if (persistent(pl)) return solve_launch(pl, 0, 1, 1, 1);
    return final_pair(pl, pl->s.batch);
}

std::string graph_key(const pm_plan* pl) {
    const auto& s = pl->s;
    char buf[512];
    snprintf(buf, sizeof buf, "%d|%d|%d|%d|%a|%a|%a|%d|%d|%a|%p|%p|%lld|%p|%p|%p|%p|%d", s.batch,
             s.prm.max_iters, s.prm.record_every, s.prm.init_complex, s.prm.early_stop_tol,
             s.prm.t_lit, s.prm.t_dark, s.prm.p_per_mask, s.prm.algorithm, s.prm.beta, s.p, s.m,
             s.p_stride, s.phases, s.levels, s.ustar, s.vstar,
             (int)s.tol_on_device * 2 + (int)s.energy_on_device + 4 * (int)s.ring + 8 * (int)s.lockstep);
    return buf;
}

// Whole solve as one CUDA graph (captured once per configuration).
int enqueue_full_solve(pm_plan* pl) {
    static const bool no_graph = getenv("PM_NO_GRAPH") != nullptr;
    auto& s = pl->s;
    if (persistent(pl)) {
        // one cooperative launch: initial iterate, all iterations, final pair
        CKR(enqueue_prologue(pl));
        CKR(enqueue_mT(pl));
        s.it = s.prm.max_iters;
        return solve_launch(pl, 1, 1, s.prm.max_iters + 1, 1);
    }
    if (no_graph) {
        CKR(enqueue_begin(pl));
        CKR(enqueue_steps(pl, s.prm.max_iters));
        return enqueue_finish(pl);
    }
    const std::string key = graph_key(pl);
    auto it = pl->graphs.find(key);
    if (it == pl->graphs.end()) {
        if (pl->graphs.size() >= 16) drop_graphs(pl);
        cudaGraph_t g;
        CK(cudaStreamBeginCapture(pl->stream, cudaStreamCaptureModeThreadLocal));
        const long long l0 = pl->launches;
        int r = enqueue_begin(pl);
        if (r == PM_OK) r = enqueue_steps(pl, s.prm.max_iters);
        if (r == PM_OK) r = enqueue_finish(pl);
        cudaError_t e = cudaStreamEndCapture(pl->stream, &g);
        pl->launches = l0;   // counted when the graph is launched
        if (r != PM_OK) {
            if (e == cudaSuccess) cudaGraphDestroy(g);
            return r;
        }
        if (e != cudaSuccess) return cuda_err(e, "cudaStreamEndCapture");
        cudaGraphExec_t ge;
        e = cudaGraphInstantiate(&ge, g, 0);
        cudaGraphDestroy(g);
        if (e != cudaSuccess) return cuda_err(e, "cudaGraphInstantiate");
        it = pl->graphs.emplace(key, ge).first;
    }
    s.it = s.prm.max_iters;
    CK(cudaGraphLaunch(it->second, pl->stream));
    pl->launches += 2LL * s.prm.max_iters + 6;
    return PM_OK;
}

// Copy history / state back and fill the host-side result fields.
int read_records(pm_plan* pl, int first, int last, double* gap, double* lit, double* dark,
                 int* iters, int* diverged, int* aborted = nullptr, int* zero = nullptr, int* pair_bad = nullptr) {
    auto& s = pl->s;
    const int B = s.batch, K = s.prm.max_iters;
    // page-locked download area after the uploads' part of the staging buffer
    const size_t up = 6 * (size_t)pl->cap * sizeof(double);
    const size_t nh = (gap || lit || dark) ? (size_t)B * pl->hist_cap * 4 : 0;
    unsigned char* stage = nullptr;
    CKR(host_stage(pl, up + B * sizeof(MaskState) + nh * sizeof(double) + 16, &stage));
    MaskState* st = reinterpret_cast<MaskState*>(stage + up);
    const double* h = reinterpret_cast<const double*>(stage + up + ((B * sizeof(MaskState) + 15) & ~(size_t)15));
    CK(cudaMemcpyAsync(st, pl->st, B * sizeof(MaskState), cudaMemcpyDeviceToHost, pl->stream));
    if (nh)
        CK(cudaMemcpyAsync(const_cast<double*>(h), pl->hist, nh * sizeof(double), cudaMemcpyDeviceToHost,
                           pl->stream));
    CK(cudaStreamSynchronize(pl->stream));
    if (zero) *zero = 0;
    if (pair_bad) *pair_bad = 0;
    for (int b = 0; b < B; ++b) {
        if (zero) *zero |= st[b].zero;
        if (pair_bad && !st[b].diverged) *pair_bad |= st[b].pair_bad;
        if (iters) iters[b] = st[b].iters_run;
        if (diverged) diverged[b] = st[b].diverged;
        if (aborted) aborted[b] = st[b].aborted;
        if (nh) {
            for (int i = first; i <= last && i <= K; ++i) {
                const double* e = &h[((size_t)b * pl->hist_cap + (i - 1)) * 4];
                const bool ok = e[3] != 0.0;
                const size_t o = (size_t)b * K + (i - 1);
                if (gap) gap[o] = ok ? e[0] : NAN;
                if (lit) lit[o] = ok ? e[1] : NAN;
                if (dark) dark[o] = ok ? e[2] : NAN;
            }
        }
    }
    return PM_OK;
}

// The reference's validation messages (src/solver.py:122-125) for masks the
// device found identically zero.
int zero_error(int z) {
    if (z & 1) return set_err(PM_ERR_ARG, "SLM amplitude is identically zero");
    if (z & 2) return set_err(PM_ERR_ARG, "target pattern is identically zero (all dark)");
    return PM_OK;
}

int any_diverged(const std::vector<int>& d) {
    for (int x : d)
        if (x) return 1;
    return 0;
}

}  // namespace

// =================================================================== C ABI
extern "C" {

int pm_version(void) { return 100; }

const char* pm_last_error(void) { return g_err.c_str(); }

int pm_device_count(int* count) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) {
        cudaGetLastError();
        n = 0;
    }
    if (count) *count = n;
    return PM_OK;
}

int pm_plan_create(int device, int n_x, int n_y, int precision, int max_batch, pm_plan** out) {
    if (!out) return set_err(PM_ERR_ARG, "null output pointer");
    *out = nullptr;
    if (precision != PM_SINGLE && precision != PM_DOUBLE)
        return set_err(PM_ERR_ARG, "precision must be 0 (single) or 1 (double)");
    int lgx = lg2_exact(n_x), lgy = lg2_exact(n_y);
    GenPlan gx{}, gy{};
    bool generic = false;
    if (lgx < 0 || lgy < 0 || lgx > kMaxLg || lgy > kMaxLg) {
        // mixed-radix path: every side a product of 2, 3, 5, 7, at most 4096
        const int rmax = env_int("PM_GEN_RMAX", 16);
        if (!gen_factor(n_x, &gx, rmax) || !gen_factor(n_y, &gy, rmax))
            return set_err(PM_ERR_UNSUPPORTED, "grid " + std::to_string(n_x) + "x" + std::to_string(n_y) +
                                                   ": n_x and n_y must be at most 4096 with prime factors 2, 3, 5, 7");
        generic = true;
        lgx = lgy = 0;                          // the power-of-two kernel sets are not used
    }
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return set_err(PM_ERR_CUDA, "no CUDA device available (phasemask_b200 has no CPU fallback)");
    }
    if (device < 0 || device >= ndev) return set_err(PM_ERR_ARG, "device index out of range");
    CK(cudaSetDevice(device));
    pm_plan* pl = new pm_plan();
    pl->device = device;
    pl->nx = n_x;
    pl->ny = n_y;
    pl->prec = precision;
    pl->lgx = lgx;
    pl->lgy = lgy;
    pl->N = (size_t)n_x * n_y;
    pl->csz = precision == PM_SINGLE ? sizeof(float2) : sizeof(double2);
    pl->rsz = precision == PM_SINGLE ? sizeof(float) : sizeof(double);
    pl->generic = generic;
    pl->gx = gx;
    pl->gy = gy;
    pl->rc = row_config(pl);
    pl->cc = col_config(pl);
    auto fail = [&](int r) {
        pm_plan_destroy(pl);
        return r;
    };
    if (cudaStreamCreateWithFlags(&pl->stream, cudaStreamNonBlocking) != cudaSuccess)
        return fail(cuda_err(cudaGetLastError(), "cudaStreamCreate"));
    pl->own_stream = true;
    if (cudaEventCreate(&pl->ev0) != cudaSuccess || cudaEventCreate(&pl->ev1) != cudaSuccess)
        return fail(cuda_err(cudaGetLastError(), "cudaEventCreate"));
    if (generic) {
        int rg = gen_setup(pl);
        if (rg != PM_OK) return fail(rg);
    }
    // twiddle tables
    for (int axis = 0; axis < 2; ++axis) {
        const int lg = axis == 0 ? lgx : lgy;
        const AxisShape& k = axis == 0 ? kset(precision, lg).row : kset(precision, lg).col;
        int r2 = axis == 0 ? upload_twiddles(precision, lg, k.lgR, k.TW, &pl->tw_row, &pl->tw_row_i)
                           : upload_twiddles(precision, lg, k.lgR, k.TW, &pl->tw_col, &pl->tw_col_i);
        if (r2 != PM_OK) return fail(r2);
    }
    {
        const KernelSet& kr = kset(precision, lgx);
        const KernelSet& kc = kset(precision, lgy);
        cudaError_t e3 = allow_smem(kr.row_iter, pl->rc.smem);
        if (e3 == cudaSuccess) e3 = allow_smem(kr.row_fft, pl->rc.smem);
        if (e3 == cudaSuccess) e3 = allow_smem(kr.row_final, pl->rc.smem);
        if (e3 == cudaSuccess) e3 = allow_smem(kc.col_iter, pl->cc.smem);
        if (e3 == cudaSuccess) e3 = allow_smem(kc.col_fft, pl->cc.smem);
        if (e3 != cudaSuccess) return fail(cuda_err(e3, "cudaFuncSetAttribute"));
    }
    {
        // persistent cooperative solve kernel (square grids, n >= 128)
        const KernelSet& ks = kset(precision, lgx);
        int coop = 0, nsm = 0, per_sm = 0;
        cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
        if (n_x == n_y && ks.solve && coop) {
            // one grid size for both algorithms' kernels: the smaller occupancy
            int per_sm_raar = 0;
            cudaError_t e4 = allow_smem(ks.solve, ks.solve_smem);
            if (e4 == cudaSuccess) e4 = allow_smem(ks.solve_raar, ks.solve_smem_raar);
            if (e4 == cudaSuccess)
                e4 = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ks.solve, ks.solve_threads,
                                                                   ks.solve_smem);
            if (e4 == cudaSuccess)
                e4 = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_raar, ks.solve_raar,
                                                                   ks.solve_threads, ks.solve_smem_raar);
            per_sm = std::min(per_sm, per_sm_raar);
            if (e4 == cudaSuccess && per_sm > 0) pl->solve_grid = per_sm * nsm;
            cudaGetLastError();
            if (e4 == cudaSuccess && ks.solve_tma) {
                int a1 = 0, a2 = 0;
                cudaError_t e5 = allow_smem(ks.solve_tma, ks.solve_smem_tma);
                if (e5 == cudaSuccess) e5 = allow_smem(ks.solve_raar_tma, ks.solve_smem_raar_tma);
                if (e5 == cudaSuccess)
                    e5 = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a1, ks.solve_tma, ks.solve_threads,
                                                                       ks.solve_smem_tma);
                if (e5 == cudaSuccess)
                    e5 = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a2, ks.solve_raar_tma, ks.solve_threads,
                                                                       ks.solve_smem_raar_tma);
                if (e5 == cudaSuccess && std::min(a1, a2) > 0) pl->solve_grid_tma = std::min(a1, a2) * nsm;
                cudaGetLastError();
            }
        }
        if (cudaMalloc((void**)&pl->bar, sizeof(GridBar)) != cudaSuccess ||
            cudaMemset(pl->bar, 0, sizeof(GridBar)) != cudaSuccess)
            return fail(cuda_err(cudaGetLastError(), "cudaMalloc(barrier)"));
    }
    int r = ensure_capacity(pl, std::max(1, max_batch), 1);
    if (r != PM_OK) return fail(r);
    *out = pl;
    return PM_OK;
}

int pm_plan_destroy(pm_plan* pl) {
    if (!pl) return PM_OK;
    cudaSetDevice(pl->device);
    if (pl->stream) cudaStreamSynchronize(pl->stream);
    drop_graphs(pl);
    free_buffers(pl);
    if (pl->tw_row_i && pl->tw_row_i != pl->tw_row) cudaFree(pl->tw_row_i);
    if (pl->tw_col_i && pl->tw_col_i != pl->tw_col) cudaFree(pl->tw_col_i);
    if (pl->tw_row) cudaFree(pl->tw_row);
    if (pl->tw_col) cudaFree(pl->tw_col);
    if (pl->gtwx) cudaFree(pl->gtwx);
    if (pl->gtwy) cudaFree(pl->gtwy);
    if (pl->red) cudaFree(pl->red);
    if (pl->bar) cudaFree(pl->bar);
    if (pl->stamps) cudaFree(pl->stamps);
    if (pl->ring_h) cudaFreeHost(pl->ring_h);
    if (pl->hostw_h) cudaFreeHost(pl->hostw_h);
    if (pl->hst) cudaFreeHost(pl->hst);
    if (pl->ev0) cudaEventDestroy(pl->ev0);
    if (pl->ev1) cudaEventDestroy(pl->ev1);
    if (pl->own_stream && pl->stream) cudaStreamDestroy(pl->stream);
    delete pl;
    return PM_OK;
}

int pm_plan_set_stream(pm_plan* pl, void* stream) {
    CKR(check_plan(pl));
    std::lock_guard<std::mutex> lk(pl->mu);
    CK(cudaStreamSynchronize(pl->stream));
    drop_graphs(pl);
    if (stream) {
        if (pl->own_stream) cudaStreamDestroy(pl->stream);
        pl->own_stream = false;
        pl->stream = (cudaStream_t)stream;
    } else if (!pl->own_stream) {
        CK(cudaStreamCreateWithFlags(&pl->stream, cudaStreamNonBlocking));
        pl->own_stream = true;
    }
    return PM_OK;
}

int pm_plan_get_stream(pm_plan* pl, void** stream) {
    if (!pl || !stream) return set_err(PM_ERR_ARG, "null argument");
    *stream = (void*)pl->stream;
    return PM_OK;
}

int pm_plan_synchronize(pm_plan* pl) {
    CKR(check_plan(pl));
    CK(cudaStreamSynchronize(pl->stream));
    return PM_OK;
}

int pm_plan_set_path(pm_plan* pl, int path) {
    if (!pl) return set_err(PM_ERR_ARG, "null plan");
    if (path < 0 || path > 2) return set_err(PM_ERR_ARG, "path must be 0, 1 or 2");
    if (path == 1 && pl->solve_grid == 0)
        return set_err(PM_ERR_UNSUPPORTED, "persistent solve kernel unavailable for this grid/device");
    pl->path = path;
    return PM_OK;
}

int pm_plan_get_path(pm_plan* pl, int* path) {
    if (!pl || !path) return set_err(PM_ERR_ARG, "null argument");
    *path = (pl->path == 2 || pl->solve_grid == 0) ? 2 : 1;
    return PM_OK;
}

int pm_plan_launch_count(pm_plan* pl, long long* count) {
    if (!pl || !count) return set_err(PM_ERR_ARG, "null argument");
    *count = pl->launches;
    return PM_OK;
}

// ----------------------------------------------------------- transforms
int pm_fft2_device(pm_plan* pl, const void* d_in, void* d_out, int direction, int batch) {
    CKR(check_plan(pl));
    if (direction != PM_FORWARD && direction != PM_INVERSE)
        return set_err(PM_ERR_ARG, "direction must be -1 (forward) or +1 (inverse)");
    if (batch < 1) return set_err(PM_ERR_ARG, "batch must be >= 1");
    std::lock_guard<std::mutex> lk(pl->mu);
    return fft2_dev(pl, d_in, d_out, direction, batch);
}

int pm_fft2(pm_plan* pl, const void* in, void* out, int direction, int batch) {
    NvtxRange nvtx_("pm_fft2");
    CKR(check_plan(pl));
    if (direction != PM_FORWARD && direction != PM_INVERSE)
        return set_err(PM_ERR_ARG, "direction must be -1 (forward) or +1 (inverse)");
    if (!in || !out || batch < 1) return set_err(PM_ERR_ARG, "null buffer or batch < 1");
    std::lock_guard<std::mutex> lk(pl->mu);
    CKR(ensure_capacity(pl, batch, 1));
    const size_t bytes = (size_t)batch * pl->N * pl->csz;
    CK(cudaMemcpyAsync(pl->field, in, bytes, cudaMemcpyHostToDevice, pl->stream));
    CKR(fft2_dev(pl, pl->field, pl->field, direction, batch));
    CK(cudaMemcpyAsync(out, pl->field, bytes, cudaMemcpyDeviceToHost, pl->stream));
    CK(cudaStreamSynchronize(pl->stream));
    return PM_OK;
}

// ---------------------------------------------------------- projections
static int replace_dev(pm_plan* pl, const void* in, const void* target, int per_field, double tol,
                       void* out, int batch) {
    const long long n = (long long)pl->N;
    const int blocks = (int)std::min<long long>((n + 255) / 256, 1184);
    if (pl->prec == PM_SINGLE)
        // fp32 decides on |u|^2 against the exact squared threshold (as the solve does)
        replace_kernel<float><<<dim3(blocks, batch), 256, 0, pl->stream>>>(
            (const float2*)in, (const float*)target, per_field ? n : 0, (float)tol, (float2*)out, n);
    else
        replace_kernel<double><<<dim3(blocks, batch), 256, 0, pl->stream>>>(
            (const double2*)in, (const double*)target, per_field ? n : 0, tol, (double2*)out, n);
    CK(cudaGetLastError());
    pl->launches++;
    return PM_OK;
}

int pm_replace_modulus_device(pm_plan* pl, const void* d_in, const void* d_target, int per_field,
                              double zero_tol, void* d_out, int batch) {
    CKR(check_plan(pl));
    if (batch < 1) return set_err(PM_ERR_ARG, "batch must be >= 1");
    std::lock_guard<std::mutex> lk(pl->mu);
    return replace_dev(pl, d_in, d_target, per_field, zero_tol, d_out, batch);
}

int pm_replace_modulus(pm_plan* pl, const void* in, const void* target, int per_field,
                       double zero_tol, void* out, int batch) {
    CKR(check_plan(pl));
    if (!in || !target || !out || batch < 1) return set_err(PM_ERR_ARG, "null buffer or batch < 1");
    std::lock_guard<std::mutex> lk(pl->mu);
    CKR(ensure_capacity(pl, batch, 1));
    const size_t cb = (size_t)batch * pl->N * pl->csz;
    const size_t rb = (size_t)(per_field ? batch : 1) * pl->N * pl->rsz;
    CK(cudaMemcpyAsync(pl->field, in, cb, cudaMemcpyHostToDevice, pl->stream));
    CK(cudaMemcpyAsync(pl->mbuf, target, rb, cudaMemcpyHostToDevice, pl->stream));
    CKR(replace_dev(pl, pl->field, pl->mbuf, per_field, zero_tol, pl->field, batch));
    CK(cudaMemcpyAsync(out, pl->field, cb, cudaMemcpyDeviceToHost, pl->stream));
    CK(cudaStreamSynchronize(pl->stream));
    return PM_OK;
}

// P_M u on the device: rows forward, fused column FFT.replace.IFFT, rows inverse.
static int project_fourier_dev(pm_plan* pl, const void* d_u, const void* d_m, double tol_m, void* d_out) {
    CKR(fft2_dev(pl, d_u, d_out, PM_FORWARD, 1));   // full forward transform
    // columns were already transformed by fft2; replace in the Fourier plane then inverse
    CKR(replace_dev(pl, d_out, d_m, 1, tol_m, d_out, 1));
    CKR(fft2_dev(pl, d_out, d_out, PM_INVERSE, 1));
    return PM_OK;
}

int pm_project_fourier(pm_plan* pl, const void* u, const void* m, double zero_tol_m, void* out) {
    CKR(check_plan(pl));
    if (!u || !m || !out) return set_err(PM_ERR_ARG, "null buffer");
    std::lock_guard<std::mutex> lk(pl->mu);
    CKR(ensure_capacity(pl, 1, 1));
    CK(cudaMemcpyAsync(pl->tmp, u, pl->N * pl->csz, cudaMemcpyHostToDevice, pl->stream));
    CK(cudaMemcpyAsync(pl->mbuf, m, pl->N * pl->rsz, cudaMemcpyHostToDevice, pl->stream));
    CKR(project_fourier_dev(pl, pl->tmp, pl->mbuf, zero_tol_m, pl->field));
    CK(cudaMemcpyAsync(out, pl->field, pl->N * pl->csz, cudaMemcpyDeviceToHost, pl->stream));
    CK(cudaStreamSynchronize(pl->stream));
    return PM_OK;
}


static void reduce_grid(long long n, int* nb, long long* chunk) {
    *nb = (int)std::max<long long>(1, std::min<long long>(1024, (n + 4095) / 4096));
    *chunk = (n + *nb - 1) / *nb;
}

int pm_gap(pm_plan* pl, const void* u, const void* p, const void* m, double zero_tol_p,
           double zero_tol_m, double* out_gap) {
    CKR(check_plan(pl));
    if (!u || !p || !m || !out_gap) return set_err(PM_ERR_ARG, "null buffer");
    std::lock_guard<std::mutex> lk(pl->mu);
    CKR(ensure_capacity(pl, 1, 1));
    const long long n = (long long)pl->N;
    int nb;
    long long chunk;
    reduce_grid(n, &nb, &chunk);
    CKR(ensure_red(pl, nb));
    CK(cudaMemcpyAsync(pl->tmp, u, n * pl->csz, cudaMemcpyHostToDevice, pl->stream));
    CK(cudaMemcpyAsync(pl->pbuf, p, n * pl->rsz, cudaMemcpyHostToDevice, pl->stream));
    CK(cudaMemcpyAsync(pl->mbuf, m, n * pl->rsz, cudaMemcpyHostToDevice, pl->stream));
    CKR(project_fourier_dev(pl, pl->tmp, pl->mbuf, zero_tol_m, pl->field));
    if (pl->prec == PM_SINGLE)
        gap_partial_kernel<float><<<nb, 256, 0, pl->stream>>>((const float2*)pl->tmp, (const float2*)pl->field,
                                                               (const float*)pl->pbuf,
                                                               (float)zero_tol_p, n, chunk,
                                                               pl->red);
    else
        gap_partial_kernel<double><<<nb, 256, 0, pl->stream>>>((const double2*)pl->tmp,
                                                                (const double2*)pl->field,
                                                                (const double*)pl->pbuf, zero_tol_p, n,
                                                                chunk, pl->red);
    final_sum_kernel<<<1, 32, 0, pl->stream>>>(pl->red, nb, pl->red + nb, 1);
    CK(cudaGetLastError());
    pl->launches += 2;
    CK(cudaMemcpyAsync(out_gap, pl->red + nb, sizeof(double), cudaMemcpyDeviceToHost, pl->stream));
    CK(cudaStreamSynchronize(pl->stream));
    return PM_OK;
}

// ----------------------------------------------------------- reductions
int pm_recon_image(pm_plan* pl, const void* u, int batch, const double* target_energy, double log_floor,
                   uint8_t* log_image, double* intensity) {
    CKR(check_plan(pl));
    if (!u || batch < 1) return set_err(PM_ERR_ARG, "null buffer or batch < 1");
    if (log_image && !(log_floor > 0.0)) return set_err(PM_ERR_ARG, "log_floor must be > 0");
    std::lock_guard<std::mutex> lk(pl->mu);
    CKR(ensure_capacity(pl, batch, 1));
    const long long n = (long long)pl->N;
    int nb;
    long long chunk;
    reduce_grid(n, &nb, &chunk);
    CKR(ensure_red(pl, batch * (2 * nb + 2) + batch));
    double* part = pl->red;
    double* sp = pl->red + (size_t)batch * 2 * nb;
    double* en = sp + 2 * batch;
    if (target_energy)
        CK(cudaMemcpyAsync(en, target_energy, batch * sizeof(double), cudaMemcpyHostToDevice, pl->stream));
    CK(cudaMemcpyAsync(pl->field, u, (size_t)batch * n * pl->csz, cudaMemcpyHostToDevice, pl->stream));
    CKR(fft2_dev(pl, pl->field, pl->field, PM_FORWARD, batch));
    uint8_t* dimg = nullptr;
    double* dint = nullptr;
    if (log_image) CK(cudaMalloc((void**)&dimg, (size_t)batch * n));
    if (intensity) {
        cudaError_t e = cudaMalloc((void**)&dint, (size_t)batch * n * sizeof(double));
        if (e != cudaSuccess) {
            cudaFree(dimg);
            return cuda_err(e, "cudaMalloc");
        }
    }
    const int blocks = (int)std::min<long long>((n + 255) / 256, 1184);
    const double lf = std::log10(log_floor > 0.0 ? log_floor : 1.0);
    if (pl->prec == PM_SINGLE) {
        recon_partial_kernel<float><<<dim3(nb, batch), 256, 0, pl->stream>>>((const float2*)pl->field, n, chunk,
                                                                              part, nb);
        recon_final_kernel<<<batch, 32, 0, pl->stream>>>(part, nb, target_energy ? en : nullptr, sp);
        recon_image_kernel<float><<<dim3(blocks, batch), 256, 0, pl->stream>>>(
            (const float2*)pl->field, pl->nx, pl->ny, sp, log_floor, lf, dint, dimg);
    } else {
        recon_partial_kernel<double><<<dim3(nb, batch), 256, 0, pl->stream>>>((const double2*)pl->field, n,
                                                                               chunk, part, nb);
        recon_final_kernel<<<batch, 32, 0, pl->stream>>>(part, nb, target_energy ? en : nullptr, sp);
        recon_image_kernel<double><<<dim3(blocks, batch), 256, 0, pl->stream>>>(
            (const double2*)pl->field, pl->nx, pl->ny, sp, log_floor, lf, dint, dimg);
    }
    cudaError_t e = cudaGetLastError();
    pl->launches += 3;
    std::vector<double> h(2 * batch);
    if (e == cudaSuccess) e = cudaMemcpyAsync(h.data(), sp, 2 * batch * sizeof(double), cudaMemcpyDeviceToHost,
                                              pl->stream);
    if (e == cudaSuccess && log_image)
        e = cudaMemcpyAsync(log_image, dimg, (size_t)batch * n, cudaMemcpyDeviceToHost, pl->stream);
    if (e == cudaSuccess && intensity)
        e = cudaMemcpyAsync(intensity, dint, (size_t)batch * n * sizeof(double), cudaMemcpyDeviceToHost,
                            pl->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(pl->stream);
    cudaFree(dimg);
    cudaFree(dint);
    if (e != cudaSuccess) return cuda_err(e, "pm_recon_image");
    if (target_energy)
        for (int b = 0; b < batch; ++b)
            if (h[2 * b] == 0.0) return set_err(PM_ERR_ARG, "reconstruction carries no energy");
    return PM_OK;
}

int pm_norm2(int device, const void* data, long long count, int dtype, double* out) {
    if (!data || !out || count < 1) return set_err(PM_ERR_ARG, "cannot reduce an empty grid");
    if (dtype < 0 || dtype > 3) return set_err(PM_ERR_ARG, "dtype must be 0..3");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return set_err(PM_ERR_CUDA, "no CUDA device available (phasemask_b200 has no CPU fallback)");
    }
    CK(cudaSetDevice(device));
    static const size_t esz[4] = {4, 8, 8, 16};
    const size_t bytes = count * esz[dtype];
    int nb;
    long long chunk;
    reduce_grid(count, &nb, &chunk);
    void* d = nullptr;
    double* part = nullptr;
    CK(cudaMalloc(&d, bytes));
    cudaError_t e = cudaMalloc((void**)&part, (nb + 1) * sizeof(double));
    if (e != cudaSuccess) {
        cudaFree(d);
        return cuda_err(e, "cudaMalloc");
    }
    e = cudaMemcpy(d, data, bytes, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        switch (dtype) {
            case 0: norm_partial_kernel<float><<<nb, 256>>>((const float*)d, count, chunk, part); break;
            case 1: norm_partial_kernel<double><<<nb, 256>>>((const double*)d, count, chunk, part); break;
            case 2: norm_partial_kernel<float2><<<nb, 256>>>((const float2*)d, count, chunk, part); break;
            default: norm_partial_kernel<double2><<<nb, 256>>>((const double2*)d, count, chunk, part); break;
        }
        final_sum_kernel<<<1, 32>>>(part, nb, part + nb, 1);
        e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaMemcpy(out, part + nb, sizeof(double), cudaMemcpyDeviceToHost);
    }
    cudaFree(d);
    cudaFree(part);
    if (e != cudaSuccess) return cuda_err(e, "pm_norm2");
    return PM_OK;
}

int pm_sum(int device, const double* data, long long count, double* out) {
    if (!data || !out || count < 1) return set_err(PM_ERR_ARG, "cannot reduce an empty grid");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return set_err(PM_ERR_CUDA, "no CUDA device available (phasemask_b200 has no CPU fallback)");
    }
    CK(cudaSetDevice(device));
    int nb;
    long long chunk;
    reduce_grid(count, &nb, &chunk);
    double *d = nullptr, *part = nullptr;
    CK(cudaMalloc((void**)&d, count * sizeof(double)));
    cudaError_t e = cudaMalloc((void**)&part, (nb + 1) * sizeof(double));
    if (e != cudaSuccess) {
        cudaFree(d);
        return cuda_err(e, "cudaMalloc");
    }
    e = cudaMemcpy(d, data, count * sizeof(double), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        sum_partial_kernel<<<nb, 256>>>(d, count, chunk, part);
        final_sum_kernel<<<1, 32>>>(part, nb, part + nb, 0);
        e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaMemcpy(out, part + nb, sizeof(double), cudaMemcpyDeviceToHost);
    }
    cudaFree(d);
    cudaFree(part);
    if (e != cudaSuccess) return cuda_err(e, "pm_sum");
    return PM_OK;
}

int pm_random_start(int device, const void* m, long long count, int batch, int precision,
                    const unsigned long long rng[4], void* out) {
    if (!m || !out || !rng || count < 1 || batch < 1) return set_err(PM_ERR_ARG, "empty input");
    if (precision != PM_SINGLE && precision != PM_DOUBLE) return set_err(PM_ERR_ARG, "bad precision");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return set_err(PM_ERR_CUDA, "no CUDA device available (phasemask_b200 has no CPU fallback)");
    }
    CK(cudaSetDevice(device));
    const size_t rsz = precision == PM_SINGLE ? 4 : 8, total = (size_t)count * batch;
    void *dm = nullptr, *dout = nullptr;
    CK(cudaMalloc(&dm, total * rsz));
    cudaError_t e = cudaMalloc(&dout, total * 2 * rsz);
    if (e != cudaSuccess) {
        cudaFree(dm);
        return cuda_err(e, "cudaMalloc");
    }
    int rc = PM_OK;
    e = cudaMemcpy(dm, m, total * rsz, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        rc = enqueue_random_start(precision, dm, dout, count, batch, rng, 0);
        if (rc == PM_OK) e = cudaMemcpy(out, dout, total * 2 * rsz, cudaMemcpyDeviceToHost);
    }
    cudaFree(dm);
    cudaFree(dout);
    if (rc != PM_OK) return rc;
    if (e != cudaSuccess) return cuda_err(e, "pm_random_start");
    return PM_OK;
}

int pm_naive_dft(int device, const void* in, int n_x, int n_y, int direction, void* out) {
    if (!in || !out || n_x < 1 || n_y < 1) return set_err(PM_ERR_ARG, "empty input");
    if ((long long)n_x * n_y > 4096)
        return set_err(PM_ERR_ARG, "grid with " + std::to_string((long long)n_x * n_y) +
                                       " pixels too large for the O(N^2) oracle (limit 4096)");
    if (direction != PM_FORWARD && direction != PM_INVERSE) return set_err(PM_ERR_ARG, "unknown direction");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return set_err(PM_ERR_CUDA, "no CUDA device available (phasemask_b200 has no CPU fallback)");
    }
    CK(cudaSetDevice(device));
    const size_t bytes = (size_t)n_x * n_y * sizeof(double2);
    void* d = nullptr;
    CK(cudaMalloc(&d, 2 * bytes));
    double2* din = (double2*)d;
    double2* dout = din + (size_t)n_x * n_y;
    cudaError_t e = cudaMemcpy(din, in, bytes, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        naive_dft_kernel<<<(n_x * n_y + 127) / 128, 128>>>(din, n_x, n_y, direction == PM_FORWARD ? -1.0 : 1.0,
                                                           dout);
        e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaMemcpy(out, dout, bytes, cudaMemcpyDeviceToHost);
    }
    cudaFree(d);
    if (e != cudaSuccess) return cuda_err(e, "pm_naive_dft");
    return PM_OK;
}

int pm_phases(int device, const void* u, long long count, int precision, double zero_tol, double* out) {
    if (!u || !out || count < 1) return set_err(PM_ERR_ARG, "empty input");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return set_err(PM_ERR_CUDA, "no CUDA device available (phasemask_b200 has no CPU fallback)");
    }
    CK(cudaSetDevice(device));
    const size_t csz = precision == PM_SINGLE ? 8 : 16;
    void* d = nullptr;
    double* o = nullptr;
    CK(cudaMalloc(&d, count * csz));
    cudaError_t e = cudaMalloc((void**)&o, count * sizeof(double));
    if (e != cudaSuccess) {
        cudaFree(d);
        return cuda_err(e, "cudaMalloc");
    }
    e = cudaMemcpy(d, u, count * csz, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        const int blocks = (int)std::min<long long>((count + 255) / 256, 1184);
        if (precision == PM_SINGLE)
            phases_kernel<float><<<blocks, 256>>>((const float2*)d, count, (float)zero_tol, o);
        else
            phases_kernel<double><<<blocks, 256>>>((const double2*)d, count, zero_tol, o);
        e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaMemcpy(out, o, count * sizeof(double), cudaMemcpyDeviceToHost);
    }
    cudaFree(d);
    cudaFree(o);
    if (e != cudaSuccess) return cuda_err(e, "pm_phases");
    return PM_OK;
}

// ---------------------------------------------------------------- solve
static int solve_enqueue(pm_plan* pl, const void* d_p, const void* d_m, const void* d_init, int batch,
                         const pm_params* prm, const double* tol_p, const double* tol_m,
                         const double* energy, pm_result* res, bool host_io, int ring = 0, int lockstep = 0) {
    if (!tol_p != !tol_m) return set_err(PM_ERR_ARG, "tolerance arrays: pass both or neither");
    trace("solve: enter");
    CKR(session_setup(pl, d_p, d_m, batch, prm, tol_p, tol_m, energy));
    trace("session_setup");
    auto& s = pl->s;
    s.ring = ring != 0;
    s.lockstep = ring && lockstep;
    CKR(stage_start(pl, d_init, host_io ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice));
    if (host_io) {
        CKR(ensure_outputs(pl, res && res->phases, res && res->levels, res && res->u_star, res && res->v_star));
        s.phases = (res && res->phases) ? pl->phases : nullptr;
        s.levels = (res && res->levels) ? pl->levels : nullptr;
        s.ustar = (res && res->u_star) ? pl->ustar : nullptr;
        s.vstar = (res && res->v_star) ? pl->vstar : nullptr;
    } else {
        s.phases = res ? res->phases : nullptr;
        s.levels = res ? res->levels : nullptr;
        s.ustar = res ? res->u_star : nullptr;
        s.vstar = res ? res->v_star : nullptr;
    }
    trace("outputs");
    CK(cudaEventRecord(pl->ev0, pl->stream));
    CKR(enqueue_full_solve(pl));
    CK(cudaEventRecord(pl->ev1, pl->stream));
    trace("enqueue_full_solve");
    return PM_OK;
}

// Outputs of an enqueued solve: host copies, records, state, the reference's errors.
static int solve_collect(pm_plan* pl, pm_result* res, bool host_io) {
    auto& s = pl->s;
    const size_t N = pl->N;
    const int batch = s.batch;
    const pm_params* prm = &s.prm;
    if (host_io && res) {
        if (res->phases)
            CK(cudaMemcpyAsync(res->phases, pl->phases, batch * N * sizeof(double), cudaMemcpyDeviceToHost,
                               pl->stream));
        if (res->levels)
            CK(cudaMemcpyAsync(res->levels, pl->levels, batch * N, cudaMemcpyDeviceToHost, pl->stream));
        if (res->u_star)
            CK(cudaMemcpyAsync(res->u_star, pl->ustar, batch * N * pl->csz, cudaMemcpyDeviceToHost, pl->stream));
        if (res->v_star)
            CK(cudaMemcpyAsync(res->v_star, pl->vstar, batch * N * pl->csz, cudaMemcpyDeviceToHost, pl->stream));
    }
    trace("D2H enqueued");
    std::vector<int> iters(batch), div(batch);
    int zero = 0, pair_bad = 0;
    CKR(read_records(pl, 1, prm->max_iters, res ? res->gap : nullptr, res ? res->err_lit : nullptr,
                     res ? res->err_dark : nullptr, iters.data(), div.data(), nullptr, &zero, &pair_bad));
    trace("read_records (synchronised)");
    if (res) {
        if (res->iters_run) std::copy(iters.begin(), iters.end(), res->iters_run);
        if (res->diverged_iter) std::copy(div.begin(), div.end(), res->diverged_iter);
        if (res->device_ms) CK(cudaEventElapsedTime(res->device_ms, pl->ev0, pl->ev1));
    }
    s.active = false;
    s.ring = s.lockstep = false;
    CKR(zero_error(zero));
    if (any_diverged(div)) return set_err(PM_ERR_DIVERGED, "non-finite values during the iteration");
    if (pair_bad) return set_err(PM_ERR_ARG, "field contains non-finite entries");
    return PM_OK;
}

static int solve_core(pm_plan* pl, const void* d_p, const void* d_m, const void* d_init, int batch,
                      const pm_params* prm, const double* tol_p, const double* tol_m,
                      const double* energy, pm_result* res, bool host_io) {
    CKR(solve_enqueue(pl, d_p, d_m, d_init, batch, prm, tol_p, tol_m, energy, res, host_io));
    return solve_collect(pl, res, host_io);
}

int pm_solve(pm_plan* pl, const void* p, const void* m, const void* m_init, int batch,
             const pm_params* prm, const double* tol_p, const double* tol_m, const double* energy,
             pm_result* res) {
    NvtxRange nvtx_("pm_solve");
    CKR(check_plan(pl));
    if (!p || !m) return set_err(PM_ERR_ARG, "null p or m");
    CKR(validate_params(prm, batch));
    std::lock_guard<std::mutex> lk(pl->mu);
    CKR(ensure_capacity(pl, batch, prm->max_iters));
    const size_t N = pl->N;
    static const bool tr = getenv("PM_TRACE") != nullptr;
    cudaEvent_t ea = nullptr, ed = nullptr;
    if (tr) {
        cudaEventCreate(&ea);
        cudaEventCreate(&ed);
        cudaEventRecord(ea, pl->stream);
        trace("pm_solve: before uploads");
    }
    CK(cudaMemcpyAsync(pl->pbuf, p, (prm->p_per_mask ? batch : 1) * N * pl->rsz, cudaMemcpyHostToDevice,
                       pl->stream));
    CK(cudaMemcpyAsync(pl->mbuf, m, batch * N * pl->rsz, cudaMemcpyHostToDevice, pl->stream));
    if (tr) trace("pm_solve: uploads enqueued");
    cudaEvent_t eb = nullptr;
    if (tr) {
        cudaEventCreate(&eb);
        cudaEventRecord(eb, pl->stream);
    }
    const int rc = solve_core(pl, pl->pbuf, pl->mbuf, m_init, batch, prm, tol_p, tol_m, energy, res, true);
    if (tr) {
        cudaEventRecord(ed, pl->stream);
        cudaEventSynchronize(ed);
        float a = 0, b = 0, c = 0, h = 0;
        cudaEventElapsedTime(&h, ea, eb);
        fprintf(stderr, "[pm] p, m uploads alone %.3f ms\n", h);
        cudaEventDestroy(eb);
        cudaEventElapsedTime(&a, ea, pl->ev0);
        cudaEventElapsedTime(&b, pl->ev0, pl->ev1);
        cudaEventElapsedTime(&c, pl->ev1, ed);
        fprintf(stderr, "[pm] device timeline: uploads %.3f ms, solve %.3f ms, downloads + records %.3f ms\n", a, b, c);
        cudaEventDestroy(ea);
        cudaEventDestroy(ed);
    }
    return rc;
}

int pm_solve_device(pm_plan* pl, const void* d_p, const void* d_m, const void* d_m_init, int batch,
                    const pm_params* prm, const double* tol_p, const double* tol_m, const double* energy,
                    pm_result* res) {
    NvtxRange nvtx_("pm_solve_device");
    CKR(check_plan(pl));
    if (!d_p || !d_m) return set_err(PM_ERR_ARG, "null p or m");
    std::lock_guard<std::mutex> lk(pl->mu);
    return solve_core(pl, d_p, d_m, d_m_init, batch, prm, tol_p, tol_m, energy, res, false);
}

static_assert(sizeof(RingSlot) == sizeof(pm_record) && offsetof(RingSlot, flags) == offsetof(pm_record, flags),
              "pm_record mirrors the device's RingSlot");
static_assert(kRecPublished == PM_REC_PUBLISHED && kRecRecorded == PM_REC_RECORDED && kRecEarly == PM_REC_EARLY &&
                  kRecDiverged == PM_REC_DIVERGED && kRecStop == PM_REC_STOP && kRecAborted == PM_REC_ABORTED &&
                  kRecTimeout == PM_REC_TIMEOUT,
              "record flags");

int pm_solve_async(pm_plan* pl, const void* p, const void* m, const void* m_init, const pm_params* prm,
                   const double* tol_p, const double* tol_m, const double* energy, int lockstep,
                   pm_result* res) {
    NvtxRange nvtx_("pm_solve_async");
    CKR(check_plan(pl));
    if (!p || !m) return set_err(PM_ERR_ARG, "null p or m");
    CKR(validate_params(prm, 1));
    std::lock_guard<std::mutex> lk(pl->mu);
    CKR(ensure_capacity(pl, 1, prm->max_iters));
    const int K = prm->max_iters;
    if (pl->ring_cap < K) {
        // mapped host memory, written by the device and polled by pm_solve_next
        CK(cudaStreamSynchronize(pl->stream));
        drop_graphs(pl);                       // captured solves hold the old ring's address
        if (pl->ring_h) cudaFreeHost(pl->ring_h);
        pl->ring_h = nullptr;
        pl->ring_cap = 0;
        CK(cudaHostAlloc((void**)&pl->ring_h, (size_t)K * sizeof(RingSlot), cudaHostAllocMapped));
        CK(cudaHostGetDevicePointer((void**)&pl->ring_d, pl->ring_h, 0));
        if (!pl->hostw_h) {
            CK(cudaHostAlloc((void**)&pl->hostw_h, 2 * sizeof(int), cudaHostAllocMapped));
            CK(cudaHostGetDevicePointer((void**)&pl->hostw_d, pl->hostw_h, 0));
        }
        pl->ring_cap = K;
    }
    CK(cudaStreamSynchronize(pl->stream));     // the previous solve no longer reads the ring
    std::memset(pl->ring_h, 0, (size_t)K * sizeof(RingSlot));
    ((volatile int*)pl->hostw_h)[0] = 0;
    ((volatile int*)pl->hostw_h)[1] = 0;
    const size_t N = pl->N;
    CK(cudaMemcpyAsync(pl->pbuf, p, N * pl->rsz, cudaMemcpyHostToDevice, pl->stream));
    CK(cudaMemcpyAsync(pl->mbuf, m, N * pl->rsz, cudaMemcpyHostToDevice, pl->stream));
    return solve_enqueue(pl, pl->pbuf, pl->mbuf, m_init, 1, prm, tol_p, tol_m, energy, res, true, 1, lockstep);
}

int pm_solve_next(pm_plan* pl, int iter, pm_record* out) {
    CKR(check_plan(pl));
    if (!out) return set_err(PM_ERR_ARG, "null record");
    const auto& s = pl->s;
    if (!s.active || !s.ring) return set_err(PM_ERR_ARG, "no streamed solve in progress (pm_solve_async)");
    if (iter < 1 || iter > s.prm.max_iters) return set_err(PM_ERR_ARG, "iteration out of range");
    volatile RingSlot* r = (volatile RingSlot*)pl->ring_h + (iter - 1);
    for (unsigned spin = 0;; ++spin) {
        if (r->flags & kRecPublished) break;
        if ((spin & 1023) == 1023) {
            const cudaError_t e = cudaStreamQuery(pl->stream);
            if (e != cudaErrorNotReady) {
                if (r->flags & kRecPublished) break;
                out->flags = 0;                  // the solve ended before this iteration
                if (e != cudaSuccess) return cuda_err(e, "streamed solve");
                return PM_OK;
            }
        }
#if defined(__x86_64__)
        __builtin_ia32_pause();
#endif
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    out->gap = r->gap;
    out->err_lit = r->err_lit;
    out->err_dark = r->err_dark;
    out->iter = r->iter;
    out->flags = r->flags;
    return PM_OK;
}

int pm_solve_answer(pm_plan* pl, int iter, int abort) {
    CKR(check_plan(pl));
    if (!pl->s.active || !pl->s.lockstep) return set_err(PM_ERR_ARG, "no lockstep solve in progress");
    volatile int* w = (volatile int*)pl->hostw_h;
    if (abort) w[1] = 1;
    else w[0] = iter;
    return PM_OK;
}

int pm_solve_wait(pm_plan* pl, pm_result* res) {
    NvtxRange nvtx_("pm_solve_wait");
    CKR(check_plan(pl));
    std::lock_guard<std::mutex> lk(pl->mu);
    if (!pl->s.active || !pl->s.ring) return set_err(PM_ERR_ARG, "no streamed solve in progress (pm_solve_async)");
    return solve_collect(pl, res, true);
}

int pm_solve_begin(pm_plan* pl, const void* p, const void* m, const void* m_init, int batch,
                   const pm_params* prm, const double* tol_p, const double* tol_m, const double* energy) {
    CKR(check_plan(pl));
    if (!p || !m || !tol_p != !tol_m) return set_err(PM_ERR_ARG, "null input");
    CKR(validate_params(prm, batch));
    std::lock_guard<std::mutex> lk(pl->mu);
    CKR(ensure_capacity(pl, batch, prm->max_iters));
    const size_t N = pl->N;
    CK(cudaMemcpyAsync(pl->pbuf, p, (prm->p_per_mask ? batch : 1) * N * pl->rsz, cudaMemcpyHostToDevice,
                       pl->stream));
    CK(cudaMemcpyAsync(pl->mbuf, m, batch * N * pl->rsz, cudaMemcpyHostToDevice, pl->stream));
    CKR(session_setup(pl, pl->pbuf, pl->mbuf, batch, prm, tol_p, tol_m, energy));
    pl->s.stepping = true;
    CKR(stage_start(pl, m_init, cudaMemcpyHostToDevice));
    CK(cudaEventRecord(pl->ev0, pl->stream));
    CKR(enqueue_begin(pl));
    CK(cudaStreamSynchronize(pl->stream));
    return PM_OK;
}

int pm_solve_step(pm_plan* pl, int n_iters, int* all_stopped) {
    CKR(check_plan(pl));
    std::lock_guard<std::mutex> lk(pl->mu);
    if (!pl->s.active) return set_err(PM_ERR_ARG, "no solve in progress (call pm_solve_begin)");
    CKR(enqueue_steps(pl, n_iters, true));
    std::vector<MaskState> st(pl->s.batch);
    CK(cudaMemcpyAsync(st.data(), pl->st, st.size() * sizeof(MaskState), cudaMemcpyDeviceToHost, pl->stream));
    CK(cudaStreamSynchronize(pl->stream));
    int all = 1;
    for (auto& x : st) all &= (x.stop || x.done) ? 1 : 0;
    if (all_stopped) *all_stopped = all;
    return PM_OK;
}

int pm_solve_records(pm_plan* pl, int first_iter, int last_iter, double* gap, double* err_lit,
                     double* err_dark, int* iters_run, int* diverged_iter) {
    CKR(check_plan(pl));
    std::lock_guard<std::mutex> lk(pl->mu);
    if (pl->s.batch < 1) return set_err(PM_ERR_ARG, "no solve in progress");
    return read_records(pl, std::max(1, first_iter), last_iter, gap, err_lit, err_dark, iters_run,
                        diverged_iter);
}

int pm_solve_finish(pm_plan* pl, int abort, pm_result* res) {
    CKR(check_plan(pl));
    std::lock_guard<std::mutex> lk(pl->mu);
    auto& s = pl->s;
    if (!s.active) return set_err(PM_ERR_ARG, "no solve in progress (call pm_solve_begin)");
    const size_t N = pl->N;
    const int batch = s.batch;
    CKR(ensure_outputs(pl, res && res->phases, res && res->levels, res && res->u_star, res && res->v_star));
    s.phases = (res && res->phases) ? pl->phases : nullptr;
    s.levels = (res && res->levels) ? pl->levels : nullptr;
    s.ustar = (res && res->u_star) ? pl->ustar : nullptr;
    s.vstar = (res && res->v_star) ? pl->vstar : nullptr;
    if (abort) {
        force_stop_kernel<<<(batch + 127) / 128, 128, 0, pl->stream>>>(pl->st, batch, s.it);
        CK(cudaGetLastError());
    }
    CKR(enqueue_finish(pl));
    CK(cudaEventRecord(pl->ev1, pl->stream));
    if (res) {
        if (res->phases)
            CK(cudaMemcpyAsync(res->phases, pl->phases, batch * N * sizeof(double), cudaMemcpyDeviceToHost,
                               pl->stream));
        if (res->levels)
            CK(cudaMemcpyAsync(res->levels, pl->levels, batch * N, cudaMemcpyDeviceToHost, pl->stream));
        if (res->u_star)
            CK(cudaMemcpyAsync(res->u_star, pl->ustar, batch * N * pl->csz, cudaMemcpyDeviceToHost, pl->stream));
        if (res->v_star)
            CK(cudaMemcpyAsync(res->v_star, pl->vstar, batch * N * pl->csz, cudaMemcpyDeviceToHost, pl->stream));
    }
    std::vector<int> iters(batch), div(batch);
    int zero = 0, pair_bad = 0;
    CKR(read_records(pl, 1, s.prm.max_iters, res ? res->gap : nullptr, res ? res->err_lit : nullptr,
                     res ? res->err_dark : nullptr, iters.data(), div.data(), nullptr, &zero, &pair_bad));
    if (res) {
        if (res->iters_run) std::copy(iters.begin(), iters.end(), res->iters_run);
        if (res->diverged_iter) std::copy(div.begin(), div.end(), res->diverged_iter);
        if (res->device_ms) CK(cudaEventElapsedTime(res->device_ms, pl->ev0, pl->ev1));
    }
    s.active = false;
    CKR(zero_error(zero));
    if (any_diverged(div)) return set_err(PM_ERR_DIVERGED, "non-finite values during the iteration");
    if (pair_bad) return set_err(PM_ERR_ARG, "field contains non-finite entries");
    return PM_OK;
}

// ---------------------------------------------------------- measurement
int pm_time_sweep(pm_plan* pl, int which, int batch, int reps, float* avg_ms) {
    CKR(check_plan(pl));
    if (!avg_ms || reps < 1 || batch < 1) return set_err(PM_ERR_ARG, "bad arguments");
    if (pl->generic) return set_err(PM_ERR_UNSUPPORTED, "sweep timing exists for power-of-two grids only");
    std::lock_guard<std::mutex> lk(pl->mu);
    auto& s = pl->s;
    if (!s.p || !s.m || batch > pl->cap) return set_err(PM_ERR_ARG, "run a solve on this plan first");
    const int saved_batch = s.batch;
    s.batch = batch;
    s.phases = s.levels = s.ustar = s.vstar = nullptr;
    CK(cudaMemsetAsync(pl->st, 0, batch * sizeof(MaskState), pl->stream));
    // one warm-up launch, then `reps` timed launches of the steady-state sweep
    // (column sweeps include the full metric reduction of a recorded iteration)
    const int big = 1 << 30;
    pm_params saved = s.prm;
    s.prm.max_iters = big;
    s.prm.record_every = 1;
    s.prm.algorithm = PM_ALGO_GS;
    s.prm.early_stop_tol = -1.0;
    int r = PM_OK;
    for (int i = 0; i <= reps && r == PM_OK; ++i) {
        if (i == 1) CK(cudaEventRecord(pl->ev0, pl->stream));
        r = which == 0 ? row(pl, batch, kRowGS, 1) : col(pl, batch, 2, 1);
    }
    s.prm = saved;
    s.batch = saved_batch;
    CKR(r);
    CK(cudaEventRecord(pl->ev1, pl->stream));
    CK(cudaEventSynchronize(pl->ev1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, pl->ev0, pl->ev1));
    *avg_ms = ms / reps;
    return PM_OK;
}

int pm_debug_phase_stamps(pm_plan* pl, int enable, unsigned long long* out, int n) {
    CKR(check_plan(pl));
    if (enable) {
        const size_t n_st = (size_t)std::max(pl->solve_grid, 1) * 1024;   // fits PM_FINE rows
        if (!pl->stamps) CK(cudaMalloc((void**)&pl->stamps, n_st * sizeof(unsigned long long)));
        CK(cudaMemset(pl->stamps, 0, n_st * sizeof(unsigned long long)));
        return PM_OK;
    }
    if (out && pl->stamps) {
        CK(cudaStreamSynchronize(pl->stream));
        const size_t n_st = (size_t)std::max(pl->solve_grid, 1) * 1024;   // fits PM_FINE rows
        CK(cudaMemcpy(out, pl->stamps, std::min<size_t>(n, n_st) * sizeof(unsigned long long),
                      cudaMemcpyDeviceToHost));
    }
    return PM_OK;
}

int pm_measure_copy(int device, long long bytes, int reps, double* gbs) {
    if (!gbs || bytes < 16 || reps < 1) return set_err(PM_ERR_ARG, "bad arguments");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return set_err(PM_ERR_CUDA, "no CUDA device available");
    }
    CK(cudaSetDevice(device));
    const long long n4 = bytes / 16;
    float4 *a = nullptr, *b = nullptr;
    CK(cudaMalloc((void**)&a, n4 * 16));
    cudaError_t e = cudaMalloc((void**)&b, n4 * 16);
    if (e != cudaSuccess) {
        cudaFree(a);
        return cuda_err(e, "cudaMalloc");
    }
    cudaMemset(a, 0, n4 * 16);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
    const int blocks = nsm * 8;
    float best = 1e30f;
    for (int i = 0; i < reps + 2; ++i) {
        cudaEventRecord(e0);
        copy_kernel<<<blocks, 256>>>(a, b, n4);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (i >= 2) best = std::min(best, ms);
    }
    e = cudaGetLastError();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(a);
    cudaFree(b);
    if (e != cudaSuccess) return cuda_err(e, "copy_kernel");
    *gbs = 2.0 * n4 * 16 / (best * 1e-3) / 1e9;
    return PM_OK;
}

int pm_host_alloc(long long bytes, void** out) {
    if (!out || bytes < 0) return set_err(PM_ERR_ARG, "bad arguments");
    *out = nullptr;
    cudaError_t e = cudaHostAlloc(out, (size_t)std::max(bytes, 1LL), cudaHostAllocPortable);
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        return set_err(PM_ERR_NOMEM, "cudaHostAlloc: out of page-locked memory");
    }
    CK(e);
    return PM_OK;
}

int pm_host_free(void* p) {
    if (p) CK(cudaFreeHost(p));
    return PM_OK;
}

int pm_measure_l2(int device, long long bytes, int passes, int mode, double* gbs) {
    if (!gbs || bytes < 16 || passes < 1 || (mode != 0 && mode != 1)) return set_err(PM_ERR_ARG, "bad arguments");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return set_err(PM_ERR_CUDA, "no CUDA device available");
    }
    CK(cudaSetDevice(device));
    const long long n4 = bytes / 16;
    float4 *a = nullptr, *b = nullptr;
    float* sink = nullptr;
    CK(cudaMalloc((void**)&a, n4 * 16));
    cudaError_t e = cudaMalloc((void**)&b, n4 * 16);
    if (e == cudaSuccess) e = cudaMalloc((void**)&sink, 16);
    if (e != cudaSuccess) {
        cudaFree(a);
        cudaFree(b);
        return cuda_err(e, "cudaMalloc");
    }
    cudaMemset(a, 0, n4 * 16);
    cudaMemset(b, 0, n4 * 16);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
    float best = 1e30f;
    for (int i = 0; i < 5; ++i) {
        cudaEventRecord(e0);
        l2_kernel<<<nsm * 4, 512>>>(a, b, n4, passes, mode, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (i >= 1) best = std::min(best, ms);    // the first launch brings the buffers into L2
    }
    e = cudaGetLastError();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(a);
    cudaFree(b);
    cudaFree(sink);
    if (e != cudaSuccess) return cuda_err(e, "l2_kernel");
    *gbs = (mode ? 2.0 : 1.0) * n4 * 16 * passes / (best * 1e-3) / 1e9;
    return PM_OK;
}

}  // extern "C"
