// Seeded random-phase start on the device: the reference
// draws phi = rng.uniform(0, 2 pi, shape) from np.random.default_rng(seed)
// and starts from m e^{i phi} (src/solver.py:100-103). numpy's default
// generator is PCG64 -- a 128-bit LCG, state' = state * A + inc, whose 64-bit
// output is the XSL-RR permutation of the stepped state
// (numpy/random/src/pcg64/pcg64.h: pcg_setseq_128_step_r,
// pcg_output_xsl_rr_128_64) -- and a double is (x >> 11) * 2^-53
// (numpy/random/_common: next_double). The host hands over the generator's
// state after seeding (bit_generator.state: SeedSequence hashing stays on
// the host); every thread jumps the LCG to its first element in O(log n)
// (Brown, "Random number generation with arbitrary strides", 1994) and then
// strides through its elements with one 128-bit multiply-add each, so the
// draws are exactly numpy's, element for element.
#pragma once
#include "pm_fft.cuh"

namespace pm {

typedef unsigned __int128 u128;

constexpr unsigned long long kPcgMultHi = 2549297995355413924ULL;
constexpr unsigned long long kPcgMultLo = 4865540595714422341ULL;

__host__ __device__ inline u128 u128_of(unsigned long long hi, unsigned long long lo) {
    return ((u128)hi << 64) | (u128)lo;
}

// The affine map (mult, plus) of `delta` LCG steps: state -> state*mult + plus.
struct PcgJump {
    u128 mult, plus;
};
__host__ __device__ inline PcgJump pcg_jump(u128 inc, unsigned long long delta) {
    u128 cur_mult = u128_of(kPcgMultHi, kPcgMultLo), cur_plus = inc;
    u128 acc_mult = 1, acc_plus = 0;
    while (delta > 0) {
        if (delta & 1) {
            acc_mult *= cur_mult;
            acc_plus = acc_plus * cur_mult + cur_plus;
        }
        cur_plus = (cur_mult + 1) * cur_plus;
        cur_mult *= cur_mult;
        delta >>= 1;
    }
    return {acc_mult, acc_plus};
}

__device__ __forceinline__ unsigned long long pcg_output(u128 state) {
    const unsigned long long hi = (unsigned long long)(state >> 64), lo = (unsigned long long)state;
    const unsigned long long x = hi ^ lo;
    const unsigned r = (unsigned)(hi >> 58);
    return (x >> r) | (x << ((64u - r) & 63u));
}

// out[b][i] = m[b][i] e^{i phi_i} for every mask b (one draw per pixel,
// shared by the masks: each reference solve re-seeds with the same seed),
// formed in fp64 like numpy's complex128 product, then cast to T.
template <typename T>
__global__ void random_start_kernel(const T* m, cx<T>* out, long long n, int batch, unsigned long long st_hi,
                                    unsigned long long st_lo, unsigned long long inc_hi, unsigned long long inc_lo,
                                    unsigned long long sm_hi, unsigned long long sm_lo, unsigned long long sp_hi,
                                    unsigned long long sp_lo) {
    const long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i0 >= n) return;
    const long long stride = (long long)gridDim.x * blockDim.x;
    const PcgJump first = pcg_jump(u128_of(inc_hi, inc_lo), (unsigned long long)i0 + 1);
    u128 state = u128_of(st_hi, st_lo) * first.mult + first.plus;
    const u128 smul = u128_of(sm_hi, sm_lo), splus = u128_of(sp_hi, sp_lo);
    for (long long i = i0; i < n; i += stride) {
        const double d = (double)(pcg_output(state) >> 11) * (1.0 / 9007199254740992.0);
        const double phi = 6.283185307179586 * d;            // 0.0 + (2 pi - 0.0) * d
        double s, c;
        sincos(phi, &s, &c);
        for (int b = 0; b < batch; ++b) {
            const double mm = (double)m[b * n + i];
            out[b * n + i] = mk<T>(T(mm * c), T(mm * s));
        }
        state = state * smul + splus;
    }
}

}  // namespace pm
