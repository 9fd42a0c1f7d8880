// Load patterns of the two sweeps of a 1024^2 complex64 field held in L2
// (148 CTAs x 256 threads, one 8-row / 8-column block per CTA), clock64 per
// CTA: how long until every thread holds its 32 values in the FFT's cyclic
// layout (thread j of warp g: element j + 32 k of its line).
//   M1 row-major rows, warp per row, LDG.64 (the row sweep today)
//   M2 row-major [1024][8] column block, thread (c, j) = (tid % 8, tid / 8) (the column sweep today)
//   M3 8x8-tiled field, row stripe: 64 KB contiguous, cooperative LDG.128 -> STS -> warp per row LDS
//   M4 8x8-tiled field, column stripe: 128 runs of 512 B, cooperative LDG.128 -> STS -> warp per column LDS
#include <cstdio>
#include <cuda_runtime.h>

constexpr int L = 1024;
__device__ __forceinline__ float2 ldcg(const float2* p) { return __ldcg(p); }

template <int M>
__global__ void __launch_bounds__(256, 1) k(const float2* __restrict__ f, float* out, long long* cyc) {
    extern __shared__ float4 sm4[];
    float2* sm = reinterpret_cast<float2*>(sm4);
    const int blk = blockIdx.x;
    if (blk >= 128) return;
    const int w = threadIdx.x >> 5, j = threadIdx.x & 31;
    float2 v[32];
    __syncthreads();
    long long t0 = clock64();
    if (M == 1) {
        const float2* row = f + (size_t)(blk * 8 + w) * L;
#pragma unroll
        for (int q = 0; q < 32; ++q) v[q] = ldcg(row + j + 32 * q);
    } else if (M == 2) {
        const int c = threadIdx.x & 7, jj = threadIdx.x >> 3;
        const float2* col = f + blk * 8 + c;
#pragma unroll
        for (int q = 0; q < 32; ++q) v[q] = ldcg(col + (size_t)(jj + 32 * q) * L);
    } else {
        // stage: 64 KB as 4096 float4 chunks; tiled layout: tile (rb, cb) of 8x8 at ((rb * 128 + cb) * 64)
        const float4* src4;
        // M3: stripe rb = blk, tiles cb = 0..127 contiguous; M4: column block cb = blk, tiles rb = 0..127 (stride 128 tiles)
#pragma unroll 4
        for (int i = threadIdx.x; i < 4096; i += 256) {
            const int tile = i >> 5, within = i & 31;            // 32 float4 per 512-B tile
            size_t toff = M == 3 ? ((size_t)blk * 128 + tile) * 64 : ((size_t)tile * 128 + blk) * 64;
            src4 = reinterpret_cast<const float4*>(f + toff) + within;
            const float4 x = __ldcg(src4);
            // smem: tile-major [tile][8][8] with a 16-B chunk swizzle on the tile row
            const int r = within >> 2, ch = within & 3;          // tile row (8 elems = 4 chunks)
            sm4[tile * 32 + r * 4 + (ch ^ (r & 3))] = x;
        }
        __syncthreads();
        if (M == 3) {
            // warp w = row w of every tile: element c = j + 32 q -> tile c / 8, col c % 8
#pragma unroll
            for (int q = 0; q < 32; ++q) {
                const int c = j + 32 * q, tile = c >> 3, cc = c & 7, r = w;
                const int ch = cc >> 1;
                v[q] = sm[(tile * 32 + r * 4 + (ch ^ (r & 3))) * 2 + (cc & 1)];
            }
        } else {
            // warp w = column w of the block: element r = j + 32 q -> tile r / 8, row r % 8
#pragma unroll
            for (int q = 0; q < 32; ++q) {
                const int rr = j + 32 * q, tile = rr >> 3, r = rr & 7, cc = w, ch = cc >> 1;
                v[q] = sm[(tile * 32 + r * 4 + (ch ^ (r & 3))) * 2 + (cc & 1)];
            }
        }
    }
    if (M >= 5) {
        // store patterns (values from registers; a fence makes the time include completion)
#pragma unroll
        for (int q = 0; q < 32; ++q) v[q] = make_float2(q + threadIdx.x, q);
        __syncthreads();
        t0 = clock64();
        float2* g = const_cast<float2*>(f);
        if (M == 5) {
            float2* row = g + (size_t)(blk * 8 + w) * L;
#pragma unroll
            for (int q = 0; q < 32; ++q) __stcg(row + j + 32 * q, v[q]);
        } else if (M == 6) {
            const int c = threadIdx.x & 7, jj = threadIdx.x >> 3;
            float2* col = g + blk * 8 + c;
#pragma unroll
            for (int q = 0; q < 32; ++q) __stcg(col + (size_t)(jj + 32 * q) * L, v[q]);
        } else if (M == 8) {
            // transposed store straight from the warp-per-row registers: element (row r0 + w,
            // column j + 32 q) to T[(j + 32 q) * L + r0 + w] (8-byte pieces; the CTA's 8 warps
            // fill each 64-byte segment)
            float2* t = g + blk * 8 + w;
#pragma unroll
            for (int q = 0; q < 32; ++q) __stcg(t + (size_t)(j + 32 * q) * L, v[q]);
        } else {
            // column block, adjacent columns paired through a shuffle: 16-byte stores
            const int c = threadIdx.x & 7, jj = threadIdx.x >> 3;
            const bool odd = c & 1;
            float4* col = reinterpret_cast<float4*>(g + blk * 8 + (c & ~1));
#pragma unroll
            for (int q = 0; q < 32; q += 2) {
                // even lane keeps row q, odd lane row q+1: exchange the other half
                const float2 send = odd ? v[q] : v[q + 1];
                float2 got;
                got.x = __shfl_xor_sync(0xffffffffu, send.x, 1);
                got.y = __shfl_xor_sync(0xffffffffu, send.y, 1);
                const int qq = odd ? q + 1 : q;
                const float4 o = odd ? make_float4(got.x, got.y, v[q + 1].x, v[q + 1].y)
                                     : make_float4(v[q].x, v[q].y, got.x, got.y);
                __stcg(col + ((size_t)(jj + 32 * qq) * L) / 2, o);
            }
        }
        __threadfence();
    }
    float s = 0.f;
#pragma unroll
    for (int q = 0; q < 32; ++q) s += v[q].x + v[q].y;
    // all values used: stamp after the adds
    long long t1 = clock64();
    out[blk * 256 + threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.x == 0) cyc[blk] = t1 - t0;
}

int main() {
    float2* f; float* out; long long* cyc;
    cudaMalloc(&f, sizeof(float2) * L * L);
    cudaMemset(f, 0, sizeof(float2) * L * L);
    cudaMalloc(&out, 148 * 256 * 4);
    cudaMalloc(&cyc, 148 * 8);
    const char* names[] = {"", "M1 rows, warp per row (row sweep today)", "M2 [1024][8] column block, (c,j) mapping (column sweep today)",
                           "M3 tiled row stripe via smem", "M4 tiled column stripe via smem",
                           "S5 store rows, warp per row", "S6 store column block, (c,j), 8-byte",
                           "S7 store column block, shuffle-paired 16-byte", "S8 transposed store, 8-byte pieces from rows"};
    for (int m = 1; m <= 8; ++m) {
        void (*fn)(const float2*, float*, long long*) = m == 1 ? k<1> : m == 2 ? k<2> : m == 3 ? k<3> : m == 4 ? k<4>
                                                      : m == 5 ? k<5> : m == 6 ? k<6> : m == 7 ? k<7> : k<8>;
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
        long long h[148];
        for (int rep = 0; rep < 5; ++rep) {
            fn<<<148, 256, 65536>>>(f, out, cyc);
            cudaMemcpy(h, cyc, 128 * 8, cudaMemcpyDeviceToHost);
        }
        long long mx = 0, sum = 0;
        for (int i = 0; i < 128; ++i) { mx = h[i] > mx ? h[i] : mx; sum += h[i]; }
        printf("%-62s mean %6lld  max %6lld cycles\n", names[m], sum / 128, mx);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
