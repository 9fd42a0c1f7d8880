// 4096^2 complex64 field in HBM (128 MB > L2): time for every CTA (148, 512
// threads) to load its share of (a) rows: 2 rows of 32 KB per task (the row
// sweep), (b) column pairs: 2 columns x 4096 rows, 16-byte row segments (the
// column sweep), (c) column quads: 4 columns, 32-byte segments (half the
// tasks, each 4 columns); whole-field sweep, tasks round-robin over CTAs.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int L = 4096;

template <int M>
__global__ void __launch_bounds__(512, 1) k(const float2* __restrict__ f, float* out) {
    const int t = threadIdx.x;
    float acc = 0.f;
    const int ntask = M == 2 ? L / 4 : L / 2;
    for (int task = blockIdx.x; task < ntask; task += gridDim.x) {
        float2 v[16];
        if (M == 0) {            // 2 rows: group g = t / 256 owns row 2*task + g, thread j = t % 256 holds j + 256 k
            const float2* row = f + (size_t)(2 * task + (t >> 8)) * L + (t & 255);
#pragma unroll
            for (int q = 0; q < 16; ++q) v[q] = __ldcg(row + 256 * q);
        } else if (M == 1) {     // 2 columns: c = t % 2, j = t / 2, rows j + 256 k
            const float2* col = f + 2 * task + (t & 1) + (size_t)(t >> 1) * L;
#pragma unroll
            for (int q = 0; q < 16; ++q) v[q] = __ldcg(col + (size_t)256 * q * L);
        } else {                 // 4 columns, 16 rows per thread... 512 threads: c = t % 4, j = t / 4 (128), rows j + 128 k
            const float2* col = f + 4 * task + (t & 3) + (size_t)(t >> 2) * L;
#pragma unroll
            for (int q = 0; q < 16; ++q) v[q] = __ldcg(col + (size_t)128 * q * L);
            // (a second half of the column would follow; loads only)
#pragma unroll
            for (int q = 0; q < 16; ++q) { float2 w = __ldcg(col + (size_t)(2048 + 128 * q) * L); v[q].x += w.x; v[q].y += w.y; }
        }
#pragma unroll
        for (int q = 0; q < 16; ++q) acc += v[q].x + v[q].y;
    }
    out[blockIdx.x * 512 + t] = acc;
}

int main() {
    float2* f; float* out; float* flush;
    cudaMalloc(&f, sizeof(float2) * L * L); cudaMemset(f, 0, sizeof(float2) * L * L);
    cudaMalloc(&out, 148 * 512 * 4); cudaMalloc(&flush, 512 << 20);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const char* names[] = {"rows (2 x 32 KB per task)", "column pairs (16-byte segments)", "column quads (32-byte segments)"};
    for (int m = 0; m < 3; ++m) {
        float best = 1e9;
        for (int r = 0; r < 5; ++r) {
            cudaMemset(flush, r, 512 << 20);
            cudaEventRecord(e0);
            if (m == 0) k<0><<<148, 512>>>(f, out); else if (m == 1) k<1><<<148, 512>>>(f, out); else k<2><<<148, 512>>>(f, out);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1); best = ms < best ? ms : best;
        }
        printf("%-34s %.1f us  (%.0f GB/s)\n", names[m], best * 1e3, 128.0 * (1 << 20) / (best * 1e-3) / 1e9);
    }
    return 0;
}
