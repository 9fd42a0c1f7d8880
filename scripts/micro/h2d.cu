// H2D / D2H of 8 MB from cudaHostAlloc memory with the statically linked runtime (as the library).
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>
int main() {
    const size_t n = 8 << 20;
    void *h, *d; cudaStream_t s; cudaEvent_t e0, e1;
    cudaHostAlloc(&h, n, cudaHostAllocPortable); cudaMalloc(&d, n); cudaStreamCreate(&s);
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    memset(h, 1, n);
    for (int dir = 0; dir < 2; ++dir)
        for (int chunks : {1, 2}) {
            float best = 1e9;
            for (int r = 0; r < 10; ++r) {
                cudaEventRecord(e0, s);
                for (int c = 0; c < chunks; ++c) {
                    char* hp = (char*)h + c * (n / chunks); char* dp = (char*)d + c * (n / chunks);
                    if (dir == 0) cudaMemcpyAsync(dp, hp, n / chunks, cudaMemcpyHostToDevice, s);
                    else cudaMemcpyAsync(hp, dp, n / chunks, cudaMemcpyDeviceToHost, s);
                }
                cudaEventRecord(e1, s); cudaEventSynchronize(e1);
                float ms; cudaEventElapsedTime(&ms, e0, e1); best = ms < best ? ms : best;
            }
            printf("%s 8 MB in %d copies: %.3f ms (%.1f GB/s)\n", dir ? "D2H" : "H2D", chunks, best, n / best / 1e6);
        }
    return 0;
}
