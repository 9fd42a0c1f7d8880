// Throughput of fp32 scalar vs packed (f32x2) instructions on one SM:
// cycles per warp-instruction per SMSP, for W warps per SMSP.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t pk(float x, float y) { uint64_t r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y)); return r; }

template <int OP>
__global__ void k(float* out, long long* cyc, int iters, float s) {
    float a[16], b[16];
    for (int i = 0; i < 16; ++i) { a[i] = threadIdx.x * 0.001f + i; b[i] = s * i + threadIdx.x * 1e-7f; }
    uint64_t p[8], q[8];
    for (int i = 0; i < 8; ++i) { p[i] = pk(a[2*i], a[2*i+1]); q[i] = pk(b[2*i], b[2*i+1]); }
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            if (OP == 0) {          // FADD scalar, 16 independent chains (2 per r)
                a[2*r] = a[2*r] + b[2*r]; a[2*r+1] = a[2*r+1] + b[2*r+1];
            } else if (OP == 1) {   // FADD2 packed, 8 chains
                asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(p[r]) : "l"(q[r]));
            } else if (OP == 2) {   // FFMA scalar
                a[2*r] = fmaf(a[2*r], b[2*r], b[(2*r+5)&15]); a[2*r+1] = fmaf(a[2*r+1], b[2*r+1], b[(2*r+6)&15]);
            } else if (OP == 3) {   // FFMA2
                asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[r]) : "l"(q[r]), "l"(q[(r+3)&7]));
            } else if (OP == 4) {   // FMUL2
                asm volatile("mul.rn.f32x2 %0, %0, %1;" : "+l"(p[r]) : "l"(q[r]));
            } else if (OP == 5) {   // FMUL scalar
                a[2*r] = a[2*r] * b[2*r]; a[2*r+1] = a[2*r+1] * b[2*r+1];
            }
        }
    }
    long long t1 = clock64();
    float acc = 0;
    for (int i = 0; i < 16; ++i) acc += a[i];
    for (int i = 0; i < 8; ++i) { float x, y; asm("mov.b64 {%0,%1}, %2;" : "=f"(x), "=f"(y) : "l"(p[i])); acc += x + y; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    float* out; long long* cyc;
    cudaMalloc(&out, 1 << 20); cudaMalloc(&cyc, 8 * 1024);
    const char* names[] = {"FADD x16 (2 per r)", "FADD2 x8", "FFMA x16", "FFMA2 x8", "FMUL2 x8", "FMUL x16"};
    const int iters = 4096;
    for (int w : {1, 2, 4, 8}) {
        for (int op = 0; op < 6; ++op) {
            void (*f)(float*, long long*, int, float) = op == 0 ? k<0> : op == 1 ? k<1> : op == 2 ? k<2> : op == 3 ? k<3> : op == 4 ? k<4> : k<5>;
            f<<<1, 128 * w>>>(out, cyc, iters, 1.0001f);
            f<<<1, 128 * w>>>(out, cyc, iters, 1.0001f);
            long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
            // per SMSP: w warps each issue iters*8 instructions (16 for scalar ops)
            const double n_inst = (double)iters * ((op == 0 || op == 2 || op == 5) ? 16 : 8) * w;
            printf("warps/SMSP %d  %-20s cycles/instr/SMSP %.3f\n", w, names[op], c / n_inst);
        }
    }
    return 0;
}
