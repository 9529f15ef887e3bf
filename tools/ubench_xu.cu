// Micro-benchmark: issue throughput of the softmax instruction mix on one SM
// (ex2.approx, cvt.rn.bf16x2.f32, fma.rn.f32x2, ex2.approx.f16x2).  Tuning aid.
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

template <int kMode>
__global__ void bench(float* out, long long* cyc, int iters) {
    float a[8];
    unsigned u[8];
    for (int i = 0; i < 8; ++i) { a[i] = -0.001f * (threadIdx.x + i); u[i] = 0x3c003c00u + i; }
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if constexpr (kMode == 0) {  // ex2
                asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
            } else if constexpr (kMode == 1) {  // cvt bf16x2
                unsigned r;
                asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[(i + 1) & 7]));
                u[i] ^= r;
            } else if constexpr (kMode == 2) {  // 2 ex2 + 1 cvt
                asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
                asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[(i + 4) & 7]));
                unsigned r;
                asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[(i + 1) & 7]));
                u[i] ^= r;
            } else if constexpr (kMode == 3) {  // ffma2
                unsigned long long x = *reinterpret_cast<unsigned long long*>(&a[i & 6]);
                asm volatile("fma.rn.f32x2 %0, %0, %0, %0;" : "+l"(x));
                *reinterpret_cast<unsigned long long*>(&a[i & 6]) = x;
            } else if constexpr (kMode == 4) {  // ex2 f16x2
                asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(u[i]));
            } else if constexpr (kMode == 5) {  // cvt f16x2
                unsigned r;
                asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[(i + 1) & 7]));
                u[i] ^= r;
            } else if constexpr (kMode == 6) {  // ex2.approx.ftz.bf16x2
                asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(u[i]));
            }
        }
    }
    long long t1 = clock64();
    float s = 0;
    for (int i = 0; i < 8; ++i) s += a[i] + __uint_as_float(u[i]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int kMode>
void run(const char* name, int threads, int opsPerIter) {
    float* out;
    long long* cyc;
    cudaMalloc(&out, 148 * 1024 * 4);
    cudaMalloc(&cyc, 148 * 8);
    const int iters = 4096;
    bench<kMode><<<148, threads>>>(out, cyc, iters);
    bench<kMode><<<148, threads>>>(out, cyc, iters);
    cudaDeviceSynchronize();
    long long c;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    double ops = double(iters) * 8 * opsPerIter * threads;
    printf("%-28s threads %4d: %6.2f thread-ops/clk/SM  (%.1f clk per warp-instr per SMSP)\n", name, threads,
           ops / c, (double(c) / (double(iters) * 8 * opsPerIter * threads / 32 / 4)));
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    for (int th : {128, 256, 512}) {
        run<0>("ex2.approx.ftz.f32", th, 1);
        run<1>("cvt.rn.bf16x2.f32", th, 1);
        run<5>("cvt.rn.f16x2.f32", th, 1);
        run<2>("2 ex2 + 1 cvt (ops=3)", th, 3);
        run<3>("fma.rn.f32x2", th, 1);
        run<4>("ex2.approx.f16x2", th, 1);
        run<6>("ex2.approx.ftz.bf16x2", th, 1);
    }
    return 0;
}
