// Micro-benchmark: tcgen05.ld (TMEM -> registers) throughput per SM with W warps
// (W/4 warps per 32-lane TMEM subpartition).  Tuning aid: nvcc -gencode
// arch=compute_100a,code=sm_100a -O3 -o /tmp/ubt tools/ubench_tmem.cu && /tmp/ubt
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2502_12784_b200/csrc/sm100_ptx.cuh"
using namespace vattn_sm100;

template <int kLoadsPerWait>
__global__ void bench(float* out, long long* cyc, int iters) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tmem_alloc<512>(&slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    const uint32_t lb = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t col0 = (warp >> 2) * 128 % 512;
    float acc = 0.f;
    float r[32];
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < kLoadsPerWait; ++c) {
            tmem_ld32f(tmem + lb + ((col0 + 32 * c) & 511), r);
        }
        tmem_wait_ld();
        acc += r[0] + r[31];
    }
    const long long t1 = clock64();
    __syncthreads();
    if ((threadIdx.x & 31) == 0) cyc[blockIdx.x * 32 + warp] = t1 - t0;
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
}

template <int kL>
void run(int warps) {
    const int iters = 2000;
    float* out;
    long long* cyc;
    cudaMalloc(&out, 148 * 1024 * 4);
    cudaMalloc(&cyc, 148 * 32 * 8);
    bench<kL><<<148, 32 * warps>>>(out, cyc, 10);
    bench<kL><<<148, 32 * warps>>>(out, cyc, iters);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return; }
    long long h[32];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int w = 0; w < warps; ++w) mx = h[w] > mx ? h[w] : mx;
    const double bytes = double(warps) * iters * kL * 32 * 32 * 4;
    printf("warps %2d, %d x32 loads per wait: %.1f B/clk/SM (%.1f clk per x32 load per warp)\n", warps, kL,
           bytes / mx, double(mx) / (iters * kL));
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    for (int w : {1, 4, 8, 16}) {
        run<1>(w);
        run<4>(w);
    }
    return 0;
}
