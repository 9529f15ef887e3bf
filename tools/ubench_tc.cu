// Microbenchmarks for design decisions (not part of the product):
//  1. tcgen05.mma kind::f16 M=128 throughput, SS vs TS, N in {64,128,256}
//  2. tcgen05.ld 32x32b.x32 throughput (4 warps)
//  3. commit -> mbarrier -> waiter wake latency
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 ubench_tc.cu -o ubench_tc
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include "../paper_2502_12784_b200/csrc/sm100_ptx.cuh"

using namespace vattn_sm100;

template <int kN, bool kTS>
__global__ void __launch_bounds__(128, 1) mma_bench(long long* out, int reps) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x / 32;
    for (int i = threadIdx.x; i < 131072 / 4; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc<512>(&tslot);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    long long t0 = 0, t1 = 0;
    if (threadIdx.x == 0) {
        constexpr uint32_t idesc = umma_idesc_f16(128, kN, 0, 0, 0);
        const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
        t0 = clock64();
        for (int r = 0; r < reps; ++r) {
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                if (kTS)
                    mma_ts(tmem + (kN == 256 ? 256 : 256), tmem + kk * 8, umma_desc_sw128(b + (kk & 3) * 32 + (kk / 4) * 32768, 16, 1024), idesc, 1);
                else
                    mma_ss(tmem + (kN == 256 ? 256 : 256), umma_desc_sw128(a + (kk & 3) * 32 + (kk / 4) * 16384, 16, 1024),
                           umma_desc_sw128(b + (kk & 3) * 32 + (kk / 4) * 32768, 16, 1024), idesc, 1);
            }
        }
        mma_commit(&bar);
        mbar_wait(&bar, 0);
        t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
}

// cta_group::2 (M = 256) throughput: the leader of each (2,1,1) cluster issues
// reps x 8 K16 steps; each CTA supplies its A rows and half of B at the same offsets.
template <int kN, bool kTS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) mma_bench_pair(long long* out, int reps) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x / 32;
    const uint32_t rank = cluster_rank();
    for (int i = threadIdx.x; i < 131072 / 4; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc_pair<512>(&tslot);
    fence_proxy_async_smem();
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (rank == 0 && warp == 0) {
        constexpr uint32_t idesc = umma_idesc_f16(256, kN, 0, 0, 0);
        const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
        const long long t0 = clock64();
        for (int r = 0; r < reps; ++r) {
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                if (kTS)
                    mma_ts_pair(tmem + 256, tmem + kk * 8, umma_desc_sw128(b + (kk & 3) * 32 + (kk / 4) * 32768, 16, 1024), idesc, 1);
                else
                    mma_ss_pair(tmem + 256, umma_desc_sw128(a + (kk & 3) * 32 + (kk / 4) * 16384, 16, 1024),
                                umma_desc_sw128(b + (kk & 3) * 32 + (kk / 4) * 32768, 16, 1024), idesc, 1);
            }
        }
        mma_commit_pair(&bar);
        mbar_wait(&bar, 0);
        out[blockIdx.x] = out[blockIdx.x + 1] = clock64() - t0;
    } else if (rank == 1 && warp == 0) {
        mbar_wait(&bar, 0);
    }
    tc_fence_before();
    cluster_sync_all();
    if (warp == 0) tmem_dealloc_pair<512>(tmem);
}

__global__ void __launch_bounds__(128, 1) ldtm_bench(long long* out, int reps) {
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x / 32;
    if (warp == 0) tmem_alloc<512>(&tslot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot + (static_cast<uint32_t>(warp * 32) << 16);
    uint32_t acc = 0;
    __syncthreads();
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        uint32_t u0[32], u1[32], u2[32], u3[32];
        tmem_ld32(tmem + 0, u0);
        tmem_ld32(tmem + 32, u1);
        tmem_ld32(tmem + 64, u2);
        tmem_ld32(tmem + 96, u3);
        tmem_wait_ld();
#pragma unroll
        for (int x = 0; x < 32; ++x) acc += u0[x] ^ u1[x] ^ u2[x] ^ u3[x];
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    if (acc == 0x12345678) out[1000] = acc;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tslot);
}

// ping-pong: thread 0 (warp 0) issues one tiny MMA + commit; warp 1 waits, arrives back.
__global__ void __launch_bounds__(64, 1) latency_bench(long long* out, int reps) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar_a, bar_b;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x / 32;
    if (threadIdx.x == 0) {
        mbar_init(&bar_a, 1);
        mbar_init(&bar_b, 1);
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc<512>(&tslot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    constexpr uint32_t idesc = umma_idesc_f16(128, 64, 0, 0, 0);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        if (threadIdx.x == 0) {
            mma_ss(tmem, umma_desc_sw128(smem_u32(smem), 16, 1024), umma_desc_sw128(smem_u32(smem), 16, 1024), idesc, 0);
            mma_commit(&bar_a);
            mbar_wait(&bar_b, r & 1);
        } else if (threadIdx.x == 32) {
            mbar_wait(&bar_a, r & 1);
            tc_fence_after();
            mbar_arrive(&bar_b);
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
}

// MUFU ex2 throughput: each thread runs 8 independent ex2 chains.
__global__ void __launch_bounds__(512) ex2_bench(long long* out, int reps) {
    float v[8];
    for (int i = 0; i < 8; ++i) v[i] = -0.001f * (threadIdx.x + i);
    __syncthreads();
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = ex2(v[i]) - 1.0f;
    }
    __syncthreads();
    long long t1 = clock64();
    float acc = 0;
    for (int i = 0; i < 8; ++i) acc += v[i];
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    if (acc == 1234.5f) out[1000] = 1;
}

template <typename K>
double run(K kern, int grid, int block, int smem, int reps) {
    long long* d;
    cudaMalloc(&d, 2000 * 8);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kern<<<grid, block, smem>>>(d, reps);
    kern<<<grid, block, smem>>>(d, reps);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return -1; }
    long long h[148];
    cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
    double s = 0;
    for (int i = 0; i < grid; ++i) s += h[i];
    cudaFree(d);
    return s / grid;
}

int main(int argc, char** argv) {
    const int which = argc > 1 ? atoi(argv[1]) : -1;
    const int reps = 2000;
    auto report = [&](const char* name, double cyc, int n) {
        const double flop = 2.0 * 128 * n * 128 * reps;  // 8 K16 steps = K128
        printf("%-22s %10.0f cyc  %7.1f flop/clk/SM  (%.1f cyc per M128xN%dxK16)\n", name, cyc, flop / cyc, cyc / (reps * 8.0), n);
    };
    if (which == 0) report("SS N=64", run(mma_bench<64, false>, 148, 128, 131072, reps), 64);
    if (which == 1) report("SS N=128", run(mma_bench<128, false>, 148, 128, 131072, reps), 128);
    if (which == 2) report("SS N=256", run(mma_bench<256, false>, 148, 128, 131072, reps), 256);
    if (which == 3) report("TS N=64", run(mma_bench<64, true>, 148, 128, 131072, reps), 64);
    if (which == 4) report("TS N=128", run(mma_bench<128, true>, 148, 128, 131072, reps), 128);
    if (which == 5) report("TS N=256", run(mma_bench<256, true>, 148, 128, 131072, reps), 256);
    // pair: per-SM flop/clk (each SM holds 128 of the 256 rows)
    if (which == 10) report("pair SS N=128", run(mma_bench_pair<128, false>, 148, 128, 131072, reps) , 128);
    if (which == 11) report("pair SS N=256", run(mma_bench_pair<256, false>, 148, 128, 131072, reps), 256);
    if (which == 12) report("pair TS N=128", run(mma_bench_pair<128, true>, 148, 128, 131072, reps), 128);
    if (which == 13) report("pair SS N=64", run(mma_bench_pair<64, false>, 148, 128, 131072, reps), 64);
    if (which == 7) {
        for (int threads : {128, 256, 512}) {
            long long* d;
            cudaMalloc(&d, 2000 * 8);
            ex2_bench<<<148, threads>>>(d, reps);
            ex2_bench<<<148, threads>>>(d, reps);
            cudaDeviceSynchronize();
            long long h;
            cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
            printf("ex2: %d threads/SM x %d ex2 in %lld cyc -> %.2f ex2/clk/SM\n", threads, reps * 8, h,
                   double(threads) * reps * 8 / h);
            cudaFree(d);
        }
        return 0;
    }
    if (which != 6) return 0;
    const double ld = run(ldtm_bench, 148, 128, 0, reps);
    printf("LDTM 4 warps x 4 x ld32 (64 KB): %.1f cyc per 64 KB -> %.1f B/clk/SM\n", ld / reps, 65536.0 * reps / ld);
    const double lat = run(latency_bench, 1, 64, 65536, reps);
    printf("MMA(N64,K16)+commit -> mbar wake -> arrive -> wake round trip: %.0f cyc\n", lat / reps);
    return 0;
}
