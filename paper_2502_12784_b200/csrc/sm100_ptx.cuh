// sm100_ptx.cuh -- thin inline-PTX layer for Blackwell (sm_100a): mbarriers,
// TMA (cp.async.bulk.tensor), tcgen05 (alloc / mma / commit / ld / st) and the
// UMMA shared-memory + instruction descriptors.  Everything the fused MHA
// kernels touch on the async path lives here; no CUTLASS/CuTe at runtime.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>
#include <cstdio>

#define VATTN_DEV __device__ __forceinline__

namespace vattn_sm100 {

// ------------------------------------------------------------------ basics --

VATTN_DEV uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

VATTN_DEV uint32_t warp_id() { return threadIdx.x >> 5; }

// Grid mapping of the tile kernels.  Default (0): tiles of one (b, h) on x, so the
// CTAs resident at any moment belong to a few heads and share their K/V (or Q/dO)
// tiles through L2 -- every kernel reads ~1.0x its algorithmic HBM bytes.  1: (b*h,
// tile) on (x, y), longest causal item of every head first; measured on B200 it
// loses that L2 sharing (C3 -10 %, C5 -22 %) and gains only ~3 % on short C4 heads.
// Block -> ((b,h) unit, tile).  The grid is (ntiles * G, BH / G): groups of G units
// dispatch one after another, and inside a group the blocks go tile-major, so the
// longest causal items of the group start first (longest-processing-time order) while
// the group's shared streams (K/V in the forward, Q/dO in the backward) stay resident
// in L2 across all of its tiles.  G = 1 is plain unit-major order (every unit's tiles
// in a row); G = BH is global tile-major order.  Tile 0 is the heaviest causal item.
VATTN_DEV int grid_tile(int ntiles) { return static_cast<int>(blockIdx.x) / (static_cast<int>(gridDim.x) / ntiles); }
VATTN_DEV int grid_bh(int ntiles) {
    const int G = static_cast<int>(gridDim.x) / ntiles;
    return static_cast<int>(blockIdx.y) * G + static_cast<int>(blockIdx.x) % G;
}
inline dim3 tile_grid(int ntiles, int bh, int G) { return dim3(ntiles * G, bh / G); }
// 1-D variant with a longest-first tail: units [0, BH - T) unit-major, then the last T
// units tile-major, so the heaviest causal items of the final units start waves before
// the end instead of in the last wave (grid = ntiles * BH blocks along x).
// Item L of `total` (= BH * ntiles) items: the same order (CTA pairs: item = cluster).
VATTN_DEV void grid_item_tail_n(int L, int total, int ntiles, int T, int& bh, int& tile) {
    const int BH = total / ntiles;
    const int head = (BH - T) * ntiles;
    if (L < head) {
        bh = L / ntiles;
        tile = L % ntiles;
    } else {
        const int r = L - head;
        tile = r / T;
        bh = BH - T + r % T;
    }
}
VATTN_DEV void grid_item_tail(int ntiles, int T, int& bh, int& tile) {
    const int BH = static_cast<int>(gridDim.x) / ntiles;
    const int L = static_cast<int>(blockIdx.x);
    const int head = (BH - T) * ntiles;
    if (L < head) {
        bh = L / ntiles;
        tile = L % ntiles;
    } else {
        const int r = L - head;
        tile = r / T;
        bh = BH - T + r % T;
    }
}
VATTN_DEV uint32_t lane_id() { return threadIdx.x & 31; }

// Per-warpgroup register budget hand-off (all 4 warps of the warpgroup execute it).
template <uint32_t kRegs>
VATTN_DEV void regs_inc() { asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegs)); }
template <uint32_t kRegs>
VATTN_DEV void regs_dec() { asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegs)); }

// Programmatic dependent launch: kernels are launched with programmatic stream
// serialisation, so the next kernel's CTAs set up (barriers, tensor memory) while
// this grid's last CTAs finish.  griddep_wait() blocks until the previous grid in
// the stream completed and its writes are visible -- every kernel calls it before
// its first global read; griddep_launch_dependents() at the end of every CTA lets
// the next grid launch once all CTAs of this one reached it (never earlier, so a
// waiting dependent can not take the SMs the remaining CTAs of this grid need).
VATTN_DEV void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
VATTN_DEV void griddep_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
// VATTN_PDL_EARLY=1: every CTA triggers its dependents as it starts (griddep_start) instead
// of at its end.  The dependent grid then launches once the LAST CTA of this grid is
// resident -- no CTA of this grid can still be waiting for an SM, so nothing is starved --
// and its CTAs take the SMs this grid's tail frees, run their prologue and wait in
// griddep_wait for this grid's completion (which is what orders the data).  Measured
// neutral to -1 % (C4 24-layer graph 4.17 vs 4.13 ms, C2 N = 512 / 1k -1 %), so off.
#ifndef VATTN_PDL_EARLY
#define VATTN_PDL_EARLY 0
#endif
constexpr bool kPdlEarly = VATTN_PDL_EARLY;
VATTN_DEV void griddep_start() {
    if constexpr (kPdlEarly) griddep_launch_dependents();
}

// Named barrier over `nthreads` threads (id 0 is __syncthreads).
VATTN_DEV void named_bar_sync(uint32_t id, uint32_t nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// --------------------------------------------------------------- mbarrier --

VATTN_DEV void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

VATTN_DEV void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

VATTN_DEV void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

VATTN_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

VATTN_DEV bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

// try_wait with a suspend-time hint: the thread is parked in hardware until the
// phase completes (or the hint elapses) instead of spinning, so a long-waiting
// warp does not steal issue slots from the math warps of its SM sub-partition
// (at the price of a slower wake-up: use it off the critical path).
VATTN_DEV bool mbar_try_wait_sleep(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity), "r"(0x989680u)
        : "memory");
    return ok != 0;
}

VATTN_DEV uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Hang guard: a wait that exceeds VATTN_WATCHDOG_NS traps (the launch fails
// with an error instead of wedging the GPU).  0 disables it.
#ifndef VATTN_WATCHDOG_NS
#define VATTN_WATCHDOG_NS 20000000000ull
#endif

// MMA-warp wait flavour (experiment knob): 0 spin, 1 spin with nanosleep backoff,
// 2 short suspend hint.
#ifndef VATTN_MMA_WAIT
#define VATTN_MMA_WAIT 0
#endif
VATTN_DEV bool mbar_try_wait_hint(uint64_t* bar, uint32_t parity, uint32_t ns) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity), "r"(ns)
        : "memory");
    return ok != 0;
}
// Whole-warp wait of an MMA-issuing warp: the lanes may leave the polling loop at
// different iterations, so they are re-converged before the caller's elect.sync.
VATTN_DEV void mbar_wait_mma_(uint64_t* bar, uint32_t parity);
VATTN_DEV void mbar_wait_mma(uint64_t* bar, uint32_t parity) {
    mbar_wait_mma_(bar, parity);
    __syncwarp();
}
VATTN_DEV void mbar_wait_mma_(uint64_t* bar, uint32_t parity) {
    if (mbar_try_wait(bar, parity)) return;
    const uint64_t t0 = globaltimer_ns();
    uint32_t n = 0;
    while (true) {
#if VATTN_MMA_WAIT == 2
        if (mbar_try_wait_hint(bar, parity, 200u)) return;
#else
        if (mbar_try_wait(bar, parity)) return;
#if VATTN_MMA_WAIT == 1
        __nanosleep(20);
#endif
#endif
        if (VATTN_WATCHDOG_NS && (++n & 255u) == 0 && globaltimer_ns() - t0 > VATTN_WATCHDOG_NS) __trap();
    }
}

// Wait until the phase with parity `parity` has completed (kSleep: park instead of spin).
// kPrint: report the stuck barrier before trapping.  Besides being a debug aid it
// changes the code ptxas emits around the wait loops; it is enabled where that
// measured faster on B200 (the dQ kernel: 1.33 vs 1.44 ms at C3).
template <bool kSleep = false, bool kPrint = false>
VATTN_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
    auto probe = [&] { return kSleep ? mbar_try_wait_sleep(bar, parity) : mbar_try_wait(bar, parity); };
    if (probe()) return;
#if VATTN_WATCHDOG_NS
    const uint64_t t0 = globaltimer_ns();
    uint32_t n = 0;
    while (!probe()) {
        if ((++n & (kSleep ? 0u : 1023u)) == 0 && globaltimer_ns() - t0 > VATTN_WATCHDOG_NS) {
#ifndef VATTN_WATCHDOG_PRINT
            if constexpr (kPrint)
#endif
                printf("vattn watchdog: block %d thread %d stuck on mbarrier smem+0x%x parity %u\n",
                       (int)(blockIdx.x + blockIdx.y * gridDim.x), (int)threadIdx.x, smem_u32(bar), parity);
            __trap();
        }
    }
#else
    while (!probe()) {
    }
#endif
}

// Schedule fuzzer (stress builds only, -DVATTN_STRESS_NS=<ns>; compiled out by
// default): parks the calling warp for a pseudo-random 0..VATTN_STRESS_NS ns at
// one in eight of the points it is called from, so warps and warpgroups drift
// apart by whole pipeline steps.  The value depends only on warp-uniform inputs
// (block, warp, call site, step), so every active lane takes the same branch (the
// producer calls it from its single elected lane).  tests/test_stress_gpu.py soaks every kernel
// under it: a barrier protocol that relies on warps staying in lock step hangs
// (watchdog trap) or races there.
#ifndef VATTN_STRESS_NS
#define VATTN_STRESS_NS 0
#endif
VATTN_DEV void stress_delay(uint32_t site, uint32_t step) {
#if VATTN_STRESS_NS
    uint32_t x = blockIdx.x * 0x9E3779B1u ^ blockIdx.y * 0x85EBCA77u ^ (threadIdx.x >> 5) * 0xC2B2AE3Du ^
                 site * 0x27D4EB2Fu ^ step * 0x165667B1u;
    x ^= x >> 15;
    x *= 0x2C1B3C6Du;
    x ^= x >> 12;
    x *= 0x297A2D39u;
    x ^= x >> 15;
    if ((x & 7u) == 0) {
        uint32_t ns = (x >> 8) % static_cast<uint32_t>(VATTN_STRESS_NS);
        while (ns > 0) {
            const uint32_t chunk = ns > 100000u ? 100000u : ns;
            __nanosleep(chunk);
            ns -= chunk;
        }
    }
#else
    (void)site;
    (void)step;
#endif
}

// Role-specific wait policy (bit set = that role parks instead of spinning).
#ifndef VATTN_SLEEP_MASK
#define VATTN_SLEEP_MASK 1
#endif
#define VATTN_SLEEP_PRODUCER ((VATTN_SLEEP_MASK & 1) != 0)
#define VATTN_SLEEP_MMA ((VATTN_SLEEP_MASK & 2) != 0)
#define VATTN_SLEEP_MATH ((VATTN_SLEEP_MASK & 4) != 0)

// -------------------------------------------------------------------- TMA --

VATTN_DEV void tma_prefetch_desc(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// 3-D tiled load: box lands in smem `dst`, completion counted on `bar` (bytes).
VATTN_DEV void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                           int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

// 3-D tiled store from smem (rows outside the tensor are clipped by the TMA unit).
VATTN_DEV void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
            reinterpret_cast<uint64_t>(map)),
        "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(src))
        : "memory");
}

// Plain 1-D bulk copy global -> smem (16-byte aligned, multiple of 16 bytes).
VATTN_DEV void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

VATTN_DEV void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
VATTN_DEV void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
VATTN_DEV void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// Make generic-proxy smem writes visible to the async proxy (TMA store, UMMA).
VATTN_DEV void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---------------------------------------------------------------- tcgen05 --

template <uint32_t kCols>
VATTN_DEV void tmem_alloc(uint32_t* smem_dst) {
    static_assert(kCols >= 32 && kCols <= 512 && (kCols & (kCols - 1)) == 0, "TMEM cols");
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(smem_dst)),
                 "n"(kCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

template <uint32_t kCols>
VATTN_DEV void tmem_dealloc(uint32_t taddr) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols)
                 : "memory");
}

VATTN_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
VATTN_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// D[tmem] (+)= A[smem] * B[smem]   (kind::f16: fp16/bf16 in, fp32 accumulate)
VATTN_DEV void mma_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                      uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// D[tmem] (+)= A[tmem] * B[smem]
VATTN_DEV void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                      uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// Warp-uniform variants: the whole warp executes them (so descriptors stay in
// uniform registers) and one elected lane issues the instruction.
VATTN_DEV void mma_ss_e(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                        uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

VATTN_DEV void mma_ts_e(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                        uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

VATTN_DEV void mma_commit_e(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
            smem_u32(bar))
        : "memory");
}

// ------------------------------------------------------------ CTA pair --
// cta_group::2: two CTAs of a (2,1,1) cluster on one TPC run M = 256 MMAs.  The
// leader (rank 0) issues every MMA; each CTA supplies its 128 A rows and half of the
// B columns from its own shared memory at the same offsets, and holds its 128 rows
// of D in its own tensor memory at the same column addresses.  Every tcgen05
// instruction of such a kernel uses cta_group::2.

VATTN_DEV uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
// shared::cluster address of `p` (a shared::cta pointer) in CTA `rank` of the cluster.
VATTN_DEV uint32_t mapa_u32(const void* p, uint32_t rank) {
    uint32_t a;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(smem_u32(p)), "r"(rank));
    return a;
}
VATTN_DEV void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Arrive on an mbarrier given by its shared::cluster address.  Relaxed: what it
// publishes is tensor memory (ordered by tcgen05.wait::st + tcgen05.fence::
// before_thread_sync), and a release.cluster arrive compiles to a MEMBAR that
// stalled the math warps (ncu: membar the top stall reason, the pair kernel 40 %
// slower than one CTA).
VATTN_DEV void mbar_arrive_cluster(uint32_t cl_addr) {
#ifdef VATTN_PAIR_ACQ_CLUSTER
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cl_addr) : "memory");
#else
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cl_addr) : "memory");
#endif
}
VATTN_DEV void mbar_arrive_expect_tx_cluster(uint32_t cl_addr, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(cl_addr), "r"(bytes)
                 : "memory");
}
// Whole-warp wait for barriers the peer CTA arrives on.  Polled with the CTA-scope
// try_wait (an acquire.cluster poll loop measured 2-3x slower MMAs and math passes on
// the whole SM); the peer's arrivals are release.cluster after tcgen05.wait::st, and the
// waiter's tcgen05.fence::after_thread_sync orders its MMAs after them.
VATTN_DEV bool mbar_try_wait_cl(uint64_t* bar, uint32_t parity) {
#ifdef VATTN_PAIR_ACQ_CLUSTER
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
#else
    return mbar_try_wait(bar, parity);
#endif
}
VATTN_DEV void mbar_wait_mma_cl(uint64_t* bar, uint32_t parity) {
    if (!mbar_try_wait_cl(bar, parity)) {
        const uint64_t t0 = globaltimer_ns();
        uint32_t n = 0;
        while (!mbar_try_wait_cl(bar, parity))
            if (VATTN_WATCHDOG_NS && (++n & 255u) == 0 && globaltimer_ns() - t0 > VATTN_WATCHDOG_NS) {
#ifdef VATTN_WATCHDOG_PRINT
                printf("vattn watchdog (MMA, cluster): block %d stuck on mbarrier smem+0x%x parity %u\n", (int)blockIdx.x,
                       smem_u32(bar), parity);
#endif
                __trap();
            }
    }
    __syncwarp();
}
// TMA load into this CTA's shared memory whose completion is counted on an mbarrier
// of the pair's leader (`bar_cl`: shared::cluster address).
VATTN_DEV void tma_load_3d_pair(void* dst, const CUtensorMap* map, uint32_t bar_cl, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar_cl)
        : "memory");
}
template <uint32_t kCols>
VATTN_DEV void tmem_alloc_pair(uint32_t* smem_dst) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_dst)), "n"(kCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
template <uint32_t kCols>
VATTN_DEV void tmem_dealloc_pair(uint32_t taddr) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols) : "memory");
}
VATTN_DEV void mma_ss_pair(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
VATTN_DEV void mma_ts_pair(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// Arrive on `bar` (same shared-memory offset) in both CTAs of the pair once every
// previously issued tcgen05.mma of this thread completes.
VATTN_DEV void mma_commit_pair(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
            smem_u32(bar)),
        "h"(static_cast<uint16_t>(3))
        : "memory");
}

// Descriptor of the kk-th K=16 slice of a 128-row SW128 operand tile whose base
// descriptor is `d0` (address field counts 16-byte units; no carry possible
// below 256 KB of shared memory).
//  K-major  (rows = M/N, 64 K-elements per 128-B row, 16 KB per 64-col box)
VATTN_DEV uint64_t desc_kmajor(uint64_t d0, int kk) {
    return d0 + static_cast<uint64_t>(((kk >> 2) * 16384 + (kk & 3) * 32) >> 4);
}
//  K-major with 64-row boxes (8 KB per 64-col box): the CTA pair's half B operand
VATTN_DEV uint64_t desc_kmajor_half(uint64_t d0, int kk) {
    return d0 + static_cast<uint64_t>(((kk >> 2) * 8192 + (kk & 3) * 32) >> 4);
}
//  MN-major (rows = K, 16 K-rows = 2048 B per slice)
VATTN_DEV uint64_t desc_mnmajor(uint64_t d0, int kk) { return d0 + static_cast<uint64_t>((kk * 2048) >> 4); }

// Arrive on `bar` once every previously issued tcgen05.mma of this thread completes.
VATTN_DEV void mma_commit(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(bar))
        : "memory");
}

VATTN_DEV void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
VATTN_DEV void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// 32 lanes x 32 consecutive 32-bit columns: thread t of the warp gets lane
// (warp's lane quarter base + t), columns [col, col + 32).
VATTN_DEV void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
        "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
          "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
          "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}

// Same as tmem_ld32 but straight into fp32 registers.
VATTN_DEV void tmem_ld32f(uint32_t taddr, float* f) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
        "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=f"(f[0]), "=f"(f[1]), "=f"(f[2]), "=f"(f[3]), "=f"(f[4]), "=f"(f[5]), "=f"(f[6]),
          "=f"(f[7]), "=f"(f[8]), "=f"(f[9]), "=f"(f[10]), "=f"(f[11]), "=f"(f[12]), "=f"(f[13]),
          "=f"(f[14]), "=f"(f[15]), "=f"(f[16]), "=f"(f[17]), "=f"(f[18]), "=f"(f[19]),
          "=f"(f[20]), "=f"(f[21]), "=f"(f[22]), "=f"(f[23]), "=f"(f[24]), "=f"(f[25]),
          "=f"(f[26]), "=f"(f[27]), "=f"(f[28]), "=f"(f[29]), "=f"(f[30]), "=f"(f[31])
        : "r"(taddr));
}

VATTN_DEV void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}

VATTN_DEV void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, "
        "%17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(
            taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
        "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
        "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
        "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}

VATTN_DEV void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
        "r"(r[15])
        : "memory");
}

// ------------------------------------------------------ UMMA descriptors --

// Shared-memory matrix descriptor, 128-byte swizzle (the layout TMA writes with
// CU_TENSOR_MAP_SWIZZLE_128B: 8-row x 128-byte atoms, 1024-byte aligned).
//  K-major operand : rows = M/N index, 64 16-bit K elements per 128-B row;
//                    sbo = 1024 (next 8 rows), lbo unused (16).
//  MN-major operand: rows = K index, 64 16-bit M/N elements per 128-B row;
//                    sbo = 1024 (next 8 K rows), lbo = bytes to the next
//                    64-element M/N chunk.
VATTN_DEV uint64_t umma_desc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4);
    d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
    d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
    d |= static_cast<uint64_t>(1) << 46;  // descriptor version (sm_100)
    d |= static_cast<uint64_t>(2) << 61;  // SWIZZLE_128B
    return d;
}

// Instruction descriptor for kind::f16 with fp32 accumulation.
//  ab_bf16: 0 = fp16 operands, 1 = bf16.  a_mn / b_mn: 1 = MN-major operand.
__host__ __device__ constexpr uint32_t umma_idesc_f16(uint32_t M, uint32_t N, uint32_t ab_bf16,
                                                      uint32_t a_mn, uint32_t b_mn) {
    return (1u << 4)                 // D format f32
           | (ab_bf16 << 7)          // A format
           | (ab_bf16 << 10)         // B format
           | (a_mn << 15) | (b_mn << 16)  //
           | ((N >> 3) << 17)        //
           | ((M >> 4) << 24);
}

// ------------------------------------------------------------ debug trace --
// Build with -DVATTN_TRACE: kernels stamp clock64() of pipeline events of the
// CTA selected by g_vattn_trace_block into g_vattn_trace (read back through
// vattn_trace_read()).  Compiled out otherwise.
#ifdef VATTN_TRACE
__device__ long long g_vattn_trace[4096];
__device__ int g_vattn_trace_block;
__device__ int g_vattn_trace_kid;  // which kernel (kVtraceKid of the kernel) is traced
#define VTRACE(slot)                                                                      \
    do {                                                                                 \
        if (kVtraceKid == g_vattn_trace_kid &&                                            \
            static_cast<int>(blockIdx.x + blockIdx.y * gridDim.x) == g_vattn_trace_block) \
            g_vattn_trace[(slot)] = clock64();                                           \
    } while (0)
// Per-CTA timeline (which SM, globaltimer at entry and exit) of every CTA of the
// kernel selected by g_vattn_trace_kid: the SM-busy fraction and the gaps between
// consecutive CTAs on one SM (tools/cta_timeline.py).
__device__ unsigned long long g_vattn_cta[16384][3];
VATTN_DEV unsigned long long vcta_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define VCTA(kid, which)                                                                  \
    do {                                                                                 \
        const int b_ = static_cast<int>(blockIdx.x + blockIdx.y * gridDim.x);            \
        if ((kid) == g_vattn_trace_kid && threadIdx.x == 0 && b_ < 16384) {               \
            g_vattn_cta[b_][which] = vcta_now();                                          \
            if ((which) == 0) {                                                          \
                unsigned sm_;                                                            \
                asm volatile("mov.u32 %0, %%smid;" : "=r"(sm_));                          \
                g_vattn_cta[b_][2] = sm_;                                                \
            }                                                                            \
        }                                                                                \
    } while (0)
#else
#define VTRACE(slot) \
    do {             \
    } while (0)
#define VCTA(kid, which) \
    do {                 \
    } while (0)
#endif

// ------------------------------------------------------------ conversions --

template <bool kBF16>
VATTN_DEV uint32_t pack2(float lo, float hi) {
    uint32_t r;
    if constexpr (kBF16) {
        asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    } else {
        asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    }
    return r;
}

template <bool kBF16>
VATTN_DEV float2 unpack2(uint32_t v) {
    if constexpr (kBF16) {
        return make_float2(__uint_as_float(v << 16), __uint_as_float(v & 0xFFFF0000u));
    } else {
        __half2 h = *reinterpret_cast<__half2*>(&v);
        return __half22float2(h);
    }
}

VATTN_DEV float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// 2^x on the FMA pipe (degree-4 minimax on [-0.5, 0.5], max rel. error 2.9e-6):
// relieves the MUFU (16 ex2/clk/SM), which every P pass of this path saturates.
// x is clamped at -127 (result ~1e-38, i.e. a zero contribution); +inf never occurs.
VATTN_DEV float ex2_poly(float x) {
    x = fmaxf(x, -127.0f);
    const float t = x + 12582912.0f;  // 1.5 * 2^23: round(x) lands in the low mantissa bits
    const float f = x - (t - 12582912.0f);
    float p = fmaf(f, 0.009582852944731712f, 0.055906426161527634f);
    p = fmaf(p, f, 0.24024099111557007f);
    p = fmaf(p, f, 0.6931241750717163f);
    p = fmaf(p, f, 1.0f);
    return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

// Share of exponentials routed to ex2_poly: element pairs with pair % period == 0
// (period 0 = MUFU only).  Tuned per kernel on B200 (bench.py, C3).
#ifndef VATTN_POLY_FWD
#define VATTN_POLY_FWD 4
#endif
#ifndef VATTN_POLY_DQ
#define VATTN_POLY_DQ 0
#endif
// d = 64: the exponentials per tile are the same as at d = 128 but the MMA work
// halves, so every kernel is MUFU-bound there and the offload pays.
#ifndef VATTN_POLY_FWD64
#define VATTN_POLY_FWD64 4
#endif
#ifndef VATTN_POLY_DQ64
#define VATTN_POLY_DQ64 0
#endif
// dK/dV P pass: element pairs out of every 4 on the polynomial, per warpgroup (d = 128
// and d = 64 knobs).  Round 1 chose an asymmetric 0 / 2 split (both warpgroups
// exponentiate at the same time; -2.2 % vs 0 / 0 at C3).  Round 2: a symmetric 1 / 1
// split is better still (dK/dV C3 -4 %, C2 / C4 d = 64 -3..-4 %; dQ recompute d = 64
// -4..-6 %, profiles/r2_experiments.md) -- equal knobs compile ONE copy of the unrolled
// P pass instead of one per warpgroup, and these kernels are sensitive to code size
// (the forward's masked-tile copy measured the same way, -3..-5 %).
#ifndef VATTN_POLY_DKDV_WG0
#define VATTN_POLY_DKDV_WG0 1
#endif
#ifndef VATTN_POLY_DKDV_WG1
#define VATTN_POLY_DKDV_WG1 1
#endif
#ifndef VATTN_POLY_DKDV64_WG0
#define VATTN_POLY_DKDV64_WG0 1
#endif
#ifndef VATTN_POLY_DKDV64_WG1
#define VATTN_POLY_DKDV64_WG1 1
#endif
// dQ recompute kernel P pass, same scheme (pairs out of every 4, per warpgroup)
#ifndef VATTN_POLY_DQ_WG0
#define VATTN_POLY_DQ_WG0 0
#endif
#ifndef VATTN_POLY_DQ_WG1
#define VATTN_POLY_DQ_WG1 0
#endif
#ifndef VATTN_POLY_DQ64_WG0
#define VATTN_POLY_DQ64_WG0 1
#endif
#ifndef VATTN_POLY_DQ64_WG1
#define VATTN_POLY_DQ64_WG1 1
#endif
template <int kD> struct PolyPeriod {
    static constexpr int fwd = kD == 64 ? VATTN_POLY_FWD64 : VATTN_POLY_FWD;
    static constexpr int dq = kD == 64 ? VATTN_POLY_DQ64 : VATTN_POLY_DQ;
};
// `pair` is an unrolled loop index, so the branch folds away at compile time.
template <int kPeriod>
VATTN_DEV float ex2_mix(int pair, float x) {
    if constexpr (kPeriod > 0) {
        if (pair % kPeriod == 0) return ex2_poly(x);
    }
    return ex2(x);
}

// fmax the compiler cannot re-associate into one dependent FMNMX3 chain.  The .NaN
// flavour (FMNMX.NAN) propagates a NaN operand instead of dropping it, so a NaN
// score reaches the row maximum (the forward's domain-error flag, like the
// reference's NaN-score check, online_softmax.cpp:33-34).
VATTN_DEV float fmax_nr(float a, float b) {
    float r;
    asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
}

// 3-input max (FMNMX3.NAN): halves the instructions of a row-max tree.
VATTN_DEV float fmax3(float a, float b, float c) {
    float r;
    asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

// Max of an unrolled register array: 8 independent chains of 3-input maxima
// (few live temporaries, depth kN/16 + 3); NaN if any element is NaN.
template <int kN>
VATTN_DEV float row_max(const float* v) {
    static_assert(kN % 16 == 0 && kN >= 16, "row_max");
    float a[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) a[c] = fmax_nr(v[c], v[c + 8]);
#pragma unroll
    for (int i = 16; i < kN; i += 16)
#pragma unroll
        for (int c = 0; c < 8; ++c) a[c] = fmax3(a[c], v[i + c], v[i + 8 + c]);
    return fmax3(fmax3(a[0], a[1], a[2]), fmax3(a[3], a[4], a[5]), fmax_nr(a[6], a[7]));
}

// Packed fp32 pairs (FFMA2 / FADD2 / FMUL2 on sm_100): one issue slot per two lanes' worth.
VATTN_DEV float2 ffma2(float2 a, float2 b, float2 c) {
    float2 d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;"
        : "=l"(*reinterpret_cast<unsigned long long*>(&d))
        : "l"(*reinterpret_cast<const unsigned long long*>(&a)), "l"(*reinterpret_cast<const unsigned long long*>(&b)),
          "l"(*reinterpret_cast<const unsigned long long*>(&c)));
    return d;
}
VATTN_DEV float2 fadd2(float2 a, float2 b) {
    float2 d;
    asm("add.f32x2 %0, %1, %2;"
        : "=l"(*reinterpret_cast<unsigned long long*>(&d))
        : "l"(*reinterpret_cast<const unsigned long long*>(&a)), "l"(*reinterpret_cast<const unsigned long long*>(&b)));
    return d;
}
VATTN_DEV float2 fmul2(float2 a, float2 b) {
    float2 d;
    asm("mul.f32x2 %0, %1, %2;"
        : "=l"(*reinterpret_cast<unsigned long long*>(&d))
        : "l"(*reinterpret_cast<const unsigned long long*>(&a)), "l"(*reinterpret_cast<const unsigned long long*>(&b)));
    return d;
}

// Per-thread 16-byte global -> shared copy (LDGSTS, L2 only); bytes = 0 zero-fills.
VATTN_DEV void cp_async16(uint32_t dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(bytes) : "memory");
}
VATTN_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
VATTN_DEV void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
VATTN_DEV uint32_t lds_u32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
    return v;
}
VATTN_DEV uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
    return d;
}
// Keep mask of packed pair x (keys 2x, 2x + 1) of a 32-key word kw, as two 16-bit lanes
// of all ones (kept) or zeros, from the word's shifts ks[s] = kw << s: key k sits in the
// sign bit of byte k / 8 of ks[7 - k % 8], and PRMT's sign-replicate selectors spread it
// over the lane -- one PRMT per pair, the eight shifts shared by the word's 16 pairs.
VATTN_DEV uint32_t keep_mask16(const uint32_t (&ks)[8], int x) {
    const int m = x >> 2, s0 = 7 - 2 * (x & 3);
    const uint32_t sel = static_cast<uint32_t>((8 | m) | ((8 | m) << 4) | ((12 | m) << 8) | ((12 | m) << 12));
    return prmt(ks[s0], ks[s0 - 1], sel);
}
// The same for one key k of the word as a 32-bit lane (all ones = kept): the sign of byte
// k / 8 of ks[7 - k % 8] replicated over the four bytes.
VATTN_DEV uint32_t keep_mask32(const uint32_t (&ks)[8], int k) {
    const uint32_t n = static_cast<uint32_t>(8 | (k >> 3));
    return prmt(ks[7 - (k & 7)], 0u, n * 0x1111u);
}

// Two ex2_poly on packed fp32 pairs (FFMA2 / FADD2): ~5.5 issue slots per element.
VATTN_DEV float2 ex2_poly2(float2 x) {
    x.x = fmaxf(x.x, -127.0f);
    x.y = fmaxf(x.y, -127.0f);
    const float2 kRnd = make_float2(12582912.0f, 12582912.0f);
    const float2 t = fadd2(x, kRnd);
    const float2 f = fadd2(x, fadd2(kRnd, make_float2(-t.x, -t.y)));
    float2 p = ffma2(f, make_float2(0.009582852944731712f, 0.009582852944731712f),
                     make_float2(0.055906426161527634f, 0.055906426161527634f));
    p = ffma2(p, f, make_float2(0.24024099111557007f, 0.24024099111557007f));
    p = ffma2(p, f, make_float2(0.6931241750717163f, 0.6931241750717163f));
    p = ffma2(p, f, make_float2(1.0f, 1.0f));
    return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                       __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}

VATTN_DEV float lg2(float x) {
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// 16-byte store into a 128-B-swizzled tile: row r (128-B line), 16-B chunk c.
VATTN_DEV void st_swz128(uint8_t* tile, uint32_t row, uint32_t chunk, uint4 v) {
    const uint32_t off = row * 128u + (((chunk ^ (row & 7u)) & 7u) << 4);
    *reinterpret_cast<uint4*>(tile + off) = v;
}

// -------------------------------------------------------------- dropout --
// The reference's stateless dropout decision (proj/src/rng.cpp:35-49):
//   keep(b,h,row,col) = bits_to_unit(position_hash(seed,b,h,row,col)) >= p
// with position_hash a chain of SplitMix64 hash_combine over (tag, b, h, row,
// col).  The (b, h) prefix is computed once per CTA and the row prefix once per
// row, so each element costs one mix64.  `u >= p` is evaluated exactly in
// integers: (h >> 11) >= ceil(p * 2^53) (computed on the host).
VATTN_DEV uint64_t mix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}
VATTN_DEV uint64_t hash_combine(uint64_t state, uint64_t v) {
    return mix64(state ^ (v + 0x9e3779b97f4a7c15ull + (state << 6) + (state >> 2)));
}
struct DropRow {
    uint64_t s;  // hash state after (tag, b, h, row)
    uint64_t k;  // 0x9e3779b97f4a7c15 + (s << 6) + (s >> 2)
};
VATTN_DEV uint64_t drop_bh_base(uint64_t seed, int b, int h) {
    return hash_combine(hash_combine(hash_combine(seed, 0x64726f70ull), static_cast<uint64_t>(b)),
                        static_cast<uint64_t>(h));
}
VATTN_DEV DropRow drop_row(uint64_t bh_base, int row) {
    DropRow r;
    r.s = hash_combine(bh_base, static_cast<uint64_t>(row));
    r.k = 0x9e3779b97f4a7c15ull + (r.s << 6) + (r.s >> 2);
    return r;
}
VATTN_DEV bool drop_keep(const DropRow& r, int col, uint64_t thresh) {
    return (mix64(r.s ^ (static_cast<uint64_t>(col) + r.k)) >> 11) >= thresh;
}
// The same decision with less integer work (the mask kernel is bound by it): with
// z = mix64(..), (z >> 11) >= thresh  <=>  z >= thresh << 11 (thresh < 2^53), and the
// high word of z decides unless it ties with that of thresh << 11 (probability 2^-32),
// so the last multiply only forms its high word; ties take the exact 64-bit path.
struct DropThresh {
    uint64_t t;       // thresh
    uint32_t hi, lo;  // thresh << 11
};
VATTN_DEV DropThresh drop_thresh_split(uint64_t thresh) {
    const uint64_t t11 = thresh << 11;
    return {thresh, static_cast<uint32_t>(t11 >> 32), static_cast<uint32_t>(t11)};
}
// 32 consecutive keys col0 .. col0 + 31 of one row at once (the mask kernel's word),
// returning the keep bits (bit b = key col0 + b) and setting `tie` when any high word
// tied (the caller then redoes the word exactly).  Per word, K = k + col0 keeps its high
// word for all 32 keys (checked: the low word does not wrap; otherwise the exact path),
// so the high word of x0 = (s ^ (K + b)) + G takes one of two values (carry of the low
// add), and so do the high words of x0 ^ (x0 >> 30) and their product with C1's low
// word: those are per-word constants selected by the carry.  Per key that leaves the
// low-word add / xor, two funnel shifts, the two 32 x 32 partial products of x1 * C1, the
// second xor-shift and the high word of x2 * C2 -- the same integers as drop_keep.
// kLowThresh (th_hi < 2^31, i.e. p < 1/2): the final z ^= z >> 31 only flips bit 0 of
// high words >= 2^31, which are above th_hi either way, so it is skipped.
//
// Issue balance (the mask kernel is bound by instruction issue, shared between the integer
// ALU pipe and the FMA pipe that runs IMAD): the low-word add's carry-out feeds the high
// word directly (add.cc / addc), hi(x1 * C1lo)'s per-word share is linear in that high
// word (one IMAD), the keys are walked downwards so each keep bit shifts in through a
// carry (w = 2 w + (zh > th_hi), two adds, no per-bit constant), the tie flag is a
// predicate AND, and the key index decrement and the >> 27 of the high word run as
// IMAD / IMAD.HI by `one` (a value the compiler cannot fold: the caller passes
// blockDim.x / 256 = 1).  ~21 SASS instructions per key against ~27 for the plain form
// (VATTN_DROPKEEP=0, kept for A/B runs).
#ifndef VATTN_DROPKEEP
#define VATTN_DROPKEEP 1
#endif
template <bool kLowThresh>
VATTN_DEV uint32_t drop_keep_word(const DropRow& r, uint32_t col0, uint32_t th_hi, uint32_t one, bool& tie, bool& wrap) {
    constexpr uint32_t kGlo = 0x7f4a7c15u, kGhi = 0x9e3779b9u;
    constexpr uint32_t kC1lo = 0x1ce4e5b9u, kC1hi = 0xbf58476du;
    constexpr uint32_t kC2lo = 0x133111ebu, kC2hi = 0x94d049bbu;
    const uint64_t K = r.k + col0;
    const uint32_t Klo = static_cast<uint32_t>(K), Khi = static_cast<uint32_t>(K >> 32);
    wrap = Klo > 0xFFFFFFFFu - 31u;
    const uint32_t slo = static_cast<uint32_t>(r.s), shi = static_cast<uint32_t>(r.s >> 32);
    const uint32_t xh = Khi ^ shi;
    const uint32_t h0a = xh + kGhi, h0b = h0a + 1u;              // high word of x0 (carry 0 / 1)
    const uint32_t h1a = h0a ^ (h0a >> 30), h1b = h0b ^ (h0b >> 30);  // high word of x1
    const uint32_t hca = h1a * kC1lo, hcb = h1b * kC1lo;          // its share of hi(x1 * C1)
#if VATTN_DROPKEEP == 0
    (void)one;
    uint32_t w = 0;
    bool t = false;
#pragma unroll 8
    for (uint32_t b = 0; b < 32; ++b) {
        const uint32_t xl = (Klo + b) ^ slo;
        const uint32_t lo0 = xl + kGlo;
        const bool c = lo0 < kGlo;                                 // carry into the high word
        const uint32_t hi0 = c ? h0b : h0a;
        const uint32_t lo1 = lo0 ^ __funnelshift_r(lo0, hi0, 30);  // x ^= x >> 30 (low word)
        const uint64_t pr = static_cast<uint64_t>(lo1) * kC1lo;
        const uint32_t lo2 = static_cast<uint32_t>(pr);
        const uint32_t hi2 = static_cast<uint32_t>(pr >> 32) + lo1 * kC1hi + (c ? hcb : hca);
        const uint32_t lo3 = lo2 ^ __funnelshift_r(lo2, hi2, 27);  // x ^= x >> 27
        const uint32_t hi3 = hi2 ^ (hi2 >> 27);
        uint32_t zh = __umulhi(lo3, kC2lo) + lo3 * kC2hi + hi3 * kC2lo;  // high word of x * C2
        if constexpr (!kLowThresh) zh ^= zh >> 31;
        t |= zh == th_hi;
        w |= static_cast<uint32_t>(zh > th_hi) << b;
    }
    tie = t;
    return w;
#else
    uint32_t hcd = hcb - hca, k2 = hca - h0a * hcd;                // hc = hi0 * hcd + k2
    asm("mov.b32 %0, %0;" : "+r"(hcd));                            // keep the compiler from
    asm("mov.b32 %0, %0;" : "+r"(k2));                             // re-expanding hc
    const uint32_t k32 = one << 5, nth = ~th_hi;                   // umulhi(x, 32) = x >> 27
    uint32_t w = 0, kb = Klo + 32u;
    bool nt = true;
#pragma unroll 8
    for (int b = 31; b >= 0; --b) {
        asm("mad.lo.u32 %0, %1, -1, %0;" : "+r"(kb) : "r"(one));  // Klo + b
        const uint32_t xl = kb ^ slo;
        uint32_t lo0, hi0;                                         // x0 = x + G
        asm("add.cc.u32 %0, %2, %3;\n\taddc.u32 %1, %4, 0;" : "=r"(lo0), "=r"(hi0) : "r"(xl), "n"(kGlo), "r"(h0a));
        const uint32_t lo1 = lo0 ^ __funnelshift_r(lo0, hi0, 30);  // x ^= x >> 30 (low word)
        const uint64_t pr = static_cast<uint64_t>(lo1) * kC1lo;
        const uint32_t lo2 = static_cast<uint32_t>(pr);
        const uint32_t hi2 = static_cast<uint32_t>(pr >> 32) + lo1 * kC1hi + (hi0 * hcd + k2);
        const uint32_t lo3 = lo2 ^ __funnelshift_r(lo2, hi2, 27);  // x ^= x >> 27
        const uint32_t hi3 = hi2 ^ __umulhi(hi2, k32);
        uint32_t zh = __umulhi(lo3, kC2lo) + lo3 * kC2hi + hi3 * kC2lo;  // high word of x * C2
        if constexpr (!kLowThresh) zh ^= zh >> 31;
        nt &= zh != th_hi;
        uint32_t sink;                                             // carry of zh + ~th_hi = (zh > th_hi)
        asm("add.cc.u32 %0, %2, %3;\n\taddc.u32 %1, %1, %1;" : "=r"(sink), "+r"(w) : "r"(zh), "r"(nth));
    }
    tie = !nt;
    return w;
#endif
}

// 32 x 32 bit transpose across a warp: lane l holds row l (bit c = column c) in, column l
// (bit r = row r) out.  Five butterfly stages of shuffles (Hacker's Delight 7-3).
VATTN_DEV uint32_t warp_transpose32(uint32_t x, int lane) {
    uint32_t m = 0x0000FFFFu;
#pragma unroll
    for (int j = 16; j >= 1; j >>= 1) {
        const uint32_t t = __shfl_xor_sync(0xffffffffu, x, j);
        x = (lane & j) ? ((x & ~m) | ((t >> j) & m)) : ((x & m) | ((t & m) << j));
        m ^= m << (j >> 1);
    }
    return x;
}

// Round to the 16-bit storage type and back (the reference narrows P once
// before dropout and once after the 1/(1-p) scaling, attention_forward.cpp:94-106).
template <bool kBF16>
VATTN_DEV float round16(float x) {
    return unpack2<kBF16>(pack2<kBF16>(x, 0.0f)).x;
}

// ------------------------------------------------ global-memory ordering --

VATTN_DEV int ld_acquire_gpu(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

VATTN_DEV void st_release_gpu(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Release-side fence for the dQ turn hand-off (lighter than __threadfence's fence.sc).
VATTN_DEV void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

VATTN_DEV void red_add_v4(float* p, float a, float b, float c, float d) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c),
                 "f"(d)
                 : "memory");
}

}  // namespace vattn_sm100
