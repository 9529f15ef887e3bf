// mha_bwd_sm100.cuh -- fused multi-head-attention backward for sm_100a.
//
// Replaces vattn::backward_fused (reference proj/src/attention_backward.cpp:59-219):
//   compute_dpsum (:44-57)           -> mha_bwd_preprocess_kernel: D = rowsum(dO o O)
//   per-(b,h,key-tile) unit (:110-211): dV += P~^T dO, dK += dS^T Q
//                                    -> mha_bwd_dkdv_kernel (key-major, 4 GEMMs / tile pair)
//   dQ master buffer + atomic adds (DqAccumulator, :22-42, :205, :215)
//                                    -> mha_bwd_dq_kernel (query-major, 3 GEMMs / tile pair):
//      each CTA owns one 128-row query tile and accumulates dQ = sum_j dS_j K_j
//      over the key tiles in ascending j inside tensor memory, then rounds once.
//      Deterministic by construction (fixed order, no atomics, no fp32 workspace);
//      costs the recompute of S and dP (2 extra GEMMs) instead of 64 KiB of L2
//      reduce-adds per (key tile, query tile) pair, which measured as the
//      bottleneck of a fused design ("dQ").
//
// Arithmetic contract (both kernels): P = exp2(S*scale*log2e - lse*log2e), the
// 16-bit operands P~ and dS are rounded once, dS = P o (dP - D) (fp32), and the
// softmax scale is applied to dK / dQ in fp32 before their single rounding.
#pragma once

#include "sm100_ptx.cuh"

namespace vattn_sm100 {

// ------------------------------------------------------------ preprocess --

// D = rowsum(dO o O) (compute_dpsum), lse2 = lse * log2(e); both padded to Npad
// (+inf / 0) so 128-row tiles never read past a head.  HBM-bound: every thread
// loads 16 bytes of O and of dO per row (kD / 8 threads per row, so a warp covers
// 32 * 8 / kD contiguous rows), products summed in fp32 and reduced over the row's
// lanes with shuffles.
template <int kD, bool kBF16>
__global__ void __launch_bounds__(256) mha_bwd_preprocess_kernel(
    const void* __restrict__ o, const void* __restrict__ dout, const float* __restrict__ lse,
    float* __restrict__ lse2, float* __restrict__ dsum, int N, int Npad, int BH, int* __restrict__ zero = nullptr,
    int zero_n = 0) {
    griddep_start();
    using T16 = typename std::conditional<kBF16, __nv_bfloat16, __half>::type;
    constexpr int kLanesPerRow = kD / 8;
    constexpr int kRowsPerWarp = 32 / kLanesPerRow;
    constexpr int kU = 4;  // rows per thread per iteration: 2 * kU 16-byte loads in flight
    const int lane = threadIdx.x & 31;
    const int sub = lane % kLanesPerRow;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    const long long rows = static_cast<long long>(BH) * Npad;
    griddep_wait();  // O / lse come from the forward kernel
    // the dQ hand-off words of this backward (BwdParams::dq_sync): the dK/dV kernel reads
    // them only after its griddep_wait, i.e. after this grid completed
    if (zero && blockIdx.x == 0)
        for (int x = threadIdx.x; x < zero_n; x += blockDim.x) zero[x] = 0;
    for (long long r0 = static_cast<long long>(gw) * kRowsPerWarp * kU; r0 < rows;
         r0 += static_cast<long long>(nwarps) * kRowsPerWarp * kU) {
        long long row[kU];
        int bh[kU], n[kU];
        bool valid[kU];
        uint4 a[kU], g[kU];
        // one division per pass (the pass's rows are consecutive; a row past the end of a
        // head moves to the next)
        const int bh0 = static_cast<int>(r0 / Npad);
        const int n0 = static_cast<int>(r0 - static_cast<long long>(bh0) * Npad);
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            row[u] = r0 + u * kRowsPerWarp + lane / kLanesPerRow;
            bh[u] = bh0;
            n[u] = n0 + u * kRowsPerWarp + lane / kLanesPerRow;
            while (n[u] >= Npad) {  // at most once unless Npad < 32 / (d / 8) * 4 (mha_dpsum, tiny N)
                n[u] -= Npad;
                ++bh[u];
            }
            valid[u] = row[u] < rows && n[u] < N;
            a[u] = g[u] = make_uint4(0u, 0u, 0u, 0u);
            if (valid[u]) {
                const size_t base = (static_cast<size_t>(bh[u]) * N + n[u]) * kD + sub * 8;
                a[u] = *reinterpret_cast<const uint4*>(reinterpret_cast<const T16*>(o) + base);
                g[u] = *reinterpret_cast<const uint4*>(reinterpret_cast<const T16*>(dout) + base);
            }
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const uint32_t av[4] = {a[u].x, a[u].y, a[u].z, a[u].w}, gv[4] = {g[u].x, g[u].y, g[u].z, g[u].w};
            float acc = 0.0f;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float2 x = unpack2<kBF16>(av[e]), y = unpack2<kBF16>(gv[e]);
                acc = fmaf(y.x, x.x, acc);
                acc = fmaf(y.y, x.y, acc);
            }
#pragma unroll
            for (int off = kLanesPerRow / 2; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
            if (sub == 0 && row[u] < rows) {
                dsum[row[u]] = valid[u] ? acc : 0.0f;
                if (lse2)
                    lse2[row[u]] = valid[u] ? lse[static_cast<size_t>(bh[u]) * N + n[u]] * 1.4426950408889634f : INFINITY;
            }
        }
    }
    if (!kPdlEarly) griddep_launch_dependents();
}

struct BwdParams {
    const float* lse2;  // [BH, Npad]
    const float* dsum;  // [BH, Npad]
    int N, Npad, n_q;
    int causal;
    float scale;        // softmax scale (applied to dK / dQ)
    float scale_log2;   // scale * log2(e)
    int H;              // heads (dropout hash uses b and h separately)
    int bh_off;         // global index of this launch's first (b, h) unit (slabs)
    float inv_keep;     // 1 / (1 - dropout_p)
    uint64_t drop_seed;
    uint64_t drop_thresh;
    // dS materialisation (optional): the dK/dV kernel also writes every dS^T tile
    // (16-bit, [128 keys][128 queries]) here and dQ = dS K becomes a streaming GEMM
    // (mha_bwd_dq_gemm_kernel) instead of the recomputing dQ kernel.  nullptr = off.
    uint16_t* ds_out;
    long long ds_tiles_per_bh;  // n_q^2, or n_q (n_q + 1) / 2 causal (lower triangle)
    int tail_units;             // dK/dV grid: last units dispatched longest-first (grid_item_tail)
    // Dropout keep bits written by mha_dropmask_kernel (nullptr = hash in place):
    // query-major [unit][query][Npad/32 words] (bit = key) and the key-major copy
    // [unit][key][Npad/32 words] (bit = query).
    const uint32_t* drop_mask;
    const uint32_t* drop_mask_k;
    // dQ overlapped with dK/dV (ds_out only): the first dq_workers CTAs of the dK/dV grid
    // run the dQ GEMM over units whose dS^T tiles are complete; the rest of the grid is
    // the dK/dV items.  dq_sync = [0] next dQ item, [1] finished dK/dV CTAs, [2 + u]
    // finished dS^T stores of unit u (2 per key tile).  nullptr = dQ is a separate launch.
    int* dq_sync;
    int dq_workers;
    int dkdv_ctas;
    int n_units;        // (b, h) units of this launch
    int ds_signals;     // dS^T store-done signals per unit (store threads per key tile x n_q)
    int dkdv_items;     // (unit, key tile) items of the dK/dV grid; a CTA takes items
                        // cta, cta + G, ... (G = its CTAs) -- persistent when G < items
};

// Dropout keep bits, hashed once per step ahead of the forward: the reference's
// position hash (rng.cpp:35-54) is data-independent, so it runs in its own
// integer-bound kernel at full occupancy instead of on the forward's softmax critical
// path (where it cost ~5 ms at C3).  Two copies, each B*H*Npad^2/8 bytes:
//   query-major  mask[unit][query][Npad/32]  bit = key    (forward, dQ recompute)
//   key-major    mask[unit][key][Npad/32]    bit = query  (dK/dV: thread = key row)
// CTA = one 128 x 128 (query tile, key tile) pair of one (b, h) unit; warp w hashes
// queries 32 (w & 3) + lane against keys 64 (w >> 2) + [0, 64) (drop_keep_word: the
// hash with per-word constants); a five-stage shuffle transpose per 32 x 32 block makes
// the key-major words, staged in shared memory so both copies leave as 16-byte stores.  Causal: tile pairs above the diagonal are skipped (masked positions; no
// kernel reads their bits).
__global__ void __launch_bounds__(256) mha_dropmask_kernel(uint32_t* __restrict__ mask, int Npad, int H, int bh_off,
                                                           uint64_t seed, uint64_t thresh, int causal) {
    griddep_start();
    __shared__ uint32_t qm[128][5];  // [query][key word] (+1 pad)
    __shared__ uint32_t km[128][5];  // [key][query word]
    const int nt = Npad / 128, W = Npad / 32;
    int i, j;  // query tile, key tile
    const int t = blockIdx.x;
    if (causal) {  // t -> (i, j <= i), row-major over the lower triangle
        i = static_cast<int>((sqrtf(8.0f * static_cast<float>(t) + 1.0f) - 1.0f) * 0.5f);
        while (i * (i + 1) / 2 > t) --i;
        while ((i + 1) * (i + 2) / 2 <= t) ++i;
        j = t - i * (i + 1) / 2;
    } else {
        i = t / nt;
        j = t - i * nt;
    }
    const int bh = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int qs = warp & 3, kh = warp >> 2;
    griddep_wait();
    const DropRow dr = drop_row(drop_bh_base(seed, (bh + bh_off) / H, (bh + bh_off) % H), i * 128 + qs * 32 + lane);
    const DropThresh th = drop_thresh_split(thresh);
    const uint32_t one = blockDim.x / 256u;  // always 256 threads: 1, opaque to the compiler (drop_keep_word)
#pragma unroll
    for (int c = 0; c < 2; ++c) {
        const int kw = kh * 2 + c;  // key word within the tile
        const uint32_t col0 = static_cast<uint32_t>(j * 128 + kw * 32);
        bool tie, wrap;
        uint32_t w = th.hi < 0x80000000u ? drop_keep_word<true>(dr, col0, th.hi, one, tie, wrap)
                                         : drop_keep_word<false>(dr, col0, th.hi, one, tie, wrap);
        if (tie || wrap) {  // a high word tied (p ~ 2^-32 per position) or K's low word wraps: exact
            w = 0;
#pragma unroll 1
            for (int b = 0; b < 32; ++b) w |= static_cast<uint32_t>(drop_keep(dr, static_cast<int>(col0) + b, thresh)) << b;
        }
        qm[qs * 32 + lane][kw] = w;
        km[kw * 32 + lane][qs] = warp_transpose32(w, lane);  // key kw*32 + lane, bit = query
    }
    __syncthreads();
    const size_t base = static_cast<size_t>(bh) * Npad;
    const size_t half = static_cast<size_t>(gridDim.y) * Npad * W;  // words per copy
    if (threadIdx.x < 128) {
        const int r = threadIdx.x;
        *reinterpret_cast<uint4*>(mask + (base + i * 128 + r) * W + j * 4) = make_uint4(qm[r][0], qm[r][1], qm[r][2], qm[r][3]);
    } else {
        const int r = threadIdx.x - 128;
        *reinterpret_cast<uint4*>(mask + half + (base + j * 128 + r) * W + i * 4) =
            make_uint4(km[r][0], km[r][1], km[r][2], km[r][3]);
    }
    if (!kPdlEarly) griddep_launch_dependents();
}

// Index of dS^T tile (query tile i, key tile kb) within one (b, h).
VATTN_DEV long long ds_tile_index(const BwdParams& p, int i, int kb) {
    return p.causal ? static_cast<long long>(i) * (i + 1) / 2 + kb : static_cast<long long>(i) * p.n_q + kb;
}

// ============================================================ dQ GEMM ==
//
// dQ_i = sum_j dS_ij K_j from the dS^T tiles the dK/dV kernel materialised (d = 128, or
// d = 64 with N <= 1024): A = dS^T tile (MN-major), B = K_j (MN-major), accumulated in
// tensor memory in ascending j (the reference's DqAccumulator order) and rounded once.
template <int kD>
struct DqGemmCfg {
    static constexpr int kKBytes = kD * 128 * 2;
    static constexpr int kDsBytes = 128 * 128 * 2;
    static constexpr int kStageBytes = kKBytes + kDsBytes;
    static constexpr int kStages = kD == 128 ? 3 : 4;
    static constexpr int kSmemOut = kStages * kStageBytes;       // persistent worker: dQ staging
    static constexpr int kSmemBar = kSmemOut + kD * 128 * 2;
    static constexpr int kNumBars = 2 * kStages + 1;
    static constexpr int kSmemBytes = kSmemBar + kNumBars * 8 + 16;
};

VATTN_DEV void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

// Persistent dQ worker (256 threads: warp 0 TMA, warp 1 MMA, warp 2 TMEM, warps 4-7
// epilogue).  Items = (unit, query tile), unit-major, longest causal tile first, taken
// from the atomic counter dq_sync[0].  `early` workers are CTAs of the dK/dV grid: they
// wait until every dS^T store of the item's unit is done (dq_sync[2 + u]) and stop
// taking items once all dK/dV CTAs have finished (dq_sync[1]), leaving the rest to the
// full-width mha_bwd_dq_tail_kernel launched after the dK/dV grid.  Same arithmetic and
// accumulation order as one dQ tile per CTA: results are bitwise identical.
template <int kD, bool kBF16>
VATTN_DEV void dq_worker(const CUtensorMap* tm_ds, const CUtensorMap* tm_k, const CUtensorMap* tm_dq, const BwdParams& p,
                         uint8_t* smem, bool early) {
    using Cfg = DqGemmCfg<kD>;
    constexpr int S = Cfg::kStages;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::kSmemBar);
    uint64_t* full = bars;
    uint64_t* empty = bars + S;
    uint64_t* dq_done = bars + 2 * S;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + Cfg::kNumBars);
    volatile int* s_item = reinterpret_cast<volatile int*>(tmem_slot + 1);  // [2]
    const int warp = warp_id();
    const int lane = lane_id();
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
        }
        mbar_init(dq_done, 1);
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc<kD>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    griddep_wait();  // dq_sync zeroed / dS^T written by the previous kernels in the stream
    const int nq = p.n_q;
    const int total = p.n_units * nq;
    uint32_t pos = 0, it = 0;  // ring position (tiles) and items done by this CTA
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(tm_ds);
        tma_prefetch_desc(tm_k);
        tma_prefetch_desc(tm_dq);
    }
    // Items come from the atomic counter (thread 0 = the producer lane).  The producer
    // takes the NEXT item as soon as it has issued the current one's loads and prefetches
    // its first min(S, tiles) dS^T / K tiles into the ring stages this item's MMAs free,
    // so those loads run under this item's epilogue instead of after the CTA barrier
    // (s_item: two slots, the next item's published before the end-of-item barrier).
    auto fetch = [&]() -> int {
        int item = -1;
        if (!early || ld_acquire_gpu(p.dq_sync + 1) < p.dkdv_ctas) {
            item = atomicAdd(p.dq_sync, 1);
            if (item >= total) {
                item = -1;
            } else if (early) {
                const int* cnt = p.dq_sync + 2 + item / nq;
                const uint64_t t0 = globaltimer_ns();
                while (ld_acquire_gpu(cnt) < p.ds_signals) {
                    __nanosleep(500);
                    if (VATTN_WATCHDOG_NS && globaltimer_ns() - t0 > VATTN_WATCHDOG_NS) __trap();
                }
                fence_proxy_async_global();  // the TMA loads below see the dS^T stores
            }
        }
        return item;
    };
    auto decode = [&](int item, int& bh, int& i, int& nk) {
        bh = item / nq;
        const int tile = item - bh * nq;
        i = p.causal ? (nq - 1 - tile) : tile;
        nk = p.causal ? i + 1 : nq;
    };
    auto issue = [&](int bh, int i, uint32_t q, int j) {  // dS^T tile (i, j) and K_j into ring slot q
        const int st = q % S;
        mbar_wait<VATTN_SLEEP_PRODUCER>(empty + st, ((q / S) & 1) ^ 1);
        mbar_arrive_expect_tx(full + st, Cfg::kStageBytes);
        uint8_t* ds = smem + st * Cfg::kStageBytes;
        uint8_t* kt = ds + Cfg::kDsBytes;
        const int tl = static_cast<int>(static_cast<long long>(bh) * p.ds_tiles_per_bh + ds_tile_index(p, i, j));
        tma_load_3d(ds, tm_ds, full + st, 0, 0, tl);
        tma_load_3d(ds + 16384, tm_ds, full + st, 64, 0, tl);
        for (int b = 0; b < kD / 64; ++b) tma_load_3d(kt + b * 16384, tm_k, full + st, b * 64, j * 128, bh);
    };
    if (threadIdx.x == 0) s_item[0] = fetch();
    __syncthreads();
    int pre = 0;  // producer: tiles of the current item issued during the previous one
    for (;;) {
        const int item = s_item[it & 1];
        if (item < 0) break;
        int bh, i, nk;
        decode(item, bh, i, nk);
        if (warp == 0) {
            if (lane == 0) {
                for (int j = pre; j < nk; ++j) issue(bh, i, pos + j, j);
                const int nxt = fetch();
                s_item[(it + 1) & 1] = nxt;
                pre = 0;
                if (nxt >= 0) {
                    int bh2, i2, nk2;
                    decode(nxt, bh2, i2, nk2);
                    pre = nk2 < S ? nk2 : S;
                    for (int j = 0; j < pre; ++j) issue(bh2, i2, pos + nk + j, j);
                }
            }
        } else if (warp == 1) {
            constexpr uint32_t idesc = umma_idesc_f16(128, kD, kBF16, 1, 1);  // A = dS (MN-major), B = K (MN-major)
            const uint64_t dA0 = umma_desc_sw128(smem_u32(smem), 16384, 1024);
            const uint64_t dB0 = umma_desc_sw128(smem_u32(smem + Cfg::kDsBytes), 16384, 1024);
            constexpr uint64_t kStage16 = Cfg::kStageBytes >> 4;
            for (int j = 0; j < nk; ++j) {
                const uint32_t q = pos + j;
                const int st = q % S;
                mbar_wait_mma(full + st, (q / S) & 1);
                tc_fence_after();
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    mma_ss_e(tmem, desc_mnmajor(dA0 + st * kStage16, kk), desc_mnmajor(dB0 + st * kStage16, kk), idesc,
                             (j > 0 || kk > 0) ? 1u : 0u);
                mma_commit_e(empty + st);
            }
            mma_commit_e(dq_done);
        } else if (warp >= 4 && warp < 8) {
            // dQ * scale -> 16-bit -> swizzled staging -> TMA store
            const int r = ((warp & 3) << 5) + lane;
            const uint32_t lb = static_cast<uint32_t>((warp & 3) * 32) << 16;
            uint8_t* sOut = smem + Cfg::kSmemOut;
            if (warp == 4 && lane == 0) bulk_wait_read0();  // the previous item's store left the staging
            mbar_wait<VATTN_SLEEP_MATH>(dq_done, it & 1);
            tc_fence_after();
            named_bar_sync(1, 128);
#pragma unroll
            for (int c = 0; c < kD / 32; ++c) {
                float a[32];
                tmem_ld32f(tmem + lb + 32 * c, a);
                tmem_wait_ld();
#pragma unroll
                for (int x = 0; x < 4; ++x) {
                    uint4 v;
                    v.x = pack2<kBF16>(a[8 * x + 0] * p.scale, a[8 * x + 1] * p.scale);
                    v.y = pack2<kBF16>(a[8 * x + 2] * p.scale, a[8 * x + 3] * p.scale);
                    v.z = pack2<kBF16>(a[8 * x + 4] * p.scale, a[8 * x + 5] * p.scale);
                    v.w = pack2<kBF16>(a[8 * x + 6] * p.scale, a[8 * x + 7] * p.scale);
                    const int cc = 32 * c + 8 * x;
                    st_swz128(sOut + (cc >> 6) * 16384, r, (cc & 63) >> 3, v);
                }
            }
            fence_proxy_async_smem();
            named_bar_sync(1, 128);
            if (warp == 4 && lane == 0) {
                for (int b = 0; b < kD / 64; ++b) tma_store_3d(tm_dq, sOut + b * 16384, b * 64, i * 128, bh);
                bulk_commit();
            }
        }
        pos += static_cast<uint32_t>(nk);
        ++it;
        tc_fence_before();
        __syncthreads();  // TMEM read out before the next item's first MMA; s_item reuse
        tc_fence_after();
    }
    if (warp == 4 && lane == 0) bulk_wait_read0();  // no store reads smem past exit
    if (!kPdlEarly) griddep_launch_dependents();
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<kD>(tmem);
    }
}

// Full-width tail of the overlapped dQ: every unit is complete when it starts.
template <int kD, bool kBF16>
__global__ void __launch_bounds__(256, 1)
    mha_bwd_dq_tail_kernel(const __grid_constant__ CUtensorMap tm_ds, const __grid_constant__ CUtensorMap tm_k,
                           const __grid_constant__ CUtensorMap tm_dq, const BwdParams p) {
    griddep_start();
    extern __shared__ __align__(1024) uint8_t smem[];
    dq_worker<kD, kBF16>(&tm_ds, &tm_k, &tm_dq, p, smem, false);
}

// ================================================================ dK / dV ==
//
// One CTA = one (b*h, 128-key tile).  Loop over query tiles i (causal: from the
// diagonal).  Per tile:   S^T = K Q_i^T      (SS -> TMEM region S)
//                         P^T = exp2(S^T c - lse2)  (registers; 16-bit -> region S)
//                         dP^T = V dO_i^T    (SS -> TMEM region DP)
//                         dS^T = P^T o (dP^T - D)   (registers; 16-bit -> region DP)
//                         dV += P^T dO_i     (TS)
//                         dK += dS^T Q_i     (TS)
// MMA order per tile: dV_i, S_(i+1), dK_i, dP_(i+1): the P pass of tile i+1
// overlaps dK_i + dP_(i+1); the dS pass overlaps dV_(i+1) + S_(i+2).
// Warps: 0 TMA, 1 MMA, 2 TMEM alloc, 4-11 two warpgroups (thread = key row;
// warpgroup h owns query columns [64h, 64h+64)).
// d = 64 frees tensor memory for a second S^T region: S_(i+2) is computed while
// the P pass of tile i+1 runs, so the P pass never waits for S (with a third Q/dO
// stage so the load of Q_(i+2) does not wait for dK_i).  d = 128 keeps one region.
// Math warpgroups of the dK/dV kernel (2: 64 query columns each; 4: 32 each, 640
// threads).  Measured (profiles/r2_experiments.md): 4 is slower at both head dims --
// d = 64 +6..14 %, d = 128 (C3) +11 % per dK/dV launch -- the step is not bound by the
// math warps' latency, so the knobs stay at 2.
#ifndef VATTN_DKDV64_WG
#define VATTN_DKDV64_WG 2
#endif
#ifndef VATTN_DKDV128_WG
#define VATTN_DKDV128_WG 2
#endif
template <int kD>
struct DkdvCfg;
// dS^T materialisation per warp (VATTN_DS_WARP_STORE, default on): each math warp stages
// its 32 key rows and issues their TMA store itself, so the staging needs only __syncwarp
// instead of two named barriers over the warpgroup per step.  Needs one warpgroup per
// 64-query box (kQW = 64).
#ifndef VATTN_DS_WARP_STORE
#define VATTN_DS_WARP_STORE 1
#endif
template <int kD>
struct DkdvCfg {
    static constexpr bool kDoubleS = kD == 64;
    static constexpr int kWG = kD == 64 ? VATTN_DKDV64_WG : VATTN_DKDV128_WG;  // math warpgroups
    static constexpr int kQW = 128 / kWG;                        // query columns per warpgroup
    static constexpr int kHalves = kQW == 64 ? 2 : 1;            // P^T publication chunks per warpgroup
    static constexpr int kThreads = 128 + 128 * kWG;
    // register split (setmaxnreg): producer / MMA / allocator warps vs math warps.  The
    // split redistributes the CTA's launch allocation (kThreads x the launch-bound
    // register count: 168 at 384 threads, 96 at 640), so 128 lo + 128 kWG hi must fit it.
    static constexpr uint32_t kRegsLo = kWG == 2 ? 88 : 56;
    static constexpr uint32_t kRegsHi = kWG == 2 ? 208 : 104;
    static_assert(128 * kRegsLo + 128 * kWG * kRegsHi <= kThreads * (kWG == 2 ? 168 : 96), "register split");
    static constexpr int kTileBytes = kD * 128 * 2;
    static constexpr int kBoxes = kD / 64;
    static constexpr int kStages = kDoubleS ? 3 : 2;
    static constexpr int kSmemK = 0;
    static constexpr int kSmemV = kTileBytes;
    static constexpr int kSmemQ = 2 * kTileBytes;
    static constexpr int kSmemDO = kSmemQ + kStages * kTileBytes;
    static constexpr int kSmemLD = kSmemDO + kStages * kTileBytes;  // [stage][lse2 128 | D 128]
    static constexpr int kSmemDrop = kSmemLD + kStages * 1024;      // dropout row hashes [128] x 16 B
    // dS^T staging for its TMA store (dS materialisation, 2 boxes of 64 queries x 128
    // keys).  It overlaps the dropout row-hash buffer, which is only used when dropout
    // bits are hashed in place (no keep-bit mask) -- and then materialisation is off.
    static constexpr int kSmemDsStage = kSmemDrop;
    static constexpr int kSmemBar = kSmemDsStage + 32768;
    // kv_full, q_full/q_empty [kStages], s_full (x2 double S), dp_full, p_full, ds_full,
    // dkv_full, ld_full [kStages] (CTA pair: lse2 / D of this CTA; Q / dO count on the
    // leader's q_full)
    static constexpr int kNumBars = 1 + 2 * kStages + 2 + 1 + 2 * kWG * kHalves + kWG + 1 + kStages + 1;  // + acc_free
    static constexpr int kSmemBytes = kSmemBar + kNumBars * 8 + 16;
    static constexpr uint32_t kTmemS = 0;                       // region r at 128 r
    static constexpr uint32_t kTmemDP = kDoubleS ? 256 : 128;
    static constexpr uint32_t kTmemDV = kTmemDP + 128, kTmemDK = kTmemDV + kD;
};
template <int kD>
constexpr bool kDsWarpStore = VATTN_DS_WARP_STORE != 0 && DkdvCfg<kD>::kQW == 64;

// kPair (d = 128): a (2,1,1) cluster = two adjacent key tiles of one unit sharing
// every query tile.  All four GEMMs run as cta_group::2 M = 256 MMAs issued by the
// leader: each CTA's A rows (K, V, P^T, dS^T) stay its own, and each CTA supplies half
// of the B operand, so the per-SM shared-memory operand reads per step fall from 192
// to 128 KiB (the SS GEMMs at N = 128 saturate the 128 B/clk shared-memory port,
// profiles/r2_experiments.md).  B halves must sit at the same offset in both CTAs:
// a Q / dO stage holds [queries 0..127 x d-half r] (16 KB, the MN-major B of dK / dV)
// and [queries 64r..64r+63 x d 0..127] (2 x 8 KB, the K-major B of S^T / dP^T).
// The math warps are unchanged (thread = key row of their own CTA); their P^T / dS^T
// publications arrive on the leader's barriers.
// kMulti: persistent CTAs looping over several items (host: N <= 1024); false compiles the
// one-item-per-CTA kernel with every item-loop variable constant (measured: the generic
// loop cost 3 % at C3 and 17 % with dropout).
template <int kD, bool kBF16, bool kDrop, bool kPair = false, bool kMulti = false>
__global__ void __launch_bounds__(DkdvCfg<kD>::kThreads, 1)
    mha_bwd_dkdv_kernel(const __grid_constant__ CUtensorMap tm_q,
                        const __grid_constant__ CUtensorMap tm_k,
                        const __grid_constant__ CUtensorMap tm_v,
                        const __grid_constant__ CUtensorMap tm_do,
                        const __grid_constant__ CUtensorMap tm_ds,
                        const __grid_constant__ CUtensorMap tm_q64,   // 64-row boxes (kPair)
                        const __grid_constant__ CUtensorMap tm_do64,  // 64-row boxes (kPair)
                        const __grid_constant__ CUtensorMap tm_dq,    // dQ (dq_workers > 0)
                        void* __restrict__ dk_out, void* __restrict__ dv_out, const BwdParams p) {
    VCTA(1, 0);
    griddep_start();
    using Cfg = DkdvCfg<kD>;
    static_assert(!kPair || (kD == 128 && !Cfg::kDoubleS), "CTA pair: d = 128 only");
    static_assert(!(kPair && kMulti), "CTA pairs take one item");
    if constexpr (!kPair) {  // the grid's first dq_workers CTAs overlap the dQ GEMM (see dq_worker)
        if (static_cast<int>(blockIdx.x) < p.dq_workers) {
            extern __shared__ __align__(1024) uint8_t smem_dq[];
            dq_worker<kD, kBF16>(&tm_ds, &tm_k, &tm_dq, p, smem_dq, true);
            return;
        }
    }
    constexpr int kVtraceKid = 1;
    (void)kVtraceKid;
    using T16 = typename std::conditional<kBF16, __nv_bfloat16, __half>::type;
    constexpr int kSt = Cfg::kStages;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* sK = smem + Cfg::kSmemK;
    uint8_t* sV = smem + Cfg::kSmemV;
    uint8_t* sQ = smem + Cfg::kSmemQ;
    uint8_t* sDO = smem + Cfg::kSmemDO;
    float* sLD = reinterpret_cast<float*>(smem + Cfg::kSmemLD);
    DropRow* sDrop = reinterpret_cast<DropRow*>(smem + Cfg::kSmemDrop);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::kSmemBar);
    uint64_t* kv_full = bars;
    uint64_t* q_full = bars + 1;          // [kSt]
    uint64_t* q_empty = q_full + kSt;     // [kSt]
    constexpr bool kDB = Cfg::kDoubleS;
    uint64_t* s_full = q_empty + kSt;     // [kDB ? 2 : 1] per S region
    uint64_t* dp_full = s_full + (kDB ? 2 : 1);
    // p_full[s & 1][warpgroup]: one barrier per step parity.  With the double S region
    // (d = 64) a warpgroup may publish P^T_(s+1) before the MMA warp consumed its P^T_s
    // phase (S_(s+1) is issued a step early); on a single barrier that second phase
    // aliases the first under parity waits (the MMA then waits for phase s + 2 -> hang)
    // and the early arrival can complete phase s before a slow warp of the same
    // warpgroup wrote its rows (race).  Two barriers keep every phase distinct: a
    // warpgroup can never run two steps ahead (dP_(s+1) needs dK_s, i.e. all of dS_s).
    // With 64 query columns a warpgroup publishes its P^T in two 32-query halves
    // (p_full[s & 1][wg][half]): the dV MMA starts on the first half while the second is
    // exponentiated.
    constexpr int kWG = Cfg::kWG, kQW = Cfg::kQW, kHv = Cfg::kHalves;
    uint64_t* p_full = dp_full + 1;              // [2][warpgroup][half]
    uint64_t* ds_full = p_full + 2 * kWG * kHv;  // [warpgroup]
    uint64_t* dkv_full = ds_full + kWG;
    // lse2 / D of a stage: the CTA pair's own barrier (its Q / dO bytes count on the
    // leader's q_full); one CTA: part of q_full
    uint64_t* ld_full = kPair ? dkv_full + 1 : q_full;  // [kSt]
    // persistent CTAs: the epilogue has read dV / dK out of tensor memory (the next item's
    // first dV / dK MMAs overwrite them)
    uint64_t* acc_free = dkv_full + 1 + kSt;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + Cfg::kNumBars);

    const int warp = warp_id();
    const int lane = lane_id();
    const uint32_t rank = kPair ? cluster_rank() : 0u;  // 0 = leader (issues the MMAs)
    // Items: (unit, key tile), in the dispatch order of grid_item_tail (causal: the key
    // tiles with the most query tiles first); CTA c takes items c, c + G, c + 2G, ...
    const int N = p.N;
    const int cta = static_cast<int>(blockIdx.x) - p.dq_workers;
    const int G = static_cast<int>(gridDim.x) - p.dq_workers;
    struct Item {
        int bh, kb, i0, n_steps;
    };
    auto item_at = [&](int it, Item& x) -> bool {
        if constexpr (kPair) {  // cluster c = key tiles (2 pr, 2 pr + 1) of unit bh; one item per cluster
            if (it > 0) return false;
            int pr;
            grid_item_tail_n(static_cast<int>(blockIdx.x >> 1), static_cast<int>(gridDim.x >> 1), (p.n_q + 1) >> 1,
                             p.tail_units, x.bh, pr);
            x.kb = 2 * pr + static_cast<int>(rank);
        } else {
            if (!kMulti && it > 0) return false;
            const int L = kMulti ? cta + it * G : cta;
            if (kMulti && !p.causal && L >= p.dkdv_items) return false;
            if (kMulti && p.causal) {
                // causal items differ n_q-fold in length: hand them out longest first (key
                // tile-major) in a zigzag over the CTAs, so every CTA's total is balanced
                // (short heads only: a key tile of every unit fits in L2 at once)
                const int units_ = p.dkdv_items / p.n_q;
                const int idx = (it & 1) ? it * G + (G - 1 - cta) : L;
                if (idx >= p.dkdv_items) return false;
                x.kb = idx / units_;
                x.bh = idx - x.kb * units_;
            } else {
                grid_item_tail_n(L, p.dkdv_items, p.n_q, p.tail_units, x.bh, x.kb);
            }
        }
        // causal: both CTAs of a pair start at the lower key tile's diagonal (the upper
        // tile's first query tile is fully masked)
        x.i0 = p.causal ? (kPair ? (x.kb & ~1) : x.kb) : 0;
        x.n_steps = p.n_q - x.i0;
        return true;
    };
    // a math warp's arrival on a barrier the MMA issuer waits on (the leader's for a pair)
    auto arrive_mma = [&](uint64_t* bar) {
        if constexpr (kPair)
            mbar_arrive_cluster(mapa_u32(bar, 0));
        else
            mbar_arrive(bar);
    };

    if (threadIdx.x == 0) {
        if ((smem_u32(smem) & 1023u) != 0) __trap();
        mbar_init(kv_full, 1);
        for (int s = 0; s < kSt; ++s) {
            mbar_init(q_full + s, 1);
            mbar_init(q_empty + s, 1 + 4 * kWG);  // MMA commit + every math warp done with lse2/D
        }
        mbar_init(s_full, 1);
        if (kDB) mbar_init(s_full + 1, 1);
        mbar_init(dp_full, 1);
        // one arrive per warp of the warpgroup (of both CTAs for a pair)
        for (int x = 0; x < 2 * kWG * kHv; ++x) mbar_init(p_full + x, kPair ? 8 : 4);
        for (int x = 0; x < kWG; ++x) mbar_init(ds_full + x, kPair ? 8 : 4);
        mbar_init(dkv_full, 1);
        if (kPair)
            for (int s = 0; s < kSt; ++s) mbar_init(ld_full + s, 1);
        mbar_init(acc_free, 4 * kWG);  // one arrive per math warp
        fence_barrier_init();
    }
    if constexpr (kPair) {
        if (warp == 2) tmem_alloc_pair<512>(tmem_slot);
        tc_fence_before();
        cluster_sync_all();  // the peer's barriers are initialised before any remote arrive
    } else {
        if (warp == 2) tmem_alloc<512>(tmem_slot);
        tc_fence_before();
        __syncthreads();
    }
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    griddep_wait();  // inputs written by the previous kernel in the stream are visible
    if (warp < 4) regs_dec<Cfg::kRegsLo>();

    if (warp == 0) {
        // ------------------------------------------------------ TMA producer
        if (lane == 0) {
            tma_prefetch_desc(&tm_q);
            tma_prefetch_desc(&tm_k);
            tma_prefetch_desc(&tm_v);
            tma_prefetch_desc(&tm_do);
            if constexpr (kPair) {
                tma_prefetch_desc(&tm_q64);
                tma_prefetch_desc(&tm_do64);
            }
            uint32_t g0 = 0;  // steps of this CTA's earlier items (ring position)
            Item x;
            for (int it = 0; item_at(it, x); ++it) {
                const int bh = x.bh, kb = x.kb;
                if (it > 0) mbar_wait(dkv_full, (it - 1) & 1);  // the previous item's MMAs are done with K / V
                if constexpr (kPair) {
                    // K, V of both CTAs count on the leader's kv_full
                    const uint32_t kv_cl = mapa_u32(kv_full, 0);
                    if (rank == 0) mbar_arrive_expect_tx(kv_full, 4 * Cfg::kTileBytes);
                    for (int b = 0; b < Cfg::kBoxes; ++b) {
                        tma_load_3d_pair(sK + b * 16384, &tm_k, kv_cl, b * 64, kb * 128, bh);
                        tma_load_3d_pair(sV + b * 16384, &tm_v, kv_cl, b * 64, kb * 128, bh);
                    }
                } else {
                    mbar_arrive_expect_tx(kv_full, 2 * Cfg::kTileBytes);
                    for (int b = 0; b < Cfg::kBoxes; ++b) {
                        tma_load_3d(sK + b * 16384, &tm_k, kv_full, b * 64, kb * 128, bh);
                        tma_load_3d(sV + b * 16384, &tm_v, kv_full, b * 64, kb * 128, bh);
                    }
                }
                for (int s = 0; s < x.n_steps; ++s) {
                    const uint32_t g = g0 + s;
                    const int st = g % kSt;
                    const int i = x.i0 + s;
                    stress_delay(4, s);
                    mbar_wait(q_empty + st, ((g / kSt) & 1) ^ 1);
                    uint8_t* q_st = sQ + st * Cfg::kTileBytes;
                    uint8_t* do_st = sDO + st * Cfg::kTileBytes;
                    if constexpr (kPair) {
                        // [all 128 queries x d-half r] then [queries 64r.. +64 x d 0..127] (2 boxes)
                        const uint32_t q_cl = mapa_u32(q_full + st, 0);
                        if (rank == 0) mbar_arrive_expect_tx(q_full + st, 4 * Cfg::kTileBytes);
                        const int r64 = static_cast<int>(rank) * 64;
                        tma_load_3d_pair(q_st, &tm_q, q_cl, r64, i * 128, bh);
                        tma_load_3d_pair(do_st, &tm_do, q_cl, r64, i * 128, bh);
                        for (int b = 0; b < 2; ++b) {
                            tma_load_3d_pair(q_st + 16384 + b * 8192, &tm_q64, q_cl, b * 64, i * 128 + r64, bh);
                            tma_load_3d_pair(do_st + 16384 + b * 8192, &tm_do64, q_cl, b * 64, i * 128 + r64, bh);
                        }
                        mbar_arrive_expect_tx(ld_full + st, 1024);
                    } else {
                        mbar_arrive_expect_tx(q_full + st, 2 * Cfg::kTileBytes + 1024);
                        for (int b = 0; b < Cfg::kBoxes; ++b) {
                            tma_load_3d(q_st + b * 16384, &tm_q, q_full + st, b * 64, i * 128, bh);
                            tma_load_3d(do_st + b * 16384, &tm_do, q_full + st, b * 64, i * 128, bh);
                        }
                    }
                    const size_t ro = static_cast<size_t>(bh) * p.Npad + static_cast<size_t>(i) * 128;
                    bulk_load(sLD + st * 256, p.lse2 + ro, 512, ld_full + st);
                    bulk_load(sLD + st * 256 + 128, p.dsum + ro, 512, ld_full + st);
                }
                g0 += x.n_steps;
            }
        }
    } else if (warp == 1 && (!kPair || rank == 0)) {
        // ------------------------------------------------ MMA issuer (whole warp)
        constexpr uint32_t kM = kPair ? 256 : 128;
        constexpr uint32_t idesc_kk = umma_idesc_f16(kM, 128, kBF16, 0, 0);  // S^T, dP^T
        constexpr uint32_t idesc_kmn = umma_idesc_f16(kM, kD, kBF16, 0, 1);  // dV, dK
        constexpr uint64_t kTile16 = Cfg::kTileBytes >> 4;
        constexpr int kHalfB = kPair ? 16384 : 0;  // pair: the K-major 64-query half follows the MN-major d-half
        const uint64_t dK = umma_desc_sw128(smem_u32(sK), 16, 1024);
        const uint64_t dV = umma_desc_sw128(smem_u32(sV), 16, 1024);
        const uint64_t dQk = umma_desc_sw128(smem_u32(sQ + kHalfB), 16, 1024);    // Q as K-major B
        const uint64_t dDOk = umma_desc_sw128(smem_u32(sDO + kHalfB), 16, 1024);  // dO as K-major B
        const uint64_t dQm = umma_desc_sw128(smem_u32(sQ), 16384, 1024);    // Q as MN-major B
        const uint64_t dDOm = umma_desc_sw128(smem_u32(sDO), 16384, 1024);  // dO as MN-major B
        auto mma_commit_e = [&](uint64_t* bar) {  // a pair's commit arrives in both CTAs
            if constexpr (kPair)
                mma_commit_pair(bar);
            else
                vattn_sm100::mma_commit_e(bar);
        };
        auto mbar_wait_mma = [&](uint64_t* bar, uint32_t ph) {  // the peer's warps arrive here too
            if constexpr (kPair)
                mbar_wait_mma_cl(bar, ph);
            else
                vattn_sm100::mbar_wait_mma(bar, ph);
        };
        auto issue_kk = [&](uint32_t dcol, uint64_t ad, uint64_t bd) {
#pragma unroll
            for (int kk = 0; kk < kD / 16; ++kk) {
                if constexpr (kPair)
                    mma_ss_pair(tmem + dcol, desc_kmajor(ad, kk), desc_kmajor_half(bd, kk), idesc_kk, kk > 0);
                else
                    mma_ss_e(tmem + dcol, desc_kmajor(ad, kk), desc_kmajor(bd, kk), idesc_kk, kk > 0);
            }
        };
        // A operand (16-bit) held in TMEM by the math warpgroups: queries
        // [kQW h, kQW h + kQW) at columns base + kQW h + [0, kQW / 2).
        // Warpgroup h's K-steps (16 queries each) are issued as soon as h published
        // (`ready[h]`), or (kHalf) as soon as their half landed (`ready[kHv h + half]`).
        auto issue_ts = [&](uint32_t dcol, uint32_t abase_col, uint64_t bd, bool acc, uint64_t* ready, uint32_t ph,
                            auto half_gran) {
            constexpr int kHalfN = decltype(half_gran)::value ? kHv : 1;  // publication chunks per warpgroup
            constexpr int kPer = kQW / 16;                                // K-steps per warpgroup
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                if (kk % (kPer / kHalfN) == 0) {
                    mbar_wait_mma(ready + (kk / kPer) * kHalfN + (kk % kPer) / (kPer / kHalfN), ph);
                    tc_fence_after();
                }
                const uint32_t a_col = tmem + abase_col + (kk / kPer) * kQW + (kk % kPer) * 8;
                if constexpr (kPair)
                    mma_ts_pair(tmem + dcol, a_col, desc_mnmajor(bd, kk), idesc_kmn, (acc || kk > 0) ? 1u : 0u);
                else
                    mma_ts_e(tmem + dcol, a_col, desc_mnmajor(bd, kk), idesc_kmn, (acc || kk > 0) ? 1u : 0u);
            }
        };
        uint32_t g0 = 0;  // steps of this CTA's earlier items
        Item x;
        for (int it = 0; item_at(it, x); ++it) {
            const int n_steps = x.n_steps;
            const uint32_t R0 = kDB ? (g0 & 1u) * 128u : 0u;  // S region of the item's first step
            mbar_wait_mma(kv_full, it & 1);
            tc_fence_after();
            mbar_wait_mma(q_full + g0 % kSt, (g0 / kSt) & 1);
            tc_fence_after();
            issue_kk(Cfg::kTmemS + R0, dK, dQk + (g0 % kSt) * kTile16);
            mma_commit_e(s_full + (kDB ? (g0 & 1u) : 0u));
            issue_kk(Cfg::kTmemDP, dV, dDOk + (g0 % kSt) * kTile16);
            mma_commit_e(dp_full);
            VTRACE(3072);
            // the previous item's epilogue has read dV / dK out of tensor memory
            auto acc_wait = [&](int s) {
                if (it > 0 && s == 0) {
                    mbar_wait_mma(acc_free, (it - 1) & 1);
                    tc_fence_after();
                }
            };
            if constexpr (kDB) {
                if (n_steps > 1) {
                    const uint32_t g1 = g0 + 1;
                    mbar_wait_mma(q_full + g1 % kSt, (g1 / kSt) & 1);
                    tc_fence_after();
                    issue_kk(Cfg::kTmemS + (g1 & 1u) * 128u, dK, dQk + (g1 % kSt) * kTile16);  // S_1: the other region
                    mma_commit_e(s_full + (g1 & 1u));
                }
                for (int s = 0; s < n_steps; ++s) {
                    const uint32_t g = g0 + s;
                    const int st = g % kSt, st1 = (g + 1) % kSt, st2 = (g + 2) % kSt;
                    const uint32_t R = (g & 1u) * 128u;
                    stress_delay(3, s);
                    acc_wait(s);
                    issue_ts(Cfg::kTmemDV, Cfg::kTmemS + R, dDOm + st * kTile16, s > 0, p_full + kWG * kHv * (g & 1u),
                             (g >> 1) & 1, std::true_type{});  // dV += P^T dO
                    issue_ts(Cfg::kTmemDK, Cfg::kTmemDP, dQm + st * kTile16, s > 0, ds_full, g & 1, std::false_type{});  // dK += dS^T Q
                    mma_commit_e(q_empty + st);
                    if (s + 1 < n_steps) {
                        issue_kk(Cfg::kTmemDP, dV, dDOk + st1 * kTile16);  // after dK read dS^T
                        mma_commit_e(dp_full);
                    }
                    if (s + 2 < n_steps) {  // region R is free once dV_s read P^T_s (in order)
                        mbar_wait_mma(q_full + st2, ((g + 2) / kSt) & 1);
                        tc_fence_after();
                        issue_kk(Cfg::kTmemS + R, dK, dQk + st2 * kTile16);
                        mma_commit_e(s_full + (g & 1u));
                    }
                }
            } else
            for (int s = 0; s < n_steps; ++s) {
                const uint32_t g = g0 + s;
                const int st = g % kSt;
                const int st1 = (g + 1) % kSt;
                stress_delay(3, s);
                acc_wait(s);
                issue_ts(Cfg::kTmemDV, Cfg::kTmemS, dDOm + st * kTile16, s > 0, p_full + kWG * kHv * (g & 1u), (g >> 1) & 1,
                         std::true_type{});  // dV += P^T dO
                VTRACE(8 * s + 0);
                if (s + 1 < n_steps) {
                    mbar_wait(q_full + st1, ((g + 1) / kSt) & 1);
                    tc_fence_after();
                    VTRACE(8 * s + 1);
                    issue_kk(Cfg::kTmemS, dK, dQk + st1 * kTile16);  // in-order after dV read P^T
                    mma_commit_e(s_full);
                }
                issue_ts(Cfg::kTmemDK, Cfg::kTmemDP, dQm + st * kTile16, s > 0, ds_full, g & 1, std::false_type{});  // dK += dS^T Q
                VTRACE(8 * s + 2);
                mma_commit_e(q_empty + st);
                if (s + 1 < n_steps) {
                    issue_kk(Cfg::kTmemDP, dV, dDOk + st1 * kTile16);  // after dK read dS^T
                    mma_commit_e(dp_full);
                }
            }
            mma_commit_e(dkv_full);
            g0 += n_steps;
        }
    } else if (warp >= 4) {
        // ------------------------------------------------------ P / dS warps
        regs_inc<Cfg::kRegsHi>();
        const int h = (warp - 4) >> 2;           // query-column group: [kQW h, kQW h + kQW)
        const int r = ((warp & 3) << 5) + lane;  // key row == TMEM lane
        const uint32_t lb = static_cast<uint32_t>((warp & 3) * 32) << 16;
        const float sc = p.scale_log2;
        constexpr int kCh = kQW / 32;            // 32-column chunks per warpgroup
        uint32_t g0 = 0;  // steps of this CTA's earlier items
        Item x_;
        for (int it = 0; item_at(it, x_); ++it) {
        const int bh = x_.bh, kb = x_.kb, i0 = x_.i0, n_steps = x_.n_steps;
        const int key = kb * 128 + r;
        const bool key_ok = key < N;
        uint64_t dbase = 0;
        if constexpr (kDrop) dbase = drop_bh_base(p.drop_seed, (bh + p.bh_off) / p.H, (bh + p.bh_off) % p.H);
        auto load_kmw = [&](int qi, uint32_t (&kw)[kCh]) {
            const uint32_t* mk = p.drop_mask_k + (static_cast<size_t>(bh) * p.Npad + key) * (p.Npad / 32) + qi * 4 + kCh * h;
            if constexpr (kCh == 2) {
                const uint2 w = __ldg(reinterpret_cast<const uint2*>(mk));
                kw[0] = w.x;
                kw[kCh - 1] = w.y;
            } else {
                kw[0] = __ldg(mk);
            }
        };
        for (int s = 0; s < n_steps; ++s) {
            const uint32_t g = g0 + s;  // ring position (all items of this CTA)
            const int st = g % kSt;
            const int i = i0 + s;
            const float* lse2 = sLD + st * 256 + kQW * h;
            const float* dsum = sLD + st * 256 + 128 + kQW * h;
            const uint32_t sR = Cfg::kTmemS + (kDB ? (g & 1u) * 128u : 0u);  // S / P^T region of this tile
            // this key row's query bits (key-major copy, mha_dropmask_kernel).  (Loading them
            // one step ahead measured 11 % slower here -- registers -- unlike the forward.)
            uint32_t kmw[kCh];
#pragma unroll
            for (int c = 0; c < kCh; ++c) kmw[c] = ~0u;
            if (kDrop && p.drop_mask_k) load_kmw(i, kmw);
            mbar_wait(ld_full + st, (g / kSt) & 1);  // lse2 / D of this tile landed
            mbar_wait(s_full + (kDB ? (g & 1u) : 0u), kDB ? ((g >> 1) & 1) : (g & 1));
            tc_fence_after();
            stress_delay(1, s);
            if ((warp == 4 || warp == 8) && lane == 0) VTRACE(1024 + 8 * s + 0 + (warp == 8 ? 4 : 0));
            float pr[kQW];
#pragma unroll
            for (int c = 0; c < kCh; ++c) tmem_ld32f(tmem + lb + sR + kQW * h + 32 * c, pr + 32 * c);
            tmem_wait_ld();
            const int qbase = i * 128 + kQW * h;
            uint64_t keepm = ~0ull;  // dropout keep bits of this thread's kQW (query, key) positions
            if (kDrop && p.drop_mask_k) {
                keepm = static_cast<uint64_t>(kmw[0]) | (static_cast<uint64_t>(kmw[kCh - 1]) << (kCh == 2 ? 32 : 0));
            } else if constexpr (kDrop) {
                // row prefixes of the reference hash for this warpgroup's queries
                named_bar_sync(1 + h, 128);  // previous step's readers are done
                if ((warp & 3) * 32 + lane < kQW)
                    sDrop[kQW * h + (warp & 3) * 32 + lane] = drop_row(dbase, qbase + (warp & 3) * 32 + lane);
                named_bar_sync(1 + h, 128);
                keepm = 0;
#pragma unroll 1
                for (int x = 0; x < kQW; ++x)  // (fallback without a mask: kept out of the i-cache)
                    keepm |= static_cast<uint64_t>(drop_keep(sDrop[kQW * h + x], key, p.drop_thresh)) << x;
            }
            // P = exp2(S c - lse2) of one 32-query chunk.  The warpgroups exponentiate at the
            // same time on the same MUFU, so VATTN_POLY_DKDV*_WG1 of every 4 element pairs of
            // the odd warpgroups go to the FMA-pipe polynomial instead (asymmetric on
            // purpose, sm100_ptx.cuh).
            auto p_chunk = [&](auto npoly, auto chunk) {
                constexpr int kNP = decltype(npoly)::value;
                constexpr int x0 = 32 * decltype(chunk)::value;
#pragma unroll
                for (int x = x0; x < x0 + 32; x += 4) {
                    const float4 l4 = *reinterpret_cast<const float4*>(lse2 + x);
                    const float2 sc2 = make_float2(sc, sc);
                    float2 a = ffma2(make_float2(pr[x], pr[x + 1]), sc2, make_float2(-l4.x, -l4.y));
                    float2 b = ffma2(make_float2(pr[x + 2], pr[x + 3]), sc2, make_float2(-l4.z, -l4.w));
                    const int pa = (x / 2) & 3, pb = (x / 2 + 1) & 3;  // pair slot within 4
                    a = pa < kNP ? ex2_poly2(a) : make_float2(ex2(a.x), ex2(a.y));
                    b = pb < kNP ? ex2_poly2(b) : make_float2(ex2(b.x), ex2(b.y));
                    pr[x + 0] = a.x;
                    pr[x + 1] = a.y;
                    pr[x + 2] = b.x;
                    pr[x + 3] = b.y;
                }
                // masks only on the (warp-uniform) diagonal tile / the last key tile:
                // P = 0 for columns x < lim (key > query on the diagonal, all for keys >= N;
                // a pair's upper CTA also sees the tile below its diagonal: all masked)
                if ((p.causal && i <= kb) || kb * 128 + 128 > N) {
                    const int lim = !key_ok ? kQW : ((p.causal && i <= kb) ? key - qbase : 0);
#pragma unroll
                    for (int x = x0; x < x0 + 32; ++x)
                        if (x < lim) pr[x] = 0.0f;
                }
            };
            auto pack_chunk = [&](uint32_t (&pk)[16], int x0) {
                if constexpr (kDrop) {  // dV operand f16(P * drop) (attention_backward.cpp:163-167)
                    const float2 ik2 = make_float2(p.inv_keep, p.inv_keep);
                    uint32_t ks[8];  // this chunk's keep word, shifted: PRMT lane masks (keep_mask16)
                    const uint32_t kw = static_cast<uint32_t>(keepm >> x0);
#pragma unroll
                    for (int sh = 0; sh < 8; ++sh) ks[sh] = kw << sh;
#pragma unroll
                    for (int x = 0; x < 16; ++x) {
                        const int e = x0 + 2 * x;
                        const float2 pd = fmul2(make_float2(pr[e], pr[e + 1]), ik2);  // packed FMUL2
                        pk[x] = pack2<kBF16>(pd.x, pd.y) & keep_mask16(ks, x);      // dropped lanes +0
                    }
                } else {
#pragma unroll
                    for (int x = 0; x < 16; ++x) pk[x] = pack2<kBF16>(pr[x0 + 2 * x], pr[x0 + 2 * x + 1]);
                }
            };
            auto publish = [&](int half) {  // this chunk's tcgen05.st has been waited on
                tc_fence_before();
                __syncwarp();
                if (lane == 0) arrive_mma(p_full + kWG * kHv * (g & 1u) + kHv * h + half);
            };
            // P^T chunk by chunk: chunk 0 is stored (tcgen05.st) and published while chunk 1
            // is exponentiated.
            auto p_pass = [&](auto npoly) {
                uint32_t pa[16];
                p_chunk(npoly, std::integral_constant<int, 0>{});
                pack_chunk(pa, 0);
                tmem_st16(tmem + lb + sR + kQW * h, pa);  // own columns only
                if constexpr (kCh == 2) {
                    uint32_t pb[16];
                    p_chunk(npoly, std::integral_constant<int, 1>{});
                    pack_chunk(pb, 32);
                    tmem_wait_st();
                    publish(0);
                    tmem_st16(tmem + lb + sR + kQW * h + 16, pb);
                    tmem_wait_st();
                    publish(1);
                } else {
                    tmem_wait_st();
                    publish(0);
                }
            };
            constexpr int kPoly0 = kD == 64 ? VATTN_POLY_DKDV64_WG0 : VATTN_POLY_DKDV_WG0;
            constexpr int kPoly1 = kD == 64 ? VATTN_POLY_DKDV64_WG1 : VATTN_POLY_DKDV_WG1;
            if constexpr (kPoly0 == kPoly1)  // one copy of the P pass
                p_pass(std::integral_constant<int, kPoly0>{});
            else if ((h & 1) == 0)  // warp-uniform
                p_pass(std::integral_constant<int, kPoly0>{});
            else
                p_pass(std::integral_constant<int, kPoly1>{});
            if ((warp == 4 || warp == 8) && lane == 0) VTRACE(1024 + 8 * s + 1 + (warp == 8 ? 4 : 0));
            stress_delay(2, s);

            mbar_wait(dp_full, g & 1);
            tc_fence_after();
            if ((warp == 4 || warp == 8) && lane == 0) VTRACE(1024 + 8 * s + 2 + (warp == 8 ? 4 : 0));
            uint32_t dsp[kQW / 2];
#pragma unroll
            for (int c = 0; c < kCh; ++c) {
                float dpv[32];
                tmem_ld32f(tmem + lb + Cfg::kTmemDP + kQW * h + 32 * c, dpv);
                tmem_wait_ld();
#pragma unroll
                for (int x = 0; x < 32; x += 4) {
                    const float4 d4 = *reinterpret_cast<const float4*>(dsum + 32 * c + x);
                    float2 t0, t1;  // dP - D, packed FADD2 / FMUL2: half the issue slots
                    if constexpr (kDrop) {
                        // dS = P o (drop o dP - D) (attention_backward.cpp:176-182): one FFMA2
                        // dP * 1/(1-p) - D per pair, then -D where the position was dropped
                        const float2 ik2 = make_float2(p.inv_keep, p.inv_keep);
                        const float2 nd0 = make_float2(-d4.x, -d4.y), nd1 = make_float2(-d4.z, -d4.w);
                        t0 = ffma2(make_float2(dpv[x], dpv[x + 1]), ik2, nd0);
                        t1 = ffma2(make_float2(dpv[x + 2], dpv[x + 3]), ik2, nd1);
                        const int b = 32 * c + x;
                        t0.x = (keepm >> b) & 1 ? t0.x : nd0.x;
                        t0.y = (keepm >> (b + 1)) & 1 ? t0.y : nd0.y;
                        t1.x = (keepm >> (b + 2)) & 1 ? t1.x : nd1.x;
                        t1.y = (keepm >> (b + 3)) & 1 ? t1.y : nd1.y;
                    } else {
                        t0 = fadd2(make_float2(dpv[x], dpv[x + 1]), make_float2(-d4.x, -d4.y));
                        t1 = fadd2(make_float2(dpv[x + 2], dpv[x + 3]), make_float2(-d4.z, -d4.w));
                    }
                    const float2 s0 = fmul2(make_float2(pr[32 * c + x], pr[32 * c + x + 1]), t0);
                    const float2 s1 = fmul2(make_float2(pr[32 * c + x + 2], pr[32 * c + x + 3]), t1);
                    dsp[16 * c + x / 2] = pack2<kBF16>(s0.x, s0.y);
                    dsp[16 * c + x / 2 + 1] = pack2<kBF16>(s1.x, s1.y);
                }
            }
            if constexpr (kCh == 2)
                tmem_st32(tmem + lb + Cfg::kTmemDP + kQW * h, dsp);  // dS^T over our dP^T columns
            else
                tmem_st16(tmem + lb + Cfg::kTmemDP + kQW * h, dsp);
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                arrive_mma(ds_full + h);
                mbar_arrive(q_empty + st);  // done with lse2 / D of this stage
            }
            // dS^T materialisation after publishing: dK_i starts while the tile is staged.
            // One 64-query x 128-key box per 64 queries (one or two warpgroups write it);
            // the box's first warpgroup's first thread issues its TMA store (replaces
            // 16-byte global stores that stalled the math warps, profiles/r2_experiments.md)
            // (a pair's tiles above the diagonal or past the last key tile hold no dS)
            if (p.ds_out && !(kPair && (kb >= p.n_q || (p.causal && kb > i)))) {
                constexpr int kBoxWG = 64 / kQW;               // warpgroups per box
                const int bx = h / kBoxWG;                      // box (64-query group)
                const bool ds_store_thread = (h % kBoxWG) == 0 && (warp & 3) == 0 && lane == 0;
                const uint32_t bar_id = kBoxWG == 1 ? 1 + h : 5 + bx, bar_n = 128 * kBoxWG;
                uint8_t* box = smem + Cfg::kSmemDsStage + bx * 16384;
                if constexpr (kDsWarpStore<kD> && !kPair) {
                    // this warp's 32 rows = a 4 KiB, 1 KiB-aligned slice of the box (the
                    // 128-byte swizzle repeats every 8 rows): stage, fence, store it alone
                    if (lane == 0) bulk_wait_read0();  // this warp's previous slice left
                    __syncwarp();
#pragma unroll
                    for (int m = 0; m < kQW / 8; ++m)
                        st_swz128(box, r, m, make_uint4(dsp[4 * m], dsp[4 * m + 1], dsp[4 * m + 2], dsp[4 * m + 3]));
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        tma_store_3d(&tm_q64, box + (warp & 3) * 4096, 64 * bx, 32 * (warp & 3),
                                     static_cast<int>(static_cast<long long>(bh) * p.ds_tiles_per_bh + ds_tile_index(p, i, kb)));
                        bulk_commit();
                    }
                } else {
                if (ds_store_thread) bulk_wait_read0();  // the previous box left the buffer
                named_bar_sync(bar_id, bar_n);
                const int m0 = (h % kBoxWG) * (kQW / 8);    // first 16-byte chunk of this warpgroup's row part
#pragma unroll
                for (int m = 0; m < kQW / 8; ++m)
                    st_swz128(box, r, m0 + m, make_uint4(dsp[4 * m], dsp[4 * m + 1], dsp[4 * m + 2], dsp[4 * m + 3]));
                fence_proxy_async_smem();
                named_bar_sync(bar_id, bar_n);
                if (ds_store_thread) {
                    tma_store_3d(&tm_ds, box, 64 * bx, 0,
                                 static_cast<int>(static_cast<long long>(bh) * p.ds_tiles_per_bh + ds_tile_index(p, i, kb)));
                    bulk_commit();
                }
                }
            }

            if ((warp == 4 || warp == 8) && lane == 0) VTRACE(1024 + 8 * s + 3 + (warp == 8 ? 4 : 0));
        }
        if (p.ds_out && ((kDsWarpStore<kD> && !kPair) || (warp & 3) == 0) && lane == 0) {
            if (p.dq_sync) {  // this CTA's dS^T stores are in memory: count them for the dQ workers
                bulk_wait0();
                fence_proxy_async_global();
                __threadfence();
                atomicAdd(p.dq_sync + 2 + bh, 1);
            } else {
                bulk_wait_read0();  // no store reads smem past exit
            }
        }
        // ---------------------------------------------------------- epilogue
        mbar_wait(dkv_full, it & 1);
        tc_fence_after();
        T16* dk = reinterpret_cast<T16*>(dk_out) + (static_cast<size_t>(bh) * N + key) * kD;
        T16* dv = reinterpret_cast<T16*>(dv_out) + (static_cast<size_t>(bh) * N + key) * kD;
        constexpr int kCols = kD / kWG;  // dK / dV columns per warpgroup (16, 32 or 64)
        constexpr int kEc = kCols < 32 ? kCols : 32;
#pragma unroll
        for (int c = 0; c < kCols / kEc; ++c) {
            const int col = h * kCols + kEc * c;
            float a[32], b[32];
            if constexpr (kEc == 32) {
                tmem_ld32f(tmem + lb + Cfg::kTmemDV + col, a);
                tmem_ld32f(tmem + lb + Cfg::kTmemDK + col, b);
            } else {
                uint32_t ua[16], ub[16];
                tmem_ld16(tmem + lb + Cfg::kTmemDV + col, ua);
                tmem_ld16(tmem + lb + Cfg::kTmemDK + col, ub);
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                    a[e] = __uint_as_float(ua[e]);
                    b[e] = __uint_as_float(ub[e]);
                }
            }
            tmem_wait_ld();
            if (key_ok) {
#pragma unroll
                for (int x = 0; x < kEc / 8; ++x) {
                    uint4 va, vb;
                    va.x = pack2<kBF16>(a[8 * x + 0], a[8 * x + 1]);
                    va.y = pack2<kBF16>(a[8 * x + 2], a[8 * x + 3]);
                    va.z = pack2<kBF16>(a[8 * x + 4], a[8 * x + 5]);
                    va.w = pack2<kBF16>(a[8 * x + 6], a[8 * x + 7]);
                    vb.x = pack2<kBF16>(b[8 * x + 0] * p.scale, b[8 * x + 1] * p.scale);
                    vb.y = pack2<kBF16>(b[8 * x + 2] * p.scale, b[8 * x + 3] * p.scale);
                    vb.z = pack2<kBF16>(b[8 * x + 4] * p.scale, b[8 * x + 5] * p.scale);
                    vb.w = pack2<kBF16>(b[8 * x + 6] * p.scale, b[8 * x + 7] * p.scale);
                    *reinterpret_cast<uint4*>(dv + col + 8 * x) = va;
                    *reinterpret_cast<uint4*>(dk + col + 8 * x) = vb;
                }
            }
        }
        // dV / dK are in registers: the next item's first dV / dK MMAs may overwrite them
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(acc_free);
        g0 += n_steps;
        }  // items
    }
    if (!kPdlEarly) griddep_launch_dependents();
    tc_fence_before();
    if constexpr (!kPair) {
        if (p.dq_sync) {  // after this CTA's dS^T counts (the barrier below orders them)
            __syncthreads();
            if (threadIdx.x == 0) {
                __threadfence();
                atomicAdd(p.dq_sync + 1, 1);
            }
        }
    }
    if constexpr (kPair) {
        cluster_sync_all();  // the leader's MMAs read the peer's smem / TMEM until dkv_full
        if (warp == 2) {
            tc_fence_after();
            tmem_dealloc_pair<512>(tmem);
        }
    } else {
        __syncthreads();
        if (warp == 2) {
            tc_fence_after();
            tmem_dealloc<512>(tmem);
        }
    }
    VCTA(1, 1);
}

// ===================================================================== dQ ==
//
// One CTA = one (b*h, 128-query tile i).  Q_i, dO_i resident; K_j, V_j stream
// through a ring (causal: j <= i).  Per key tile j:
//   S = Q_i K_j^T (SS -> region j&1)   dP = dO_i V_j^T (SS -> region DP)
//   P = exp2(S c - lse2_row),  dS = P o (dP - D_row)   (thread = query row)
//   dS (16-bit) -> region j&1 over the consumed S columns
//   dQ += dS K_j (TS, accumulated in TMEM across j in ascending order)
// MMA order: S_0, dP_0, S_1, then per j: dQ_j, dP_(j+1), S_(j+2).
// Tensor memory: S/dS regions [0,128) and [128,256), dP [256,384), dQ [384,384+D).
template <int kD>
struct DqCfg {
    static constexpr int kTileBytes = kD * 128 * 2;
    static constexpr int kBoxes = kD / 64;
    // separate rings: K_j is held until dQ_j, V_j only until dP_j
    static constexpr int kKSlots = kD == 128 ? 3 : 4;
    static constexpr int kVSlots = kD == 128 ? 2 : 4;
    static constexpr int kSmemQ = 0;
    static constexpr int kSmemDO = kTileBytes;
    static constexpr int kSmemK = 2 * kTileBytes;
    static constexpr int kSmemV = kSmemK + kKSlots * kTileBytes;
    static constexpr int kSmemBar = kSmemV + kVSlots * kTileBytes;
    static constexpr int kNumBars = 1 + 2 * kKSlots + 2 * kVSlots + 2 + 1 + 2 + 1 + 1;
    // d = 64: dP_(j+1) is issued as soon as the math warps hold dP_j in registers
    // (measured -4..5 % on the dQ kernel at d = 64; at d = 128 it delays S_(j+2) and loses)
    static constexpr bool kEarlyDP = kD == 64;
    static constexpr int kSmemBytes = kSmemBar + kNumBars * 8 + 16;
    static constexpr uint32_t kTmemDP = 256, kTmemDQ = 384;
};

template <int kD, bool kBF16, bool kDrop>
__global__ void __launch_bounds__(384, 1)
    mha_bwd_dq_kernel(const __grid_constant__ CUtensorMap tm_q,
                      const __grid_constant__ CUtensorMap tm_k,
                      const __grid_constant__ CUtensorMap tm_v,
                      const __grid_constant__ CUtensorMap tm_do,
                      const __grid_constant__ CUtensorMap tm_dq, const BwdParams p) {
    VCTA(2, 0);
    griddep_start();
    using Cfg = DqCfg<kD>;
    constexpr int kVtraceKid = 2;
    (void)kVtraceKid;
    constexpr int SK = Cfg::kKSlots, SV = Cfg::kVSlots;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* sQ = smem + Cfg::kSmemQ;
    uint8_t* sDO = smem + Cfg::kSmemDO;
    uint8_t* sK = smem + Cfg::kSmemK;
    uint8_t* sV = smem + Cfg::kSmemV;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::kSmemBar);
    uint64_t* qd_full = bars;               // Q, dO
    uint64_t* k_full = bars + 1;            // [SK]
    uint64_t* k_empty = k_full + SK;        // [SK]
    uint64_t* v_full = k_empty + SK;        // [SV]
    uint64_t* v_empty = v_full + SV;        // [SV]
    uint64_t* s_full = v_empty + SV;        // [2] per S region
    uint64_t* dp_full = s_full + 2;
    // ds_full[j & 1] (8 arrivals each).  With the early dP (d = 64) a fast warp can
    // finish dS_(j+1) before a slow warp arrived for dS_j (dP_(j+1) only needs every
    // warp to have LOADED dP_j); on one barrier its arrival would complete phase j
    // early (the MMA would read the slow warp's dS_j half written).  Two barriers
    // separate the phases; no warp can reach dS_(j+2) before all finished dS_j.
    uint64_t* ds_full = dp_full + 1;        // [2]
    uint64_t* dq_done = ds_full + 2;
    uint64_t* dp_empty = dq_done + 1;       // kEarlyDP: all 8 math warps loaded dP_j
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + Cfg::kNumBars);

    const int warp = warp_id();
    const int lane = lane_id();
    const int nqb = p.n_q;
    const int bh = grid_bh(nqb);
    const int i = p.causal ? (nqb - 1 - grid_tile(nqb)) : grid_tile(nqb);
    const int N = p.N;
    const int nk = p.causal ? i + 1 : p.n_q;

    if (threadIdx.x == 0) {
        if ((smem_u32(smem) & 1023u) != 0) __trap();
        mbar_init(qd_full, 1);
        for (int s = 0; s < SK; ++s) {
            mbar_init(k_full + s, 1);
            mbar_init(k_empty + s, 1);
        }
        for (int s = 0; s < SV; ++s) {
            mbar_init(v_full + s, 1);
            mbar_init(v_empty + s, 1);
        }
        mbar_init(s_full + 0, 1);
        mbar_init(s_full + 1, 1);
        mbar_init(dp_full, 1);
        mbar_init(ds_full + 0, 8);
        mbar_init(ds_full + 1, 8);
        mbar_init(dq_done, 1);
        mbar_init(dp_empty, 8);
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    griddep_wait();  // inputs written by the previous kernel in the stream are visible
    if (warp < 4) regs_dec<88>();

    if (warp == 0) {
        // ------------------------------------------------------ TMA producer
        if (lane == 0) {
            tma_prefetch_desc(&tm_q);
            tma_prefetch_desc(&tm_k);
            tma_prefetch_desc(&tm_v);
            tma_prefetch_desc(&tm_do);
            tma_prefetch_desc(&tm_dq);
            mbar_arrive_expect_tx(qd_full, 2 * Cfg::kTileBytes);
            for (int b = 0; b < Cfg::kBoxes; ++b) {
                tma_load_3d(sQ + b * 16384, &tm_q, qd_full, b * 64, i * 128, bh);
                tma_load_3d(sDO + b * 16384, &tm_do, qd_full, b * 64, i * 128, bh);
            }
            // K runs ahead of V (S_(j+1) is issued before dP_(j+1))
            auto load_k = [&](int j) {
                const int sl = j % SK;
                mbar_wait<VATTN_SLEEP_PRODUCER, true>(k_empty + sl, ((j / SK) & 1) ^ 1);
                mbar_arrive_expect_tx(k_full + sl, Cfg::kTileBytes);
                for (int b = 0; b < Cfg::kBoxes; ++b)
                    tma_load_3d(sK + sl * Cfg::kTileBytes + b * 16384, &tm_k, k_full + sl, b * 64, j * 128, bh);
            };
            auto load_v = [&](int j) {
                const int sl = j % SV;
                mbar_wait<VATTN_SLEEP_PRODUCER, true>(v_empty + sl, ((j / SV) & 1) ^ 1);
                mbar_arrive_expect_tx(v_full + sl, Cfg::kTileBytes);
                for (int b = 0; b < Cfg::kBoxes; ++b)
                    tma_load_3d(sV + sl * Cfg::kTileBytes + b * 16384, &tm_v, v_full + sl, b * 64, j * 128, bh);
            };
            load_k(0);
            if (nk > 1) load_k(1);
            for (int j = 0; j < nk; ++j) {
                stress_delay(4, j);
                load_v(j);
                if (j + 2 < nk) load_k(j + 2);
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer (whole warp)
        constexpr uint32_t idesc_kk = umma_idesc_f16(128, 128, kBF16, 0, 0);  // S, dP
        constexpr uint32_t idesc_dq = umma_idesc_f16(128, kD, kBF16, 0, 1);   // dQ (B = K MN-major)
        constexpr uint64_t kTile16 = Cfg::kTileBytes >> 4;
        const uint64_t dQd = umma_desc_sw128(smem_u32(sQ), 16, 1024);
        const uint64_t dDOd = umma_desc_sw128(smem_u32(sDO), 16, 1024);
        const uint64_t dKk = umma_desc_sw128(smem_u32(sK), 16, 1024);     // K slots, K-major (S)
        const uint64_t dKm = umma_desc_sw128(smem_u32(sK), 16384, 1024);  // K slots, MN-major (dQ)
        const uint64_t dVk = umma_desc_sw128(smem_u32(sV), 16, 1024);
        auto kslot = [&](int j) {
            mbar_wait_mma(k_full + j % SK, (j / SK) & 1);
            tc_fence_after();
            return static_cast<uint64_t>(j % SK) * kTile16;
        };
        auto vslot = [&](int j) {
            mbar_wait_mma(v_full + j % SV, (j / SV) & 1);
            tc_fence_after();
            return static_cast<uint64_t>(j % SV) * kTile16;
        };
        auto issue_kk = [&](uint32_t dcol, uint64_t ad, uint64_t bd) {
#pragma unroll
            for (int kk = 0; kk < kD / 16; ++kk)
                mma_ss_e(tmem + dcol, desc_kmajor(ad, kk), desc_kmajor(bd, kk), idesc_kk, kk > 0);
        };
        mbar_wait_mma(qd_full, 0);
        tc_fence_after();
        issue_kk(0, dQd, dKk + kslot(0));  // S_0
        mma_commit_e(s_full + 0);
        issue_kk(Cfg::kTmemDP, dDOd, dVk + vslot(0));  // dP_0
        mma_commit_e(dp_full);
        mma_commit_e(v_empty + 0);
        if (nk > 1) {
            issue_kk(128, dQd, dKk + kslot(1));  // S_1
            mma_commit_e(s_full + 1);
        }
        VTRACE(3072);
        for (int j = 0; j < nk; ++j) {
            const uint32_t R = (j & 1) ? 128u : 0u;
            const uint64_t kd = dKm + static_cast<uint64_t>(j % SK) * kTile16;
            if constexpr (Cfg::kEarlyDP) {
                if (j + 1 < nk) {  // the dP region is free once every math warp loaded dP_j
                    mbar_wait_mma(dp_empty, j & 1);
                    tc_fence_after();
                    const uint64_t vo = vslot(j + 1);
                    issue_kk(Cfg::kTmemDP, dDOd, dVk + vo);
                    mma_commit_e(dp_full);
                    mma_commit_e(v_empty + (j + 1) % SV);
                }
            }
            stress_delay(3, j);
            mbar_wait_mma(ds_full + (j & 1), (j >> 1) & 1);
            tc_fence_after();
            VTRACE(8 * j + 0);
            // dQ += dS K_j : A = dS in TMEM (warpgroup h: keys [64h, 64h+64) at R + 64h + [0,32))
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
                mma_ts_e(tmem + Cfg::kTmemDQ, tmem + R + (kk >> 2) * 64 + (kk & 3) * 8, desc_mnmajor(kd, kk),
                         idesc_dq, (j > 0 || kk > 0) ? 1u : 0u);
            VTRACE(8 * j + 3);
            mma_commit_e(k_empty + j % SK);  // K_j consumed (S_j and dQ_j)
            VTRACE(8 * j + 4);
            // dP_(j+1) after dQ_j (measured: issuing it first delays S_(j+2) and the
            // next P pass more than it shortens the dS chain)
            if (!Cfg::kEarlyDP && j + 1 < nk) {
                const uint64_t vo = vslot(j + 1);
                VTRACE(8 * j + 1);
                issue_kk(Cfg::kTmemDP, dDOd, dVk + vo);
                VTRACE(8 * j + 5);
                mma_commit_e(dp_full);
                mma_commit_e(v_empty + (j + 1) % SV);
            }
            if (j + 2 < nk) {
                const uint64_t ko = kslot(j + 2);
                VTRACE(8 * j + 2);
                issue_kk(R, dQd, dKk + ko);  // S_(j+2): in-order after dQ_j read dS_j
                VTRACE(8 * j + 6);
                mma_commit_e(s_full + (j & 1));
            }
        }
        mma_commit_e(dq_done);
    } else if (warp >= 4) {
        regs_inc<208>();
        const int h = (warp - 4) >> 2;           // key-column half
        const int r = ((warp & 3) << 5) + lane;  // query row == TMEM lane
        const uint32_t lb = static_cast<uint32_t>((warp & 3) * 32) << 16;
        const int q = i * 128 + r;
        const float sc = p.scale_log2;
        const float lse2 = p.lse2[static_cast<size_t>(bh) * p.Npad + q];  // +inf past N
        const float dsum = p.dsum[static_cast<size_t>(bh) * p.Npad + q];
        DropRow drow{};
        if constexpr (kDrop) drow = drop_row(drop_bh_base(p.drop_seed, (bh + p.bh_off) / p.H, (bh + p.bh_off) % p.H), q);
        for (int j = 0; j < nk; ++j) {
            const uint32_t R = (j & 1) ? 128u : 0u;
            mbar_wait<VATTN_SLEEP_MATH, true>(s_full + (j & 1), (j >> 1) & 1);
            tc_fence_after();
            stress_delay(1, j);
            if (warp == 4 && lane == 0) VTRACE(1024 + 8 * j + 0);
            float pr[64];
            tmem_ld32f(tmem + lb + R + 64 * h, pr);
            tmem_ld32f(tmem + lb + R + 64 * h + 32, pr + 32);
            tmem_wait_ld();
            // masks: causal diagonal (key > query) and keys beyond N
            int lim = 63;  // last valid column of this half
            const int kbase = j * 128 + 64 * h;
            if (p.causal && j == i) lim = min(lim, q - kbase);
            lim = min(lim, N - 1 - kbase);
            // P = exp2(S c - lse2): packed scale-subtract; VATTN_POLY_DQ*_WG1 of every 4
            // element pairs of warpgroup 1 on the FMA-pipe polynomial (asymmetric, as in
            // the dK/dV kernel: the two warpgroups exponentiate at the same time)
            auto p_pass = [&](auto npoly) {
                constexpr int kNP = decltype(npoly)::value;
                const float2 sc2 = make_float2(sc, sc), nl2 = make_float2(-lse2, -lse2);
#pragma unroll
                for (int x = 0; x < 64; x += 2) {
                    float2 a = ffma2(make_float2(pr[x], pr[x + 1]), sc2, nl2);
                    a = ((x / 2) & 3) < kNP ? ex2_poly2(a) : make_float2(ex2(a.x), ex2(a.y));
                    pr[x] = a.x;
                    pr[x + 1] = a.y;
                }
            };
            constexpr int kPoly0 = kD == 64 ? VATTN_POLY_DQ64_WG0 : VATTN_POLY_DQ_WG0;
            constexpr int kPoly1 = kD == 64 ? VATTN_POLY_DQ64_WG1 : VATTN_POLY_DQ_WG1;
            if constexpr (kPoly0 == kPoly1)  // one copy of the P pass
                p_pass(std::integral_constant<int, kPoly0>{});
            else if (h == 0)  // warp-uniform
                p_pass(std::integral_constant<int, kPoly0>{});
            else
                p_pass(std::integral_constant<int, kPoly1>{});
            // masks only on the (warp-uniform) causal diagonal tile / the tile holding key N-1
            if ((p.causal && j == i) || kbase + 64 > N) {
#pragma unroll
                for (int x = 0; x < 64; ++x)
                    if (x > lim) pr[x] = 0.0f;
            }
            if (warp == 4 && lane == 0) VTRACE(1024 + 8 * j + 1);
            stress_delay(2, j);
            mbar_wait<VATTN_SLEEP_MATH, true>(dp_full, j & 1);
            tc_fence_after();
            if (warp == 4 && lane == 0) VTRACE(1024 + 8 * j + 2);
            uint32_t dsp[32];
            float dpa[Cfg::kEarlyDP ? 64 : 1];
            if constexpr (Cfg::kEarlyDP) {
                tmem_ld32f(tmem + lb + Cfg::kTmemDP + 64 * h, dpa);
                tmem_ld32f(tmem + lb + Cfg::kTmemDP + 64 * h + 32, dpa + 32);
                tmem_wait_ld();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(dp_empty);  // the MMA warp may overwrite dP now
            }
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                float dpb[32];
                float* dpv = dpb;
                if constexpr (Cfg::kEarlyDP) {
                    dpv = dpa + 32 * c;
                } else {
                    tmem_ld32f(tmem + lb + Cfg::kTmemDP + 64 * h + 32 * c, dpb);
                    tmem_wait_ld();
                }
                const float2 nd2 = make_float2(-dsum, -dsum);
                if constexpr (kDrop) {
                    // dS = P o (drop o dP - D), the dK/dV kernel's arithmetic exactly: one FFMA2
                    // dP * 1/(1-p) - D per pair, -D where the position was dropped
                    uint32_t kw;
                    if (p.drop_mask) {
                        kw = p.drop_mask[(static_cast<size_t>(bh) * p.Npad + q) * (p.Npad / 32) + (j * 128 + 64 * h + 32 * c) / 32];
                    } else {
                        kw = 0;
#pragma unroll 1
                        for (int x = 0; x < 32; ++x)
                            kw |= static_cast<uint32_t>(drop_keep(drow, j * 128 + 64 * h + 32 * c + x, p.drop_thresh)) << x;
                    }
                    const float2 ik2 = make_float2(p.inv_keep, p.inv_keep);
#pragma unroll
                    for (int x = 0; x < 16; ++x) {
                        float2 t = ffma2(make_float2(dpv[2 * x], dpv[2 * x + 1]), ik2, nd2);
                        t.x = (kw >> (2 * x)) & 1u ? t.x : nd2.x;
                        t.y = (kw >> (2 * x + 1)) & 1u ? t.y : nd2.y;
                        const float2 ds = fmul2(make_float2(pr[32 * c + 2 * x], pr[32 * c + 2 * x + 1]), t);
                        dsp[16 * c + x] = pack2<kBF16>(ds.x, ds.y);
                    }
                } else {
#pragma unroll
                    for (int x = 0; x < 16; ++x) {  // packed FADD2 / FMUL2: half the issue slots
                        const float2 ds = fmul2(make_float2(pr[32 * c + 2 * x], pr[32 * c + 2 * x + 1]),
                                                fadd2(make_float2(dpv[2 * x], dpv[2 * x + 1]), nd2));
                        dsp[16 * c + x] = pack2<kBF16>(ds.x, ds.y);
                    }
                }
            }
            tmem_st32(tmem + lb + R + 64 * h, dsp);  // dS over our (consumed) S columns
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(ds_full + (j & 1));
            if (warp == 4 && lane == 0) VTRACE(1024 + 8 * j + 3);
        }
        // ------------------------------------- epilogue: dQ * scale -> 16-bit
        mbar_wait<VATTN_SLEEP_MATH, true>(dq_done, 0);
        tc_fence_after();
        uint8_t* sOut = sQ;  // Q tile is dead once the last S landed
#pragma unroll
        for (int c = 0; c < kD / 64; ++c) {
            const int col = h * (kD / 2) + 32 * c;
            float a[32];
            tmem_ld32f(tmem + lb + Cfg::kTmemDQ + col, a);
            tmem_wait_ld();
#pragma unroll
            for (int x = 0; x < 4; ++x) {
                uint4 v;
                v.x = pack2<kBF16>(a[8 * x + 0] * p.scale, a[8 * x + 1] * p.scale);
                v.y = pack2<kBF16>(a[8 * x + 2] * p.scale, a[8 * x + 3] * p.scale);
                v.z = pack2<kBF16>(a[8 * x + 4] * p.scale, a[8 * x + 5] * p.scale);
                v.w = pack2<kBF16>(a[8 * x + 6] * p.scale, a[8 * x + 7] * p.scale);
                const int cc = col + 8 * x;
                st_swz128(sOut + (cc >> 6) * 16384, r, (cc & 63) >> 3, v);
            }
        }
        fence_proxy_async_smem();
        named_bar_sync(1, 256);
        if (warp == 4 && lane == 0) {
            for (int b = 0; b < Cfg::kBoxes; ++b) tma_store_3d(&tm_dq, sOut + b * 16384, b * 64, i * 128, bh);
            bulk_commit();
            bulk_wait_read0();
        }
    }
    if (!kPdlEarly) griddep_launch_dependents();
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
    VCTA(2, 1);
}

// ============================================================ dQ = dS K ==
//
// With dS materialised by the dK/dV kernel, dQ_i = sum_j dS_ij K_j is a plain
// streaming GEMM: one CTA per (b*h, 128-query tile i), dS_ij (from its dS^T tile,
// an MN-major A operand) and K_j (MN-major B) through a TMA ring, accumulated in
// tensor memory in ascending j (the same fixed order and single rounding as the
// reference's DqAccumulator, attention_backward.cpp:205,215) -- deterministic, and
// none of the S / dP recompute of mha_bwd_dq_kernel.  HBM-bound on the dS stream.
template <int kD, bool kBF16>
__global__ void __launch_bounds__(256, 1)
    mha_bwd_dq_gemm_kernel(const __grid_constant__ CUtensorMap tm_ds, const __grid_constant__ CUtensorMap tm_k,
                           const __grid_constant__ CUtensorMap tm_dq, const BwdParams p) {
    VCTA(3, 0);
    griddep_start();
    using Cfg = DqGemmCfg<kD>;
    constexpr int S = Cfg::kStages;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::kSmemBar);
    uint64_t* full = bars;
    uint64_t* empty = bars + S;
    uint64_t* dq_done = bars + 2 * S;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + Cfg::kNumBars);
    const int warp = warp_id();
    const int lane = lane_id();
    const int nqb = p.n_q;
    int bh, tile;
    grid_item_tail(nqb, p.tail_units, bh, tile);  // same dispatch as the dK/dV grid
    const int i = p.causal ? (nqb - 1 - tile) : tile;
    const int nk = p.causal ? i + 1 : p.n_q;
    if (threadIdx.x == 0) {
        if ((smem_u32(smem) & 1023u) != 0) __trap();
        for (int s = 0; s < S; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
        }
        mbar_init(dq_done, 1);
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc<kD>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    griddep_wait();  // inputs written by the previous kernel in the stream are visible
    if (warp == 0) {
        if (lane == 0) {
            tma_prefetch_desc(&tm_ds);
            tma_prefetch_desc(&tm_k);
            tma_prefetch_desc(&tm_dq);
            const long long tile0 = static_cast<long long>(bh) * p.ds_tiles_per_bh + ds_tile_index(p, i, 0);
            for (int j = 0; j < nk; ++j) {
                const int st = j % S;
                stress_delay(4, j);
                mbar_wait<VATTN_SLEEP_PRODUCER>(empty + st, ((j / S) & 1) ^ 1);
                mbar_arrive_expect_tx(full + st, Cfg::kStageBytes);
                uint8_t* ds = smem + st * Cfg::kStageBytes;
                uint8_t* kt = ds + Cfg::kDsBytes;
                const int tile = static_cast<int>(tile0 + j);
                tma_load_3d(ds, &tm_ds, full + st, 0, 0, tile);
                tma_load_3d(ds + 16384, &tm_ds, full + st, 64, 0, tile);
                for (int b = 0; b < kD / 64; ++b) tma_load_3d(kt + b * 16384, &tm_k, full + st, b * 64, j * 128, bh);
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t idesc = umma_idesc_f16(128, kD, kBF16, 1, 1);  // A = dS (MN-major), B = K (MN-major)
        const uint64_t dA0 = umma_desc_sw128(smem_u32(smem), 16384, 1024);
        const uint64_t dB0 = umma_desc_sw128(smem_u32(smem + Cfg::kDsBytes), 16384, 1024);
        constexpr uint64_t kStage16 = Cfg::kStageBytes >> 4;
        for (int j = 0; j < nk; ++j) {
            const int st = j % S;
            stress_delay(3, j);
            mbar_wait_mma(full + st, (j / S) & 1);
            tc_fence_after();
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
                mma_ss_e(tmem, desc_mnmajor(dA0 + st * kStage16, kk), desc_mnmajor(dB0 + st * kStage16, kk), idesc,
                         (j > 0 || kk > 0) ? 1u : 0u);
            mma_commit_e(empty + st);
        }
        mma_commit_e(dq_done);
    } else if (warp >= 4) {
        // epilogue: dQ * scale -> 16-bit -> swizzled smem (stage 0's dS buffer) -> TMA store
        const int r = ((warp & 3) << 5) + lane;
        const uint32_t lb = static_cast<uint32_t>((warp & 3) * 32) << 16;
        mbar_wait<VATTN_SLEEP_MATH>(dq_done, 0);
        tc_fence_after();
        uint8_t* sOut = smem;
#pragma unroll
        for (int c = 0; c < kD / 32; ++c) {
            float a[32];
            tmem_ld32f(tmem + lb + 32 * c, a);
            tmem_wait_ld();
#pragma unroll
            for (int x = 0; x < 4; ++x) {
                uint4 v;
                v.x = pack2<kBF16>(a[8 * x + 0] * p.scale, a[8 * x + 1] * p.scale);
                v.y = pack2<kBF16>(a[8 * x + 2] * p.scale, a[8 * x + 3] * p.scale);
                v.z = pack2<kBF16>(a[8 * x + 4] * p.scale, a[8 * x + 5] * p.scale);
                v.w = pack2<kBF16>(a[8 * x + 6] * p.scale, a[8 * x + 7] * p.scale);
                const int cc = 32 * c + 8 * x;
                st_swz128(sOut + (cc >> 6) * 16384, r, (cc & 63) >> 3, v);
            }
        }
        fence_proxy_async_smem();
        named_bar_sync(1, 128);
        if (warp == 4 && lane == 0) {
            for (int b = 0; b < kD / 64; ++b) tma_store_3d(&tm_dq, sOut + b * 16384, b * 64, i * 128, bh);
            bulk_commit();
            bulk_wait_read0();
        }
    }
    if (!kPdlEarly) griddep_launch_dependents();
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<kD>(tmem);
    }
    VCTA(3, 1);
}

}  // namespace vattn_sm100
