// mha_bwd_sm100.cuh -- fused multi-head-attention backward for sm_100a.
//
// Replaces the per-(batch, head, key-tile) unit loop of vattn::backward_fused
// (reference: proj/src/attention_backward.cpp:110-211) and its dQ master-buffer
// accumulation (DqAccumulator / dq_atomic_add, :22-42, applied at :205,
// finalized once at :215).  Per key tile (128 keys) and query tile i:
//   S^T  = K Q_i^T                      (SS MMA -> TMEM)
//   P^T  = exp2(S^T * scale*log2e - lse2_i)   (registers, -> TMEM as 16-bit)
//   dP^T = V dO_i^T                     (SS MMA -> TMEM)
//   dV  += P^T dO_i                     (TS MMA: P^T from TMEM)
//   dS^T = P^T o (dP^T - D_i)           (registers, -> SMEM as 16-bit, swizzled)
//   dK  += dS^T Q_i                     (SS MMA, dS^T K-major)
//   dQ_i = dS K                         (SS MMA, dS MN-major: the same SMEM tile)
// dK is scaled by softmax_scale in the epilogue; dQ in the final split reduction.
//
// Deterministic dQ ("split reduction", BASELINE north_star): key tiles are split
// into groups of kGroup consecutive tiles.  Each group owns an fp32 partial
// buffer; inside a group the contributions to a query tile are applied in a
// FIXED order (semaphore per (group, bh, q-tile); the rank-0 contributor
// stores, the others reduce-add).  Query tiles are visited in an order that
// makes every CTA of a group reach its turn in lock-step (causal: ascending
// from the diagonal, contributions in descending key-tile order; non-causal:
// rotated start).  mha_dq_convert then sums the group partials in ascending
// group order and rounds once -- bit-reproducible run to run.  Work items are
// taken from a ticket counter so a CTA only ever waits on CTAs that were
// handed work earlier (deadlock-free whenever >= kGroup CTAs can be resident).
//
// Warp roles (512 threads):
//   warp 0 TMA producer      warp 1 MMA issuer      warp 2 TMEM allocator
//   warps 4-11  two "dS" warpgroups: thread = key row (TMEM lane); WG h owns
//               query columns [64h, 64h+64) of every tile
//   warps 12-15 dQ writer: thread = query row; drains dQ from TMEM and applies
//               it to the group partial buffer in the fixed order
// Tensor memory: S^T [0,128) dP^T [128,256) dV [256,256+D) dK [256+D,256+2D)
//   dQ: D == 64 -> [384,448); D == 128 -> aliases dP^T (free once dS is built).
#pragma once

#include "sm100_ptx.cuh"

namespace vattn_sm100 {

constexpr int kBwdGroup = 64;  // key tiles per deterministic dQ group

struct BwdParams {
    const float* lse2;   // [BH, Npad]  lse * log2(e), +inf padding
    const float* dsum;   // [BH, Npad]  D = rowsum(dO o O), 0 padding
    float* dq_acc;       // [n_groups, BH, N, D] fp32 partials
    int* sems;           // [n_groups, BH, n_q] contribution counters (zeroed)
    int* ticket;         // work-item counter (zeroed)
    void* dk;            // [BH, N, D] 16-bit
    void* dv;            // [BH, N, D] 16-bit
    int N, Npad, BH, n_q;
    int causal;
    float scale;         // softmax scale (applied to dK here, dQ in convert)
    float scale_log2;    // scale * log2(e)
};

template <int kD>
struct BwdCfg {
    static constexpr int kTileBytes = kD * 128 * 2;
    static constexpr int kBoxes = kD / 64;
    static constexpr int kSmemK = 0;
    static constexpr int kSmemV = kTileBytes;
    static constexpr int kSmemQ = 2 * kTileBytes;             // 2 stages
    static constexpr int kSmemDO = 4 * kTileBytes;            // 2 stages
    static constexpr int kSmemDS = 6 * kTileBytes;            // 128 x 128 16-bit = 32 KB
    static constexpr int kSmemLD = kSmemDS + 32768;           // 2 stages x (lse2[128], D[128])
    static constexpr int kSmemBar = kSmemLD + 2 * 1024;
    static constexpr int kNumBars = 1 + 2 + 2 + 1 + 1 + 1 + 1 + 1 + 1 + 1 + 1;
    static constexpr int kSmemBytes = kSmemBar + kNumBars * 8 + 16;
    static constexpr uint32_t kTmemS = 0, kTmemDP = 128, kTmemDV = 256, kTmemDK = 256 + kD;
    static constexpr uint32_t kTmemDQ = kD == 64 ? 384 : 128;
    static constexpr bool kDqAlias = kD == 128;
};

// Rank of key tile `kb` among the contributors of its group to query tile `i`
// at this CTA's step `s` (0 = first: plain store).
__device__ __forceinline__ int bwd_dq_rank(int causal, int kb, int i, int s, int lo, int hi, int n_q) {
    if (causal) {
        const int top = min(hi - 1, i);
        return top - kb;
    }
    int rank = 0;
    for (int kp = lo; kp < hi; ++kp) {
        const int sp = (i - kp + n_q) % n_q;
        rank += sp < s;
    }
    return rank;
}

template <int kD, bool kBF16>
__global__ void __launch_bounds__(512, 1)
    mha_bwd_sm100_kernel(const __grid_constant__ CUtensorMap tm_q,
                         const __grid_constant__ CUtensorMap tm_k,
                         const __grid_constant__ CUtensorMap tm_v,
                         const __grid_constant__ CUtensorMap tm_do, const BwdParams p) {
    using Cfg = BwdCfg<kD>;
    using T16 = typename std::conditional<kBF16, __nv_bfloat16, __half>::type;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* sK = smem + Cfg::kSmemK;
    uint8_t* sV = smem + Cfg::kSmemV;
    uint8_t* sQ = smem + Cfg::kSmemQ;
    uint8_t* sDO = smem + Cfg::kSmemDO;
    uint8_t* sDS = smem + Cfg::kSmemDS;
    float* sLD = reinterpret_cast<float*>(smem + Cfg::kSmemLD);  // [stage][lse2 128 | D 128]
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::kSmemBar);
    uint64_t* kv_full = bars;
    uint64_t* q_full = bars + 1;   // [2]
    uint64_t* q_empty = bars + 3;  // [2]
    uint64_t* s_full = bars + 5;
    uint64_t* dp_full = bars + 6;
    uint64_t* p_full = bars + 7;
    uint64_t* ds_full = bars + 8;
    uint64_t* ds_free = bars + 9;
    uint64_t* dq_full = bars + 10;
    uint64_t* dq_empty = bars + 11;
    uint64_t* dkv_full = bars + 12;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + Cfg::kNumBars);
    int* item_slot = reinterpret_cast<int*>(tmem_slot + 1);

    const int warp = warp_id();
    const int lane = lane_id();

    if (threadIdx.x == 0) {
        if ((smem_u32(smem) & 1023u) != 0) __trap();
        *item_slot = atomicAdd(p.ticket, 1);
        mbar_init(kv_full, 1);
        for (int s = 0; s < 2; ++s) {
            mbar_init(q_full + s, 1);
            mbar_init(q_empty + s, 1 + 8);
        }
        mbar_init(s_full, 1);
        mbar_init(dp_full, 1);
        mbar_init(p_full, 8);
        mbar_init(ds_full, 8);
        mbar_init(ds_free, 1);
        mbar_init(dq_full, 1);
        mbar_init(dq_empty, 4);
        mbar_init(dkv_full, 1);
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int item = *item_slot;
    const int n_kb = p.n_q;
    const int bh = item / n_kb;
    const int kb = item % n_kb;
    const int N = p.N;
    const int n_steps = p.causal ? (p.n_q - kb) : p.n_q;
    auto tile_of = [&](int s) { return p.causal ? (kb + s) : ((kb + s) % p.n_q); };

    if (warp == 0) {
        // ------------------------------------------------------ TMA producer
        if (lane == 0) {
            tma_prefetch_desc(&tm_q);
            tma_prefetch_desc(&tm_k);
            tma_prefetch_desc(&tm_v);
            tma_prefetch_desc(&tm_do);
            mbar_arrive_expect_tx(kv_full, 2 * Cfg::kTileBytes);
            for (int b = 0; b < Cfg::kBoxes; ++b) {
                tma_load_3d(sK + b * 16384, &tm_k, kv_full, b * 64, kb * 128, bh);
                tma_load_3d(sV + b * 16384, &tm_v, kv_full, b * 64, kb * 128, bh);
            }
            for (int s = 0; s < n_steps; ++s) {
                const int st = s & 1;
                const int i = tile_of(s);
                mbar_wait(q_empty + st, ((s >> 1) & 1) ^ 1);
                mbar_arrive_expect_tx(q_full + st, 2 * Cfg::kTileBytes + 1024);
                for (int b = 0; b < Cfg::kBoxes; ++b) {
                    tma_load_3d(sQ + st * Cfg::kTileBytes + b * 16384, &tm_q, q_full + st, b * 64, i * 128, bh);
                    tma_load_3d(sDO + st * Cfg::kTileBytes + b * 16384, &tm_do, q_full + st, b * 64, i * 128, bh);
                }
                const size_t ro = static_cast<size_t>(bh) * p.Npad + static_cast<size_t>(i) * 128;
                bulk_load(sLD + st * 256, p.lse2 + ro, 512, q_full + st);
                bulk_load(sLD + st * 256 + 128, p.dsum + ro, 512, q_full + st);
            }
        }
    } else if (warp == 1) {
        // -------------------------------------------------------- MMA issuer
        if (lane == 0) {
            constexpr uint32_t idesc_kk = umma_idesc_f16(128, 128, kBF16, 0, 0);   // S^T, dP^T
            constexpr uint32_t idesc_kmn = umma_idesc_f16(128, kD, kBF16, 0, 1);   // dV, dK
            constexpr uint32_t idesc_mnmn = umma_idesc_f16(128, kD, kBF16, 1, 1);  // dQ
            const uint32_t aK = smem_u32(sK), aV = smem_u32(sV), aQ = smem_u32(sQ),
                           aDO = smem_u32(sDO), aDS = smem_u32(sDS);
            // X^T = A B^T with A (keys) and B (queries) both K-major [rows][D]
            auto issue_kk = [&](uint32_t dcol, uint32_t abase, uint32_t bbase) {
#pragma unroll
                for (int kk = 0; kk < kD / 16; ++kk) {
                    const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
                    mma_ss(tmem + dcol, umma_desc_sw128(abase + off, 16, 1024),
                           umma_desc_sw128(bbase + off, 16, 1024), idesc_kk, kk > 0);
                }
            };
            mbar_wait(kv_full, 0);
            tc_fence_after();
            mbar_wait(q_full + 0, 0);
            tc_fence_after();
            issue_kk(Cfg::kTmemS, aK, aQ);
            mma_commit(s_full);
            issue_kk(Cfg::kTmemDP, aV, aDO);
            mma_commit(dp_full);
            for (int s = 0; s < n_steps; ++s) {
                const int st = s & 1;
                const uint32_t qb = aQ + st * Cfg::kTileBytes;
                const uint32_t dob = aDO + st * Cfg::kTileBytes;
                // dV += P^T dO_i   (A = P^T in TMEM, 16 queries = 8 columns per step;
                // queries [64h, 64h+64) sit at columns [64h, 64h+32))
                mbar_wait(p_full, s & 1);
                tc_fence_after();
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    mma_ts(tmem + Cfg::kTmemDV, tmem + Cfg::kTmemS + (kk >> 2) * 64 + (kk & 3) * 8,
                           umma_desc_sw128(dob + kk * 2048, 16384, 1024), idesc_kmn,
                           (s > 0 || kk > 0) ? 1u : 0u);
                // next S^T can go as soon as dV has consumed P^T (in-order pipe)
                if (s + 1 < n_steps) {
                    mbar_wait(q_full + (st ^ 1), ((s + 1) >> 1) & 1);
                    tc_fence_after();
                    issue_kk(Cfg::kTmemS, aK, aQ + (st ^ 1) * Cfg::kTileBytes);
                    mma_commit(s_full);
                }
                // dK += dS^T Q_i   (A = dS^T K-major [key][query], B = Q_i MN-major)
                mbar_wait(ds_full, s & 1);
                tc_fence_after();
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
                    mma_ss(tmem + Cfg::kTmemDK, umma_desc_sw128(aDS + off, 16, 1024),
                           umma_desc_sw128(qb + kk * 2048, 16384, 1024), idesc_kmn,
                           (s > 0 || kk > 0) ? 1u : 0u);
                }
                // dQ_i = dS K   (A = dS MN-major: same tile; B = K MN-major)
                if (!Cfg::kDqAlias && s > 0) {
                    mbar_wait(dq_empty, (s - 1) & 1);
                    tc_fence_after();
                }
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    mma_ss(tmem + Cfg::kTmemDQ, umma_desc_sw128(aDS + kk * 2048, 16384, 1024),
                           umma_desc_sw128(aK + kk * 2048, 16384, 1024), idesc_mnmn, kk > 0);
                mma_commit(dq_full);
                mma_commit(ds_free);
                mma_commit(q_empty + st);
                if (s + 1 < n_steps) {
                    if (Cfg::kDqAlias) {
                        mbar_wait(dq_empty, s & 1);
                        tc_fence_after();
                    }
                    issue_kk(Cfg::kTmemDP, aV, aDO + (st ^ 1) * Cfg::kTileBytes);
                    mma_commit(dp_full);
                }
            }
            mma_commit(dkv_full);
        }
    } else if (warp >= 4 && warp < 12) {
        // ---------------------------------------------------- dS warpgroups
        const int h = (warp - 4) >> 2;                 // query-column half
        const int r = ((warp & 3) << 5) + lane;        // key row == TMEM lane
        const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
        const int key = kb * 128 + r;
        const bool key_ok = key < N;
        const float sc = p.scale_log2;
        for (int s = 0; s < n_steps; ++s) {
            const int st = s & 1;
            const int i = tile_of(s);
            const float* lse2 = sLD + st * 256 + 64 * h;
            const float* dsum = sLD + st * 256 + 128 + 64 * h;
            mbar_wait(q_full + st, (s >> 1) & 1);  // lse2 / D landed (TMA)
            mbar_wait(s_full, s & 1);
            tc_fence_after();
            uint32_t u0[32], u1[32];
            tmem_ld32(tmem + lane_base + Cfg::kTmemS + 64 * h, u0);
            tmem_ld32(tmem + lane_base + Cfg::kTmemS + 64 * h + 32, u1);
            tmem_wait_ld();
            // mask: causal diagonal tile (key > query) and keys beyond N
            const int qbase = i * 128 + 64 * h;
            const bool diag = p.causal && i == kb;
            float pr[64];
#pragma unroll
            for (int x = 0; x < 64; x += 4) {
                const float4 l4 = *reinterpret_cast<const float4*>(lse2 + x);
                const float sv[4] = {__uint_as_float(x < 32 ? u0[x] : u1[x - 32]),
                                     __uint_as_float(x < 32 ? u0[x + 1] : u1[x - 31]),
                                     __uint_as_float(x < 32 ? u0[x + 2] : u1[x - 30]),
                                     __uint_as_float(x < 32 ? u0[x + 3] : u1[x - 29])};
                const float lv[4] = {l4.x, l4.y, l4.z, l4.w};
#pragma unroll
                for (int y = 0; y < 4; ++y) {
                    float pv = ex2(fmaf(sv[y], sc, -lv[y]));
                    if (!key_ok || (diag && key > qbase + x + y)) pv = 0.0f;
                    pr[x + y] = pv;
                }
            }
            {
                uint32_t pk[32];
#pragma unroll
                for (int x = 0; x < 32; ++x) pk[x] = pack2<kBF16>(pr[2 * x], pr[2 * x + 1]);
                // own half only: the other warpgroup may still be reading its S^T columns
                tmem_st32(tmem + lane_base + Cfg::kTmemS + 64 * h, pk);
            }
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(p_full);

            // dS^T = P^T o (dP^T - D)
            mbar_wait(dp_full, s & 1);
            tc_fence_after();
            tmem_ld32(tmem + lane_base + Cfg::kTmemDP + 64 * h, u0);
            tmem_ld32(tmem + lane_base + Cfg::kTmemDP + 64 * h + 32, u1);
            tmem_wait_ld();
            uint32_t dsp[32];
#pragma unroll
            for (int x = 0; x < 64; x += 4) {
                const float4 d4 = *reinterpret_cast<const float4*>(dsum + x);
                const float dv[4] = {d4.x, d4.y, d4.z, d4.w};
                float ds[4];
#pragma unroll
                for (int y = 0; y < 4; ++y) {
                    const float dpv = __uint_as_float((x + y) < 32 ? u0[x + y] : u1[x + y - 32]);
                    ds[y] = pr[x + y] * (dpv - dv[y]);
                }
                dsp[x / 2] = pack2<kBF16>(ds[0], ds[1]);
                dsp[x / 2 + 1] = pack2<kBF16>(ds[2], ds[3]);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(q_empty + st);  // done with lse2 / D of this stage
            if (s > 0) mbar_wait(ds_free, (s - 1) & 1);
            // dS^T tile, block h = queries [64h, 64h+64): row = key, 8 x 16-B chunks
            uint8_t* blk = sDS + h * 16384;
#pragma unroll
            for (int c = 0; c < 8; ++c)
                st_swz128(blk, r, c, make_uint4(dsp[4 * c], dsp[4 * c + 1], dsp[4 * c + 2], dsp[4 * c + 3]));
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(ds_full);
        }
        // ------------------------------------------------ dK / dV epilogue
        mbar_wait(dkv_full, 0);
        tc_fence_after();
        T16* dk = reinterpret_cast<T16*>(p.dk) + (static_cast<size_t>(bh) * N + key) * kD;
        T16* dv = reinterpret_cast<T16*>(p.dv) + (static_cast<size_t>(bh) * N + key) * kD;
#pragma unroll
        for (int c = 0; c < kD / 64; ++c) {
            const int col = h * (kD / 2) + 32 * c;
            uint32_t a[32], b[32];
            tmem_ld32(tmem + lane_base + Cfg::kTmemDV + col, a);
            tmem_ld32(tmem + lane_base + Cfg::kTmemDK + col, b);
            tmem_wait_ld();
            if (key_ok) {
#pragma unroll
                for (int x = 0; x < 4; ++x) {
                    uint4 va, vb;
                    va.x = pack2<kBF16>(__uint_as_float(a[8 * x + 0]), __uint_as_float(a[8 * x + 1]));
                    va.y = pack2<kBF16>(__uint_as_float(a[8 * x + 2]), __uint_as_float(a[8 * x + 3]));
                    va.z = pack2<kBF16>(__uint_as_float(a[8 * x + 4]), __uint_as_float(a[8 * x + 5]));
                    va.w = pack2<kBF16>(__uint_as_float(a[8 * x + 6]), __uint_as_float(a[8 * x + 7]));
                    vb.x = pack2<kBF16>(__uint_as_float(b[8 * x + 0]) * p.scale, __uint_as_float(b[8 * x + 1]) * p.scale);
                    vb.y = pack2<kBF16>(__uint_as_float(b[8 * x + 2]) * p.scale, __uint_as_float(b[8 * x + 3]) * p.scale);
                    vb.z = pack2<kBF16>(__uint_as_float(b[8 * x + 4]) * p.scale, __uint_as_float(b[8 * x + 5]) * p.scale);
                    vb.w = pack2<kBF16>(__uint_as_float(b[8 * x + 6]) * p.scale, __uint_as_float(b[8 * x + 7]) * p.scale);
                    *reinterpret_cast<uint4*>(dv + col + 8 * x) = va;
                    *reinterpret_cast<uint4*>(dk + col + 8 * x) = vb;
                }
            }
        }
    } else if (warp >= 12) {
        // ------------------------------------------------------- dQ writer
        const int r = ((warp & 3) << 5) + lane;  // query row within the tile
        const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
        const int g = kb / kBwdGroup;
        const int lo = g * kBwdGroup;
        const int hi = min(lo + kBwdGroup, n_kb);
        const bool leader = warp == 12 && lane == 0;
        for (int s = 0; s < n_steps; ++s) {
            const int i = tile_of(s);
            const int rank = bwd_dq_rank(p.causal, kb, i, s, lo, hi, p.n_q);
            int* sem = p.sems + (static_cast<size_t>(g) * p.BH + bh) * p.n_q + i;
            // our turn in the group's fixed order (independent of our own dQ_i)
            if (leader && rank > 0) {
                const uint64_t t0 = globaltimer_ns();
                while (ld_acquire_gpu(sem) != rank) {
                    __nanosleep(64);
#if VATTN_WATCHDOG_NS
                    if (globaltimer_ns() - t0 > VATTN_WATCHDOG_NS) __trap();
#endif
                }
            }
            named_bar_sync(3, 128);
            mbar_wait(dq_full, s & 1);
            tc_fence_after();
            const int q = i * 128 + r;
            float* dst = p.dq_acc + ((static_cast<size_t>(g) * p.BH + bh) * N + q) * kD;
#pragma unroll
            for (int hh = 0; hh < kD / 64; ++hh) {
                uint32_t u0[32], u1[32];
                tmem_ld32(tmem + lane_base + Cfg::kTmemDQ + 64 * hh, u0);
                tmem_ld32(tmem + lane_base + Cfg::kTmemDQ + 64 * hh + 32, u1);
                tmem_wait_ld();
                if (hh == kD / 64 - 1) {
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(dq_empty);
                }
                if (q < N) {
                    float* dp = dst + 64 * hh;
#pragma unroll
                    for (int x = 0; x < 64; x += 4) {
                        const float a = __uint_as_float(x < 32 ? u0[x] : u1[x - 32]);
                        const float b = __uint_as_float(x < 32 ? u0[x + 1] : u1[x - 31]);
                        const float c = __uint_as_float(x < 32 ? u0[x + 2] : u1[x - 30]);
                        const float d = __uint_as_float(x < 32 ? u0[x + 3] : u1[x - 29]);
                        if (rank == 0)
                            *reinterpret_cast<float4*>(dp + x) = make_float4(a, b, c, d);
                        else
                            red_add_v4(dp + x, a, b, c, d);
                    }
                }
            }
            __threadfence();
            named_bar_sync(3, 128);
            if (leader) st_release_gpu(sem, rank + 1);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

// ------------------------------------------------------------ aux kernels --

// D = rowsum(dO o O) (reference compute_dpsum, attention_backward.cpp:44-57),
// lse2 = lse * log2(e), both padded to Npad (+inf / 0), plus zeroing of the
// dQ semaphores and the work ticket.  One warp per row.
template <int kD, bool kBF16>
__global__ void __launch_bounds__(256) mha_bwd_preprocess_kernel(
    const void* __restrict__ o, const void* __restrict__ dout, const float* __restrict__ lse,
    float* __restrict__ lse2, float* __restrict__ dsum, int* __restrict__ sems, int n_sems,
    int* __restrict__ ticket, int N, int Npad, int BH) {
    using T16 = typename std::conditional<kBF16, __nv_bfloat16, __half>::type;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int gthreads = gridDim.x * blockDim.x;
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < n_sems; x += gthreads) sems[x] = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) *ticket = 0;
    const int nwarps = gthreads >> 5;
    for (int row = gw; row < BH * Npad; row += nwarps) {
        const int bh = row / Npad;
        const int n = row - bh * Npad;
        float acc = 0.0f;
        float l2 = INFINITY;
        if (n < N) {
            const size_t base = (static_cast<size_t>(bh) * N + n) * kD;
            constexpr int kPer = kD / 32;  // 2 or 4 elements per lane
            const T16* po = reinterpret_cast<const T16*>(o) + base + lane * kPer;
            const T16* pd = reinterpret_cast<const T16*>(dout) + base + lane * kPer;
#pragma unroll
            for (int e = 0; e < kPer; ++e) acc += static_cast<float>(pd[e]) * static_cast<float>(po[e]);
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
            l2 = lse[static_cast<size_t>(bh) * N + n] * 1.4426950408889634f;
        }
        if (lane == 0) {
            dsum[row] = n < N ? acc : 0.0f;
            lse2[row] = l2;
        }
    }
}

// dQ = round16(scale * sum_g partial_g), groups summed in ascending order.
template <int kD, bool kBF16>
__global__ void __launch_bounds__(256) mha_dq_convert_kernel(const float* __restrict__ acc,
                                                             void* __restrict__ dq, int N, int BH,
                                                             int n_groups, int causal,
                                                             float scale) {
    using T16 = typename std::conditional<kBF16, __nv_bfloat16, __half>::type;
    const size_t total4 = static_cast<size_t>(BH) * N * kD / 4;
    const size_t gstride = static_cast<size_t>(BH) * N * kD;
    for (size_t x = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; x < total4;
         x += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int n = static_cast<int>((x * 4 / kD) % N);
        float4 s = reinterpret_cast<const float4*>(acc)[x];
        for (int g = 1; g < n_groups; ++g) {
            if (causal && n < g * kBwdGroup * 128) break;  // group g never reached this row
            const float4 t = reinterpret_cast<const float4*>(acc + g * gstride)[x];
            s.x += t.x;
            s.y += t.y;
            s.z += t.z;
            s.w += t.w;
        }
        uint2 v;
        v.x = pack2<kBF16>(s.x * scale, s.y * scale);
        v.y = pack2<kBF16>(s.z * scale, s.w * scale);
        reinterpret_cast<uint2*>(dq)[x] = v;
    }
}

}  // namespace vattn_sm100
