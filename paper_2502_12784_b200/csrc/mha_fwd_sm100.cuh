// mha_fwd_sm100.cuh -- fused multi-head-attention forward for sm_100a.
//
// Replaces vattn::forward_fused (reference: proj/src/attention_forward.cpp:191-227,
// per-unit body run_forward_unit :110-187).  Same contract: S = Q K^T * scale,
// top-left causal mask (key j visible iff j <= i, :128 and :140-144), online
// softmax (proj/src/online_softmax.cpp:21-87), P rounded to 16 bit exactly
// once before P V (:163-167), O = acc / l rounded once (:179), and
// lse = m + ln(l) in natural-log units (online_softmax.cpp:84).
//
// One CTA = one (batch*head, 256-query block) = two 128-row Q tiles that share
// every K/V tile staged in shared memory:
//   warp 0      TMA producer: Q0, Q1 once; K_j, V_j through a STAGES-deep ring
//   warp 1      MMA issuer (one thread): S_t = Q_t K_j^T (SS), O_t += P_t V_j (TS:
//               P read from tensor memory, V from shared memory, MN-major)
//   warp 2      TMEM allocator
//   warps 4-7   softmax for tile 0 (thread = query row = TMEM lane)
//   warps 8-11  softmax for tile 1
// Tensor memory (512 columns): S0 [0,128) S1 [128,256) O0 [256,256+D) O1 [256+D, 256+2D).
// P_t (16-bit, two per column) overwrites the first 64 columns of S_t.
// The MMA issue order S0(j+1) right after PV0(j), S1(j+1) right after PV1(j)
// keeps the tensor pipe busy while the other tile's softmax runs.
// O is rescaled lazily: only when a row maximum grows by more than 2^8.
#pragma once

#include "sm100_ptx.cuh"

namespace vattn_sm100 {

struct FwdParams {
    float* lse;          // [BH, N] natural-log logsumexp
    int N;               // sequence length
    int n_kv;            // ceil(N / 128)
    int causal;
    float scale_log2;    // softmax_scale * log2(e)
    int H;               // heads (dropout hash uses b and h separately)
    int bh_off;          // global index of this launch's first (b, h) unit (slabs)
    float inv_keep;      // 1 / (1 - dropout_p), binary32 like the reference
    uint64_t drop_seed;
    uint64_t drop_thresh;  // keep iff (hash >> 11) >= drop_thresh
    // optional: the keep bits, query-major [unit][query][Npad/32] words (bit = key), hashed
    // ahead of the forward by mha_dropmask_kernel (mha_forward_dropout_mask); nullptr =
    // hash every position here
    const uint32_t* drop_mask;
    int mask_words;        // Npad / 32
    // optional device word: bit VATTN_DOMAIN_ROW (1) is OR-ed in when a query row had a
    // NaN / +inf score or an empty softmax sum (l == 0), the reference's domain_error
    // cases (online_softmax.cpp:33-34, 81-82); nullptr = unchecked
    unsigned int* status;
};

template <int kD>
struct FwdCfg {
    static constexpr int kTileBytes = kD * 128 * 2;     // one 128-row 16-bit tile
    static constexpr int kBoxes = kD / 64;              // 64-column TMA boxes per tile
#ifndef VATTN_FWD_STAGES128
#define VATTN_FWD_STAGES128 4
#endif
    static constexpr int kStages = kD == 128 ? VATTN_FWD_STAGES128 : 8;   // K/V ring depth
    static constexpr int kSmemQ = 0;                    // Q0, Q1
    static constexpr int kSmemKV = 2 * kTileBytes;
    static constexpr int kSmemBar = kSmemKV + kStages * kTileBytes;
    static constexpr int kNumBars = 1 + 2 * kStages + 2 + 8 + 2;
    static constexpr int kSmemBytes = kSmemBar + kNumBars * 8 + 16;
    static constexpr int kThreads = 384;
    static constexpr uint32_t kTmemO = 256;
};

template <int kD, bool kBF16, bool kDrop>
__global__ void __launch_bounds__(384, 1)
    mha_fwd_sm100_kernel(const __grid_constant__ CUtensorMap tm_q,
                         const __grid_constant__ CUtensorMap tm_k,
                         const __grid_constant__ CUtensorMap tm_v,
                         const __grid_constant__ CUtensorMap tm_o, const FwdParams p) {
    VCTA(0, 0);
    using Cfg = FwdCfg<kD>;
    constexpr int kVtraceKid = 0;
    (void)kVtraceKid;
    constexpr int S = Cfg::kStages;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* sQ = smem + Cfg::kSmemQ;
    uint8_t* sKV = smem + Cfg::kSmemKV;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::kSmemBar);
    uint64_t* q_full = bars;
    uint64_t* kv_full = bars + 1;
    uint64_t* kv_empty = kv_full + S;
    uint64_t* s_full = kv_empty + S;
    uint64_t* p_full = s_full + 2;
    uint64_t* o_done = p_full + 8;  // p_full: [tile][quarter]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + Cfg::kNumBars);

    const int warp = warp_id();
    const int lane = lane_id();
    const int nqb = (p.N + 255) / 256;
    const int bh = grid_bh(nqb);
    const int qblk = p.causal ? (nqb - 1 - grid_tile(nqb)) : grid_tile(nqb);
    const int q0 = qblk * 256;
    const int N = p.N;

    int nk[2];
#pragma unroll
    for (int t = 0; t < 2; ++t) {
        const int r0 = q0 + 128 * t;
        nk[t] = r0 >= N ? 0 : (p.causal ? (r0 / 128 + 1) : p.n_kv);
    }
    const int nkmax = nk[0] > nk[1] ? nk[0] : nk[1];

    if (threadIdx.x == 0) {
        if ((smem_u32(smem) & 1023u) != 0) __trap();
        mbar_init(q_full, 1);
        for (int s = 0; s < S; ++s) {
            mbar_init(kv_full + s, 1);
            mbar_init(kv_empty + s, 1);
        }
        for (int t = 0; t < 2; ++t) {
            mbar_init(s_full + t, 1);
            for (int qq = 0; qq < 4; ++qq) mbar_init(p_full + 4 * t + qq, 4);  // one arrive per warp
            mbar_init(o_done + t, 1);
        }
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    griddep_wait();  // inputs written by the previous kernel in the stream are visible
    // registers: producer/MMA warpgroup 88, softmax warpgroups 208 (384 x 168 budget);
    // each role lowers/raises its own budget inside its branch.
    if (warp < 4) regs_dec<88>();

    if (warp == 0) {
        // ------------------------------------------------------ TMA producer
        if (lane == 0) {
            tma_prefetch_desc(&tm_q);
            tma_prefetch_desc(&tm_k);
            tma_prefetch_desc(&tm_v);
            tma_prefetch_desc(&tm_o);
            const int nvalid = (nk[0] > 0) + (nk[1] > 0);
            mbar_arrive_expect_tx(q_full, nvalid * Cfg::kTileBytes);
            for (int t = 0; t < 2; ++t) {
                if (nk[t] == 0) continue;
                for (int b = 0; b < Cfg::kBoxes; ++b)
                    tma_load_3d(sQ + t * Cfg::kTileBytes + b * 16384, &tm_q, q_full, b * 64,
                                q0 + 128 * t, bh);
            }
            for (int j = 0; j < nkmax; ++j) {
                stress_delay(4, j);
#pragma unroll
                for (int w = 0; w < 2; ++w) {
                    const int pos = 2 * j + w;
                    const int slot = pos % S;
                    const uint32_t ph = (pos / S) & 1;
                    mbar_wait<VATTN_SLEEP_PRODUCER>(kv_empty + slot, ph ^ 1);
                    mbar_arrive_expect_tx(kv_full + slot, Cfg::kTileBytes);
                    uint8_t* dst = sKV + slot * Cfg::kTileBytes;
                    const CUtensorMap* map = w == 0 ? &tm_k : &tm_v;
                    for (int b = 0; b < Cfg::kBoxes; ++b)
                        tma_load_3d(dst + b * 16384, map, kv_full + slot, b * 64, j * 128, bh);
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer (whole warp,
        // warp-uniform descriptors; one elected lane issues each tcgen05 op)
        constexpr uint32_t idesc_s = umma_idesc_f16(128, 128, kBF16, 0, 0);
        constexpr uint32_t idesc_o = umma_idesc_f16(128, kD, kBF16, 0, 1);
        constexpr uint64_t kTile16 = Cfg::kTileBytes >> 4;
        const uint64_t dQ0 = umma_desc_sw128(smem_u32(sQ), 16, 1024);      // K-major Q tiles
        const uint64_t dK0 = umma_desc_sw128(smem_u32(sKV), 16, 1024);     // K-major K slots
        const uint64_t dV0 = umma_desc_sw128(smem_u32(sKV), 16384, 1024);  // MN-major V slots
        auto issue_s = [&](int t, int j) {
            const uint64_t qd = dQ0 + t * kTile16;
            const uint64_t kd = dK0 + ((2 * j) % S) * kTile16;
#pragma unroll
            for (int kk = 0; kk < kD / 16; ++kk)
                mma_ss_e(tmem + 128 * t, desc_kmajor(qd, kk), desc_kmajor(kd, kk), idesc_s, kk > 0);
            mma_commit_e(s_full + t);
        };
        auto issue_pv = [&](int t, int j) {
            const uint64_t vd = dV0 + ((2 * j + 1) % S) * kTile16;
            // P arrives in four 32-key quarters: each pair of K=16 steps starts as
            // soon as its quarter is in tensor memory (the softmax is still
            // exponentiating the rest of the row).
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) {
                mbar_wait_mma(p_full + 4 * t + qq, j & 1);
                tc_fence_after();
#pragma unroll
                for (int k2 = 0; k2 < 2; ++k2) {
                    const int kk = 2 * qq + k2;
                    mma_ts_e(tmem + Cfg::kTmemO + kD * t, tmem + 128 * t + kk * 8, desc_mnmajor(vd, kk),
                             idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
                }
            }
            mma_commit_e(o_done + t);
        };
        auto wait_kv = [&](int pos) {
            mbar_wait_mma(kv_full + (pos % S), (pos / S) & 1);
            tc_fence_after();
        };
        mbar_wait_mma(q_full, 0);
        tc_fence_after();
        VTRACE(3072);
        if (nkmax > 0) {
            wait_kv(0);
            for (int t = 0; t < 2; ++t)
                if (nk[t] > 0) issue_s(t, 0);
            mma_commit_e(kv_empty + 0);
        }
        for (int j = 0; j < nkmax; ++j) {
            stress_delay(3, j);
            wait_kv(2 * j + 1);
            bool k_next = false;
#pragma unroll
            for (int t = 0; t < 2; ++t) {
                if (j < nk[t]) {
                    issue_pv(t, j);
                    VTRACE(8 * j + 4 * t + 0);
                    if (j + 1 < nk[t]) {
                        if (!k_next) {
                            wait_kv(2 * j + 2);
                            k_next = true;
                        }
                        VTRACE(8 * j + 4 * t + 1);
                        issue_s(t, j + 1);
                    }
                }
            }
            mma_commit_e(kv_empty + (2 * j + 1) % S);
            if (k_next) mma_commit_e(kv_empty + (2 * j + 2) % S);
        }
    } else if (warp >= 4) {
        // ----------------------------------------------------------- softmax
        regs_inc<208>();
        const int t = (warp - 4) >> 2;           // Q tile of this warpgroup
        const int r = ((warp & 3) << 5) + lane;  // row within tile == TMEM lane
        const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
        const uint32_t tS = tmem + lane_base + 128 * t;
        const uint32_t tO = tmem + lane_base + Cfg::kTmemO + kD * t;
        const int row = q0 + 128 * t + r;
        const float sc = p.scale_log2;
        DropRow drow{};
        if constexpr (kDrop) drow = drop_row(drop_bh_base(p.drop_seed, (bh + p.bh_off) / p.H, (bh + p.bh_off) % p.H), row);
        float m_run = -INFINITY;  // running max, log2 units (already scaled)
        float l_run = 0.0f;
        bool bad = false;         // a NaN or +inf score in this row (FMNMX.NAN keeps NaN in mx)
        const int ntile = t ? nk[1] : nk[0];
        for (int j = 0; j < ntile; ++j) {
            mbar_wait<VATTN_SLEEP_MATH>(s_full + t, j & 1);
            // O += P V of the previous tile has landed (issued before S(j), so this wait
            // returns at once): observing every o_done phase in order keeps the parity
            // waits unambiguous by construction (compute-sanitizer synccheck clean)
            if (j > 0) mbar_wait<VATTN_SLEEP_MATH>(o_done + t, (j - 1) & 1);
            tc_fence_after();
            stress_delay(1, j);
            if ((warp & 3) == 0 && lane == 0) VTRACE(1024 + 8 * j + 4 * t + 0);
            uint4 kw4 = make_uint4(0u, 0u, 0u, 0u);  // this row's keep bits of key tile j
            if (kDrop && p.drop_mask && row < p.mask_words * 32)
                kw4 = __ldg(reinterpret_cast<const uint4*>(p.drop_mask + (static_cast<size_t>(bh) * p.mask_words * 32 + row) *
                                                                             p.mask_words + j * 4));
            float s[128];
            tmem_ld32f(tS + 0, s);
            tmem_ld32f(tS + 32, s + 32);
            tmem_ld32f(tS + 64, s + 64);
            tmem_ld32f(tS + 96, s + 96);
            tmem_wait_ld();
            if ((warp & 3) == 0 && lane == 0) VTRACE(2048 + 8 * j + 4 * t + 0);
            // (tile-uniform) masking: causal diagonal tile (keys > row) or keys beyond N
            const bool tile_masked = p.causal ? (j == ntile - 1) : (j == p.n_kv - 1 && (N & 127) != 0);
            int lim = 127;
            if (p.causal && j == ntile - 1) lim = r;  // diagonal: j*128 == tile row base
            if (!p.causal && j == p.n_kv - 1) lim = min(lim, N - j * 128 - 1);
            if (tile_masked) {
#pragma unroll
                for (int c = 0; c < 128; ++c)
                    if (c > lim) s[c] = -INFINITY;
            }
            // row max: tree of 3-input maxima
            const float mx = row_max<128>(s);
            bad |= !(mx < INFINITY);
            const float m_tile = mx * sc;
            if ((warp & 3) == 0 && lane == 0) VTRACE(2048 + 8 * j + 4 * t + 1);
            if (j == 0) {
                m_run = m_tile;
            } else if (__any_sync(0xffffffffu, m_tile > m_run + 8.0f)) {
                // Lazy rescale (warp-uniform: tcgen05.ld/st are .sync.aligned).  The
                // previous P V must have landed before O is touched.  Rows whose max
                // did not grow enough keep their stale max (factor 1).
                float f = 1.0f;
                if (m_tile > m_run) {
                    f = ex2(m_run - m_tile);
                    m_run = m_tile;
                }
                l_run *= f;
#pragma unroll
                for (int c = 0; c < kD / 32; ++c) {
                    uint32_t u[32];
                    tmem_ld32(tO + 32 * c, u);
                    tmem_wait_ld();
#pragma unroll
                    for (int x = 0; x < 32; ++x) u[x] = __float_as_uint(__uint_as_float(u[x]) * f);
                    tmem_st32(tO + 32 * c, u);
                }
            }
            const float m_use = m_run == -INFINITY ? 0.0f : m_run;
            if ((warp & 3) == 0 && lane == 0) VTRACE(2048 + 8 * j + 4 * t + 2);
            const float2 sc2 = make_float2(sc, sc);
            const float2 nm2 = make_float2(-m_use, -m_use);
            float2 ls2[2] = {make_float2(0.0f, 0.0f), make_float2(0.0f, 0.0f)};  // row-sum partials
            // P in four 32-key quarters (16 packed columns each); the MMA warp
            // starts P V on a quarter as soon as it lands.  The tensor-memory store
            // of quarter q completes (wait::st) while quarter q+1 is computed, so
            // the store latency never sits on the softmax's critical path.
            auto quarter = [&](int qq, uint32_t (&pk)[16], auto poly_pair) {
                uint32_t kw = qq == 0 ? kw4.x : qq == 1 ? kw4.y : qq == 2 ? kw4.z : kw4.w;
                if (kDrop && !p.drop_mask) {  // no pre-hashed bits: hash this quarter's 32 keys here
                    kw = 0;
#pragma unroll 1
                    for (int b = 0; b < 32; ++b)
                        kw |= static_cast<uint32_t>(drop_keep(drow, j * 128 + 32 * qq + b, p.drop_thresh)) << b;
                }
#pragma unroll
                for (int x = 0; x < 16; ++x) {
                    const int c = 32 * qq + 2 * x;
                    const float2 v = ffma2(make_float2(s[c], s[c + 1]), sc2, nm2);
                    float2 pp;
                    if (poly_pair(qq * 16 + x)) {
                        pp = ex2_poly2(v);
                    } else {
                        pp.x = ex2(v.x);
                        pp.y = ex2(v.y);
                    }
                    ls2[x & 1] = fadd2(ls2[x & 1], pp);  // l uses the weights before dropout
                    pk[x] = pack2<kBF16>(pp.x, pp.y);
                    if constexpr (kDrop) {
                        // dropout on the 16-bit P: f16(f16(P) * 1/(1-p)) or 0
                        // (attention_forward.cpp:94-106)
                        const float2 f = unpack2<kBF16>(pk[x]);
                        const bool k0 = (kw >> (2 * x)) & 1u, k1 = (kw >> (2 * x + 1)) & 1u;
                        pk[x] = pack2<kBF16>(k0 ? f.x * p.inv_keep : 0.0f, k1 ? f.y * p.inv_keep : 0.0f);
                    }
                }
                (void)kw;
            };
            auto publish = [&](int qq) {  // quarter qq's tcgen05.st has been waited on
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(p_full + 4 * t + qq);
                if ((warp & 3) == 0 && lane == 0) VTRACE((qq < 3 ? 1024 + 1 + qq : 2048 + 3) + 8 * j + 4 * t);
            };
            auto emit_row = [&](auto poly_pair) {
                uint32_t pa[16], pb[16];
                quarter(0, pa, poly_pair);
                tmem_st16(tS + 0, pa);
                quarter(1, pb, poly_pair);
                tmem_wait_st();
                publish(0);
                tmem_st16(tS + 16, pb);
                quarter(2, pa, poly_pair);
                tmem_wait_st();
                publish(1);
                tmem_st16(tS + 32, pa);
                quarter(3, pb, poly_pair);
                tmem_wait_st();
                publish(2);
                tmem_st16(tS + 48, pb);
                tmem_wait_st();
                publish(3);
            };
            constexpr int kPer = PolyPeriod<kD>::fwd;
            auto poly_fast = [](int pair) {
                if constexpr (kPer > 0) return pair % kPer == kPer - 1;
                return false;
            };
            auto poly_none = [](int) { return false; };  // -inf -> exact 0 on masked tiles
            if (tile_masked)  // warp-uniform: tcgen05.st is .sync.aligned
                emit_row(poly_none);
            else
                emit_row(poly_fast);
            const float2 lsum = fadd2(ls2[0], ls2[1]);
            l_run += lsum.x + lsum.y;
        }
        if (ntile > 0) {
            // ------------------------------------------------------ epilogue
            mbar_wait<VATTN_SLEEP_MATH>(o_done + t, (ntile - 1) & 1);
            tc_fence_after();
            const float inv_l = l_run > 0.0f ? 1.0f / l_run : 0.0f;
            if (row < N) {
                const float m_use = m_run == -INFINITY ? 0.0f : m_run;
                p.lse[static_cast<size_t>(bh) * N + row] = (m_use + lg2(l_run)) * 0.69314718055994530942f;
                if (p.status && (bad || !(l_run > 0.0f))) atomicOr(p.status, 1u);
            }
            uint8_t* sO = sQ + t * Cfg::kTileBytes;  // Q_t is dead once the last S_t landed
#pragma unroll
            for (int c = 0; c < kD / 32; ++c) {
                uint32_t u[32];
                tmem_ld32(tO + 32 * c, u);
                tmem_wait_ld();
#pragma unroll
                for (int x = 0; x < 4; ++x) {
                    uint4 v;
                    v.x = pack2<kBF16>(__uint_as_float(u[8 * x + 0]) * inv_l, __uint_as_float(u[8 * x + 1]) * inv_l);
                    v.y = pack2<kBF16>(__uint_as_float(u[8 * x + 2]) * inv_l, __uint_as_float(u[8 * x + 3]) * inv_l);
                    v.z = pack2<kBF16>(__uint_as_float(u[8 * x + 4]) * inv_l, __uint_as_float(u[8 * x + 5]) * inv_l);
                    v.w = pack2<kBF16>(__uint_as_float(u[8 * x + 6]) * inv_l, __uint_as_float(u[8 * x + 7]) * inv_l);
                    const int col = 32 * c + 8 * x;  // first of 8 columns
                    st_swz128(sO + (col >> 6) * 16384, r, (col & 63) >> 3, v);
                }
            }
            fence_proxy_async_smem();
            named_bar_sync(1 + t, 128);
            if (warp == 4 + 4 * t && lane == 0) {
                for (int b = 0; b < Cfg::kBoxes; ++b)
                    tma_store_3d(&tm_o, sO + b * 16384, b * 64, q0 + 128 * t, bh);
                bulk_commit();
                bulk_wait_read0();
            }
        }
    }
    griddep_launch_dependents();
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
    VCTA(0, 1);
}

}  // namespace vattn_sm100
