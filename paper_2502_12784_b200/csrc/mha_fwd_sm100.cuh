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
// Option (VATTN_FWD_SEPP=1, d = 64 only -- O needs only 128 columns): P_t lives in its
// own region [384 + 64t, +64), so S_t(j+1) is issued as soon as the softmax has read
// S_t(j) into registers (s_free) and the softmax warpgroups never wait for S (issue
// order S0(j+1), S1(j+1), PV0(j), PV1(j)).  Measured (profiles/r2_experiments.md): the
// two warpgroups then run in lock step on the shared MUFU and the step period stays
// ~3500 clk -- C4 forward +4 %, C2 N >= 1k -4..-9 % -- so it is off.
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
    // items = (unit, 256-query block) in the order of the (nqb * G, units / G) grid
    // (tile_grid); CTA c takes items c, c + stride, ... (persistent when stride < items)
    int items, group, stride;
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
    // Softmax warpgroups per Q tile (VATTN_FWD_HALVES): 1 = one warpgroup per tile owns
    // whole rows (default); 2 = each owns 64 of the 128 key columns of its rows (four
    // softmax warpgroups, 640 threads), the row max / sum exchanged through shared
    // memory.  Measured 1.2-2.7x slower (register cap 104 at 640 threads -- 112 deadlocks
    // setmaxnreg.inc, the launch allocation is 640 x 96 -- spills at d = 128, and a
    // 256-thread barrier per step), profiles/r2_experiments.md.
#ifndef VATTN_FWD_HALVES
#define VATTN_FWD_HALVES 1
#endif
    static constexpr int kHalves = VATTN_FWD_HALVES;
    static constexpr int kSmemX = kSmemKV + kStages * kTileBytes;  // [3 slots][2 tiles][kHalves][128] f32
    static constexpr int kSmemBar = kSmemX + 3 * 2 * kHalves * 128 * 4;
    static constexpr int kNumBars = 1 + 2 * kStages + 2 + 8 + 2 + 2 + 3;  // ..., o_done[2], s_free[2], q_free, o_free[2]
    // dropout keep bits, staged per softmax thread one key tile ahead (cp.async):
    // [2 buffers][256 kHalves threads][16 B] -- in registers the prefetch spilled S
    static constexpr int kSmemMask = (kSmemBar + kNumBars * 8 + 16 + 127) / 128 * 128;
    static constexpr int kMaskBuf = 256 * kHalves * 16;
    static constexpr int kSmemBytes = kSmemMask + 2 * kMaskBuf;
    // Warps: producer 0, MMA 1, TMEM allocator 2, idle 3, softmax warpgroups from warp 4.
    // setmaxnreg split of the CTA's launch allocation: 88 / 208 (384 threads x 168) or,
    // two halves (640 threads x 96), VATTN_FWD_REGS_LO / VATTN_FWD_REGS_HI.
#ifndef VATTN_FWD_REGS_LO
#define VATTN_FWD_REGS_LO 56
#endif
    static constexpr int kMathWarp0 = 4;
    static constexpr int kAllocWarp = 2;
    static constexpr int kThreads = 128 + 256 * kHalves;
    static constexpr uint32_t kRegsLo = kHalves == 1 ? 88 : VATTN_FWD_REGS_LO;
#ifndef VATTN_FWD_REGS_HI
#define VATTN_FWD_REGS_HI 104
#endif
    static constexpr uint32_t kRegsHi = kHalves == 1 ? 208 : VATTN_FWD_REGS_HI;
    static_assert(128 * kRegsLo + 256 * kHalves * kRegsHi <= 65536, "register split");
    static constexpr uint32_t kTmemO = 256;
#ifndef VATTN_FWD_SEPP
#define VATTN_FWD_SEPP 0
#endif
    static constexpr bool kSepP = kD == 64 && VATTN_FWD_SEPP;  // P in its own region (see above)
    static constexpr uint32_t kTmemP = 384;          // kSepP: P_t at [384 + 64t, +64)
};
#ifndef VATTN_FWD_SPEC_MAX
#define VATTN_FWD_SPEC_MAX 0
#endif
constexpr bool kSpecMax = VATTN_FWD_SPEC_MAX;  // speculative first quarter (see the softmax loop)
// Masked (diagonal / ragged) tiles on MUFU only (a second unrolled copy of the softmax
// body); 0 = the same polynomial split as every tile (ex2_poly2(-inf) is exactly 0 too).
#ifndef VATTN_FWD_MASKED_MUFU
#define VATTN_FWD_MASKED_MUFU 0
#endif
constexpr bool kMaskedMufu = VATTN_FWD_MASKED_MUFU;
// O rescale / epilogue column loops: 1 = rolled (smaller kernel), 4 = unrolled
#ifndef VATTN_FWD_RESCALE_UNROLL
#define VATTN_FWD_RESCALE_UNROLL 4
#endif
constexpr int kRescaleUnroll = VATTN_FWD_RESCALE_UNROLL;

// kMulti: persistent CTAs looping over several items (host: N <= 1024); false compiles the
// one-item-per-CTA kernel with the item loop folded away.
// kDropMode: 0 no dropout; 1 keep bits read from the pre-hashed mask (mha_dropmask_kernel);
// 2 keep bits hashed in the softmax (no mask buffer).  Separate instantiations: the
// in-softmax hash loop needs registers that, compiled into the mask path, made ptxas spill
// S columns to local memory on every tile.
template <int kD, bool kBF16, int kDropMode, bool kMulti = false>
__global__ void __launch_bounds__(FwdCfg<kD>::kThreads, 1)
    mha_fwd_sm100_kernel(const __grid_constant__ CUtensorMap tm_q,
                         const __grid_constant__ CUtensorMap tm_k,
                         const __grid_constant__ CUtensorMap tm_v,
                         const __grid_constant__ CUtensorMap tm_o, const FwdParams p) {
    VCTA(0, 0);
    griddep_start();
    constexpr bool kDrop = kDropMode != 0;
    constexpr bool kMaskBits = kDropMode == 1;
    using Cfg = FwdCfg<kD>;
    constexpr int kVtraceKid = 0;
    (void)kVtraceKid;
    constexpr int S = Cfg::kStages;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* sQ = smem + Cfg::kSmemQ;
    uint8_t* sKV = smem + Cfg::kSmemKV;
    float* sX = reinterpret_cast<float*>(smem + Cfg::kSmemX);  // row max / sum exchange between column halves
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::kSmemBar);
    uint64_t* q_full = bars;
    uint64_t* kv_full = bars + 1;
    uint64_t* kv_empty = kv_full + S;
    uint64_t* s_full = kv_empty + S;
    uint64_t* p_full = s_full + 2;
    uint64_t* o_done = p_full + 8;  // p_full: [tile][quarter]
    uint64_t* s_free = o_done + 2;  // kSepP: the softmax has S_t(j) in registers
    // persistent CTAs: both tiles' O stores have left sQ (the next item's Q may land) /
    // the epilogue has read O_t out of tensor memory (the next item's first P V may write)
    uint64_t* q_free = s_free + 2;
    uint64_t* o_free = q_free + 1;  // [2]
    constexpr bool kSepP = Cfg::kSepP;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + Cfg::kNumBars);

    const int warp = warp_id();
    const int lane = lane_id();
    const int nqb = (p.N + 255) / 256;
    const int N = p.N;
    const int lin = static_cast<int>(blockIdx.x + blockIdx.y * gridDim.x);
    struct Item {
        int bh, q0, nk[2], nkmax;
    };
    auto item_at = [&](int it, Item& x) -> bool {
        if (!kMulti && it > 0) return false;
        const int L = kMulti ? lin + it * p.stride : lin;
        if (kMulti && !p.causal && L >= p.items) return false;
        int tile;
        if (kMulti && p.causal) {
            // causal items differ in length: longest first (tile-major) in a zigzag over
            // the CTAs so every CTA's total is balanced (short heads: their K/V fit in L2)
            const int units_ = p.items / nqb;
            const int idx = (it & 1) ? it * p.stride + (p.stride - 1 - lin) : L;
            if (idx >= p.items) return false;
            tile = idx / units_;
            x.bh = idx - tile * units_;
        } else {
            const int W = nqb * p.group;  // grid x extent of tile_grid
            const int bx = L % W, by = L / W;
            x.bh = by * p.group + bx % p.group;
            tile = bx / p.group;
        }
        const int qblk = p.causal ? (nqb - 1 - tile) : tile;
        x.q0 = qblk * 256;
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            const int r0 = x.q0 + 128 * t;
            x.nk[t] = r0 >= N ? 0 : (p.causal ? (r0 / 128 + 1) : p.n_kv);
        }
        x.nkmax = x.nk[0] > x.nk[1] ? x.nk[0] : x.nk[1];
        return true;
    };

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
            mbar_init(s_free + t, 4 * Cfg::kHalves);  // one arrive per warp of the tile
            mbar_init(o_free + t, 4 * Cfg::kHalves);
        }
        mbar_init(q_free, 2);  // one arrive per tile (its O store thread)
        fence_barrier_init();
    }
    if (warp == Cfg::kAllocWarp) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    griddep_wait();  // inputs written by the previous kernel in the stream are visible
    // registers (one warpgroup per tile): producer/MMA warpgroup 88, softmax warpgroups
    // 208 (384 x 168 budget); each role lowers/raises its own budget inside its branch.
    if (warp < 4) regs_dec<Cfg::kRegsLo>();

    if (warp == 0) {
        // ------------------------------------------------------ TMA producer
        if (lane == 0) {
            tma_prefetch_desc(&tm_q);
            tma_prefetch_desc(&tm_k);
            tma_prefetch_desc(&tm_v);
            tma_prefetch_desc(&tm_o);
            uint32_t kvb = 0;  // K/V ring position at the item's start (2 per key step)
            Item x;
            for (int it = 0; item_at(it, x); ++it) {
                const int bh = x.bh;
                if (it > 0) mbar_wait(q_free, (it - 1) & 1);  // the previous item's O stores left sQ
                const int nvalid = (x.nk[0] > 0) + (x.nk[1] > 0);
                mbar_arrive_expect_tx(q_full, nvalid * Cfg::kTileBytes);
                for (int t = 0; t < 2; ++t) {
                    if (x.nk[t] == 0) continue;
                    for (int b = 0; b < Cfg::kBoxes; ++b)
                        tma_load_3d(sQ + t * Cfg::kTileBytes + b * 16384, &tm_q, q_full, b * 64, x.q0 + 128 * t, bh);
                }
                for (int j = 0; j < x.nkmax; ++j) {
                    stress_delay(4, j);
#pragma unroll
                    for (int w = 0; w < 2; ++w) {
                        const uint32_t pos = kvb + 2 * j + w;
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
                kvb += 2 * x.nkmax;
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
        uint32_t kvb = 0;              // K/V ring position at the item's start
        uint32_t ts[2] = {0u, 0u};     // steps of tile t in this CTA's earlier items (phases)
        auto issue_s = [&](int t, int j) {
            const uint64_t qd = dQ0 + t * kTile16;
            const uint64_t kd = dK0 + ((kvb + 2 * j) % S) * kTile16;
#pragma unroll
            for (int kk = 0; kk < kD / 16; ++kk)
                mma_ss_e(tmem + 128 * t, desc_kmajor(qd, kk), desc_kmajor(kd, kk), idesc_s, kk > 0);
            mma_commit_e(s_full + t);
        };
        int it = 0;  // item of this CTA (o_free phases)
        auto issue_pv = [&](int t, int j) {
            const uint64_t vd = dV0 + ((kvb + 2 * j + 1) % S) * kTile16;
            if (j == 0 && it > 0) {  // the previous item's epilogue has read O_t
                mbar_wait_mma(o_free + t, (it - 1) & 1);
                tc_fence_after();
            }
            // P arrives in four 32-key quarters: each pair of K=16 steps starts as
            // soon as its quarter is in tensor memory (the softmax is still
            // exponentiating the rest of the row).
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) {
                mbar_wait_mma(p_full + 4 * t + qq, (ts[t] + j) & 1);
                tc_fence_after();
#pragma unroll
                for (int k2 = 0; k2 < 2; ++k2) {
                    const int kk = 2 * qq + k2;
                    const uint32_t pcol = kSepP ? Cfg::kTmemP + 64 * t : 128 * t;
                    mma_ts_e(tmem + Cfg::kTmemO + kD * t, tmem + pcol + kk * 8, desc_mnmajor(vd, kk),
                             idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
                }
            }
            mma_commit_e(o_done + t);
        };
        auto wait_kv = [&](uint32_t pos) {
            mbar_wait_mma(kv_full + (pos % S), (pos / S) & 1);
            tc_fence_after();
        };
        Item x;
        for (; item_at(it, x); ++it) {
            const int nk[2] = {x.nk[0], x.nk[1]};  // (registers: every use is unrolled over t)
            const int nkmax = x.nkmax;
            mbar_wait_mma(q_full, it & 1);
            tc_fence_after();
            VTRACE(3072);
            if (nkmax > 0) {
                wait_kv(kvb);
                for (int t = 0; t < 2; ++t)
                    if (nk[t] > 0) issue_s(t, 0);
                mma_commit_e(kv_empty + kvb % S);
            }
            for (int j = 0; j < nkmax; ++j) {
                stress_delay(3, j);
                bool k_next = false;
                if constexpr (kSepP) {
                    // S_t(j+1) as soon as the softmax read S_t(j); then P V of tile j
#pragma unroll
                    for (int t = 0; t < 2; ++t) {
                        if (j + 1 < nk[t]) {
                            if (!k_next) {
                                wait_kv(kvb + 2 * j + 2);
                                k_next = true;
                            }
                            mbar_wait_mma(s_free + t, (ts[t] + j) & 1);
                            tc_fence_after();
                            VTRACE(8 * j + 4 * t + 1);
                            issue_s(t, j + 1);
                        }
                    }
                    wait_kv(kvb + 2 * j + 1);
#pragma unroll
                    for (int t = 0; t < 2; ++t) {
                        if (j < nk[t]) {
                            issue_pv(t, j);
                            VTRACE(8 * j + 4 * t + 0);
                        }
                    }
                    mma_commit_e(kv_empty + (kvb + 2 * j + 1) % S);
                    if (k_next) mma_commit_e(kv_empty + (kvb + 2 * j + 2) % S);
                    continue;
                }
                wait_kv(kvb + 2 * j + 1);
#pragma unroll
                for (int t = 0; t < 2; ++t) {
                    if (j < nk[t]) {
                        issue_pv(t, j);
                        VTRACE(8 * j + 4 * t + 0);
                        if (j + 1 < nk[t]) {
                            if (!k_next) {
                                wait_kv(kvb + 2 * j + 2);
                                k_next = true;
                            }
                            VTRACE(8 * j + 4 * t + 1);
                            issue_s(t, j + 1);
                        }
                    }
                }
                mma_commit_e(kv_empty + (kvb + 2 * j + 1) % S);
                if (k_next) mma_commit_e(kv_empty + (kvb + 2 * j + 2) % S);
            }
            kvb += 2 * nkmax;
            ts[0] += nk[0];
            ts[1] += nk[1];
        }
    } else if (warp >= Cfg::kMathWarp0) {
        // ----------------------------------------------------------- softmax
        // Warpgroup g: Q tile t = g / kH, key-column half c = g % kH (kC columns of S,
        // kD / kH columns of O, P quarters [kQ c, kQ c + kQ)).  Thread = query row = TMEM
        // lane.  With two halves the row max and the final row sum are exchanged
        // through shared memory (one 256-thread named barrier per step).
        regs_inc<Cfg::kRegsHi>();
        constexpr int kH = Cfg::kHalves;
        constexpr int kC = 128 / kH;             // S columns per warpgroup
        constexpr int kQ = 4 / kH;               // P quarters per warpgroup
        constexpr int kOC = kD / kH;             // O columns per warpgroup
        const int g = (warp - Cfg::kMathWarp0) >> 2;
        const int t = g / kH;                    // Q tile of this warpgroup
        const int c = g % kH;                    // column half
        const int r = ((warp & 3) << 5) + lane;  // row within tile == TMEM lane
        const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
        const uint32_t tS = tmem + lane_base + 128 * t + kC * c;
        const uint32_t tO = tmem + lane_base + Cfg::kTmemO + kD * t + kOC * c;
        // P_t (16-bit pairs, 64 columns per tile; quarter q at +16 q)
        const uint32_t tP = (kSepP ? tmem + lane_base + Cfg::kTmemP + 64 * t : tmem + lane_base + 128 * t) + 16 * kQ * c;
        const uint32_t xbar = 3 + t;             // named barrier of the tile's warpgroups
        auto xslot = [&](int slot, int half) { return sX + ((slot * 2 + t) * kH + half) * 128; };
        const float sc = p.scale_log2;
        uint32_t ts = 0;  // steps of this tile in the CTA's earlier items (phases)
        Item x_;
        for (int it = 0; item_at(it, x_); ++it) {
        const int bh = x_.bh, q0 = x_.q0;
        const int row = q0 + 128 * t + r;
        float m_run = -INFINITY;  // running max, log2 units (already scaled)
        float l_run = 0.0f;       // this half's row sum
        bool bad = false;         // a NaN or +inf score in this row (FMNMX.NAN keeps NaN in mx)
        const int ntile = t ? x_.nk[1] : x_.nk[0];
        // this row's keep bits of key tile jt -> staging buffer buf (cp.async, one tile ahead;
        // rows past the mask (padding) read zeros)
        const uint32_t mslot = smem_u32(smem + Cfg::kSmemMask) + static_cast<uint32_t>(g * 128 + r) * 16u;
        auto mask_fetch = [&](int jt, uint32_t buf) {
            const bool ok = row < p.mask_words * 32;
            const uint32_t* src =
                ok ? p.drop_mask + (static_cast<size_t>(bh) * p.mask_words * 32 + row) * p.mask_words + jt * 4 : p.drop_mask;
            cp_async16(mslot + buf * Cfg::kMaskBuf, src, ok ? 16u : 0u);
            cp_async_commit();
        };
        if (kMaskBits && ntile > 0) mask_fetch(0, ts & 1);
        for (int j = 0; j < ntile; ++j) {
            const uint32_t gj = ts + j;  // this tile's step across items (barrier phases)
            mbar_wait<VATTN_SLEEP_MATH>(s_full + t, gj & 1);
            // O += P V of the previous tile has landed (issued before S(j), so this wait
            // returns at once): observing every o_done phase in order keeps the parity
            // waits unambiguous by construction (compute-sanitizer synccheck clean).
            // kSepP: S(j) is issued before P V(j-1), so that wait moves to just before O
            // or the P region is first touched in this step (o_wait below).
            if (!kSepP && j > 0) mbar_wait<VATTN_SLEEP_MATH>(o_done + t, (gj - 1) & 1);
            tc_fence_after();
            bool o_waited = !kSepP || j == 0;
            auto o_wait = [&] {
                if (!o_waited) {
                    mbar_wait<VATTN_SLEEP_MATH>(o_done + t, (gj - 1) & 1);
                    tc_fence_after();
                    o_waited = true;
                }
            };
            stress_delay(1, j);
            if ((warp & 3) == 0 && lane == 0 && c == 0) VTRACE(1024 + 8 * j + 4 * t + 0);
            // this row's keep bits of key tile j landed during the previous step; fetch j + 1
            // (the mask streams from HBM: its latency stays off the softmax)
            if constexpr (kMaskBits) {
                cp_async_wait_all();
                if (j + 1 < ntile) mask_fetch(j + 1, (gj + 1) & 1);
            }
            float s[kC];
#pragma unroll
            for (int x = 0; x < kC / 32; ++x) tmem_ld32f(tS + 32 * x, s + 32 * x);
            tmem_wait_ld();
            if constexpr (kSepP) {  // S_t(j) is in registers: the MMA may overwrite it with S_t(j+1)
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(s_free + t);
            }
            if ((warp & 3) == 0 && lane == 0 && c == 0) VTRACE(2048 + 8 * j + 4 * t + 0);
            // (tile-uniform) masking: causal diagonal tile (keys > row) or keys beyond N
            const bool tile_masked = p.causal ? (j == ntile - 1) : (j == p.n_kv - 1 && (N & 127) != 0);
            int lim = 127;
            if (p.causal && j == ntile - 1) lim = r;  // diagonal: j*128 == tile row base
            if (!p.causal && j == p.n_kv - 1) lim = min(lim, N - j * 128 - 1);
            if (tile_masked) {
#pragma unroll
                for (int x = 0; x < kC; ++x)
                    if (kC * c + x > lim) s[x] = -INFINITY;
            }
            // P of one 32-key quarter (16 packed columns) with offset mu (log2 units)
            float2 ls2[2] = {make_float2(0.0f, 0.0f), make_float2(0.0f, 0.0f)};  // row-sum partials
            auto quarter = [&](int qi, uint32_t (&pk)[16], auto poly_pair, float mu) {
                const int qq = kQ * c + qi;  // quarter of the tile row
                const float2 sc2 = make_float2(sc, sc);
                const float2 nm2 = make_float2(-mu, -mu);
                uint32_t kw = 0;
                if constexpr (kMaskBits) kw = lds_u32(mslot + (gj & 1) * Cfg::kMaskBuf + 4u * qq);
                if constexpr (kDropMode == 2) {  // no pre-hashed bits: hash this quarter's 32 keys here
                    // (the row's hash prefix is rebuilt per quarter rather than held in four
                    // registers across the tile loop)
                    const DropRow drow = drop_row(drop_bh_base(p.drop_seed, (bh + p.bh_off) / p.H, (bh + p.bh_off) % p.H), row);
                    kw = 0;
#pragma unroll 1
                    for (int b = 0; b < 32; ++b)
                        kw |= static_cast<uint32_t>(drop_keep(drow, j * 128 + 32 * qq + b, p.drop_thresh)) << b;
                }
                uint32_t ks[8];
#pragma unroll
                for (int sh = 0; sh < 8; ++sh) ks[sh] = kw << sh;
                const float2 inv2 = make_float2(p.inv_keep, p.inv_keep);
#pragma unroll
                for (int x = 0; x < 16; ++x) {
                    const int e = 32 * qi + 2 * x;
                    const float2 v = ffma2(make_float2(s[e], s[e + 1]), sc2, nm2);
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
                        // (attention_forward.cpp:94-106); dropped lanes masked to +0
                        const float2 f = fmul2(unpack2<kBF16>(pk[x]), inv2);
                        pk[x] = pack2<kBF16>(f.x, f.y) & keep_mask16(ks, x);
                    }
                }
                (void)kw;
            };
            constexpr int kPer = PolyPeriod<kD>::fwd;
            auto poly_fast = [](int pair) {
                if constexpr (kPer > 0) return pair % kPer == kPer - 1;
                return false;
            };
            auto poly_none = [](int) { return false; };  // -inf -> exact 0 on masked tiles
            auto quarter0 = [&](uint32_t (&pk)[16], float mu) {
                if (kMaskedMufu && tile_masked)
                    quarter(0, pk, poly_none, mu);
                else
                    quarter(0, pk, poly_fast, mu);
            };
            uint32_t pa[16], pb[16];
            // Speculative first quarter (j > 0): exponentiated with the running max while the
            // row max is still being reduced (the two are independent instruction streams);
            // a row whose max then grows by more than 2^8 (lazy rescale below) redoes it.
            // Bitwise identical to computing the max first.
            const bool spec = kSpecMax && j > 0;
            const float m_spec = m_run == -INFINITY ? 0.0f : m_run;
            if (spec) quarter0(pa, m_spec);
            // row max: tree of 3-input maxima, then (two halves) the other half's through smem
            float mx = row_max<kC>(s);
            if constexpr (kH == 2) {
                xslot(gj & 1, c)[r] = mx;
                named_bar_sync(xbar, 256);  // also: every S column of the tile is in registers
                mx = fmax_nr(mx, xslot(gj & 1, c ^ 1)[r]);
            }
            bad |= !(mx < INFINITY);
            const float m_tile = mx * sc;
            if ((warp & 3) == 0 && lane == 0 && c == 0) VTRACE(2048 + 8 * j + 4 * t + 1);
            if (j == 0) {
                m_run = m_tile;
            } else if (__any_sync(0xffffffffu, m_tile > m_run + 8.0f)) {
                // Lazy rescale (warp-uniform: tcgen05.ld/st are .sync.aligned; both halves of
                // a row see the same maxima, so they take the same branch).  The previous
                // P V must have landed before O is touched.  Rows whose max did not grow
                // enough keep their stale max (factor 1).
                float f = 1.0f;
                if (m_tile > m_run) {
                    f = ex2(m_run - m_tile);
                    m_run = m_tile;
                }
                l_run *= f;
                o_wait();
#pragma unroll kRescaleUnroll
                for (int x = 0; x < kOC / 32; ++x) {
                    uint32_t u[32];
                    tmem_ld32(tO + 32 * x, u);
                    tmem_wait_ld();
#pragma unroll
                    for (int y = 0; y < 32; ++y) u[y] = __float_as_uint(__uint_as_float(u[y]) * f);
                    tmem_st32(tO + 32 * x, u);
                }
            }
            const float m_use = m_run == -INFINITY ? 0.0f : m_run;
            if ((warp & 3) == 0 && lane == 0 && c == 0) VTRACE(2048 + 8 * j + 4 * t + 2);
            if (!spec || m_use != m_spec) {  // (per row: only rescaled rows redo)
                ls2[0] = ls2[1] = make_float2(0.0f, 0.0f);
                quarter0(pa, m_use);
            }
            auto publish = [&](int qi) {  // quarter qi's tcgen05.st has been waited on
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(p_full + 4 * t + kQ * c + qi);
                if ((warp & 3) == 0 && lane == 0 && c == 0) VTRACE((qi < 3 ? 1024 + 1 + qi : 2048 + 3) + 8 * j + 4 * t);
            };
            // The tensor-memory store of one quarter completes (wait::st) while the next is
            // computed; the MMA warp starts P V on a quarter as soon as it lands.
            auto emit_rest = [&](auto poly_pair) {
                o_wait();  // (kSepP) P V(j-1) has read the P region
                tmem_st16(tP + 0, pa);
#pragma unroll
                for (int qi = 1; qi < kQ; ++qi) {
                    quarter(qi, (qi & 1) ? pb : pa, poly_pair, m_use);
                    tmem_wait_st();
                    publish(qi - 1);
                    tmem_st16(tP + 16 * qi, (qi & 1) ? pb : pa);
                }
                tmem_wait_st();
                publish(kQ - 1);
            };
            if (kMaskedMufu && tile_masked)  // warp-uniform: tcgen05.st is .sync.aligned
                emit_rest(poly_none);
            else
                emit_rest(poly_fast);
            const float2 lsum = fadd2(ls2[0], ls2[1]);
            l_run += lsum.x + lsum.y;
        }
        if (ntile > 0) {
            // ------------------------------------------------------ epilogue
            mbar_wait<VATTN_SLEEP_MATH>(o_done + t, (ts + ntile - 1) & 1);
            tc_fence_after();
            float l_tot = l_run;
            if constexpr (kH == 2) {  // the row sum over both halves
                xslot(2, c)[r] = l_run;
                named_bar_sync(xbar, 256);
                l_tot += xslot(2, c ^ 1)[r];
            }
            const float inv_l = l_tot > 0.0f ? 1.0f / l_tot : 0.0f;
            if (row < N) {
                const float m_use = m_run == -INFINITY ? 0.0f : m_run;
                if (c == 0) p.lse[static_cast<size_t>(bh) * N + row] = (m_use + lg2(l_tot)) * 0.69314718055994530942f;
                if (p.status && (bad || !(l_tot > 0.0f))) atomicOr(p.status, 1u);
            }
            uint8_t* sO = sQ + t * Cfg::kTileBytes;  // Q_t is dead once the last S_t landed
#pragma unroll kRescaleUnroll
            for (int x = 0; x < kOC / 32; ++x) {
                uint32_t u[32];
                tmem_ld32(tO + 32 * x, u);
                tmem_wait_ld();
#pragma unroll
                for (int y = 0; y < 4; ++y) {
                    uint4 v;
                    v.x = pack2<kBF16>(__uint_as_float(u[8 * y + 0]) * inv_l, __uint_as_float(u[8 * y + 1]) * inv_l);
                    v.y = pack2<kBF16>(__uint_as_float(u[8 * y + 2]) * inv_l, __uint_as_float(u[8 * y + 3]) * inv_l);
                    v.z = pack2<kBF16>(__uint_as_float(u[8 * y + 4]) * inv_l, __uint_as_float(u[8 * y + 5]) * inv_l);
                    v.w = pack2<kBF16>(__uint_as_float(u[8 * y + 6]) * inv_l, __uint_as_float(u[8 * y + 7]) * inv_l);
                    const int col = kOC * c + 32 * x + 8 * y;  // first of 8 columns
                    st_swz128(sO + (col >> 6) * 16384, r, (col & 63) >> 3, v);
                }
            }
            fence_proxy_async_smem();
            named_bar_sync(xbar, 128 * kH);
            if (warp == Cfg::kMathWarp0 + 4 * kH * t && lane == 0) {
                for (int b = 0; b < Cfg::kBoxes; ++b)
                    tma_store_3d(&tm_o, sO + b * 16384, b * 64, q0 + 128 * t, bh);
                bulk_commit();
                bulk_wait_read0();
            }
        }
        // persistent hand-offs (also for a tile with no rows in this item): O_t has been
        // read out of tensor memory, and this tile's O store has left sQ
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(o_free + t);
        if (warp == Cfg::kMathWarp0 + 4 * kH * t && lane == 0) mbar_arrive(q_free);
        ts += ntile;
        }  // items
    }
    if (!kPdlEarly) griddep_launch_dependents();
    tc_fence_before();
    __syncthreads();
    if (warp == Cfg::kAllocWarp) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
    VCTA(0, 1);
}

}  // namespace vattn_sm100
