// capi.cu -- the C ABI (include/vattn_b200.h) over the sm_100a kernels.
//
// Host-side responsibilities: validate the config the way AttnConfig::validate
// does (reference proj/src/attention_forward.cpp:31-40, plus the B200 limits),
// build TMA descriptors for the [B*H, N, d] tensors, size/carve the backward
// workspace, and launch.  There is no CPU or library fallback anywhere.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <atomic>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "../../include/vattn_b200.h"
#include "mha_bwd_sm100.cuh"
#include "mha_fwd_sm100.cuh"
#include "dropout_digest.cuh"

using namespace vattn_sm100;

namespace {

thread_local std::string g_err;
thread_local cudaError_t g_launch_err = cudaSuccess;
thread_local int g_launches = 0;

// ---- measurement hooks (vattn_profile_*): event pairs around the hot kernels
struct ProfPair {
    cudaEvent_t a, b;
    int kind;  // VATTN_KERNEL_* (include/vattn_b200.h)
};
std::mutex g_prof_mu;
bool g_prof_on = false;
std::vector<ProfPair> g_prof;

struct ProfScope {
    cudaStream_t s;
    int kind;
    cudaEvent_t a = nullptr, b = nullptr;
    ProfScope(cudaStream_t s_, int kind_) : s(s_), kind(kind_) {
        bool on;
        {
            std::lock_guard<std::mutex> l(g_prof_mu);
            on = g_prof_on;
        }
        if (!on) return;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a, s);
    }
    ~ProfScope() {
        if (!a) return;
        cudaEventRecord(b, s);
        std::lock_guard<std::mutex> l(g_prof_mu);
        g_prof.push_back({a, b, kind});
    }
};

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
    static EncodeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(ptr);
    });
    return fn;
}

// Encoded tensor maps, cached per (kind, pointer, shape, dtype): a map is
// a pure function of those values, so a hit is exact even when the memory behind the
// pointer was freed and reallocated.  Encoding costs ~1-2 us of host time per map and
// a call needs 4-6 of them, which matters for launch-bound configs (C1, C4).
// Direct-mapped, 256 entries, one mutex (lookups are ~100 ns).
struct MapKey {
    int kind;  // 0 = [BH, N, d] operand, 1 = dS^T scratch, 2 = operand in 64-row boxes
    const void* ptr;
    long long a, b, c;
    bool bf16;
    bool operator==(const MapKey& o) const {
        return kind == o.kind && ptr == o.ptr && a == o.a && b == o.b && c == o.c && bf16 == o.bf16;
    }
};
struct MapCache {
    static constexpr int kSlots = 256;
    std::mutex mu;
    MapKey key[kSlots];
    CUtensorMap map[kSlots];
    bool used[kSlots] = {};
    static size_t slot(const MapKey& k) {
        // tensors of one call sit at multiples of their (large, power-of-two-ish) size:
        // mix every address bit into the slot (murmur3 finaliser)
        uint64_t h = reinterpret_cast<uintptr_t>(k.ptr);
        h ^= static_cast<uint64_t>(k.a) * 0x9E3779B97F4A7C15ull + static_cast<uint64_t>(k.b) * 0xC2B2AE3D27D4EB4Full +
             static_cast<uint64_t>(k.c) * 0x165667B19E3779F9ull + static_cast<uint64_t>(k.kind * 2 + k.bf16);
        h ^= h >> 33;
        h *= 0xff51afd7ed558ccdull;
        h ^= h >> 33;
        h *= 0xc4ceb9fe1a85ec53ull;
        h ^= h >> 33;
        return static_cast<size_t>(h % kSlots);
    }
    bool get(const MapKey& k, CUtensorMap* out) {
        std::lock_guard<std::mutex> l(mu);
        const size_t s = slot(k);
        if (!used[s] || !(key[s] == k)) return false;
        *out = map[s];
        return true;
    }
    void put(const MapKey& k, const CUtensorMap& m) {
        std::lock_guard<std::mutex> l(mu);
        const size_t s = slot(k);
        key[s] = k;
        map[s] = m;
        used[s] = true;
    }
};
MapCache g_maps;
std::atomic<long long> g_map_hits{0}, g_map_misses{0};

// [B*H, N, d] 16-bit tensor, `rows` (128, or 64 for the CTA pair's half tiles) x 64
// columns per box, 128-byte swizzle.
bool encode_map(CUtensorMap* m, const void* ptr, int BH, int N, int D, bool bf16, int rows = 128) {
    EncodeFn enc = encode_fn();
    if (!enc) {
        g_err = "cuTensorMapEncodeTiled: driver entry point unavailable";
        return false;
    }
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(D), static_cast<cuuint64_t>(N),
                                static_cast<cuuint64_t>(BH)};
    const cuuint64_t strides[2] = {static_cast<cuuint64_t>(D) * 2,
                                   static_cast<cuuint64_t>(D) * 2 * static_cast<cuuint64_t>(N)};
    const cuuint32_t box[3] = {64, static_cast<cuuint32_t>(rows), 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    auto encode = [&] {
        return enc(m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3,
                   const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    };
    CUresult r = encode();
    if (r == CUDA_ERROR_INVALID_CONTEXT) {
        // a host thread that never made the device's primary context current (e.g. the
        // torch autograd engine's worker thread): the driver call needs one.  Any runtime
        // call binds it; retry once.
        cudaFree(nullptr);
        r = encode();
    }
    if (r != CUDA_SUCCESS) {
        char buf[160];
        snprintf(buf, sizeof(buf), "cuTensorMapEncodeTiled failed (CUresult %d, ptr %p, [%d, %d, %d])", static_cast<int>(r),
                 ptr, BH, N, D);
        g_err = buf;
    }
    return r == CUDA_SUCCESS;
}

bool make_map(CUtensorMap* m, const void* ptr, int BH, int N, int D, bool bf16, int rows = 128) {
    const MapKey k{rows == 128 ? 0 : 2, ptr, BH, N, D, bf16};
    if (g_maps.get(k, m)) {
        g_map_hits.fetch_add(1, std::memory_order_relaxed);
        return true;
    }
    g_map_misses.fetch_add(1, std::memory_order_relaxed);
    if (!encode_map(m, ptr, BH, N, D, bf16, rows)) return false;
    g_maps.put(k, *m);
    return true;
}

// dS^T scratch viewed as [tiles][128 keys][128 queries] 16-bit, 64-query x `rows`-key
// boxes (128: the dQ GEMM's loads; 32: the dK/dV kernel's per-warp stores).
bool encode_ds_map(CUtensorMap* m, const void* ptr, long long tiles, bool bf16, int rows = 128) {
    EncodeFn enc = encode_fn();
    if (!enc || tiles > (1ll << 31) - 1) return false;
    const cuuint64_t dims[3] = {128, 128, static_cast<cuuint64_t>(tiles)};
    const cuuint64_t strides[2] = {256, 32768};
    const cuuint32_t box[3] = {64, static_cast<cuuint32_t>(rows), 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    auto encode = [&] {
        return enc(m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3,
                   const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    };
    CUresult r = encode();
    if (r == CUDA_ERROR_INVALID_CONTEXT) {  // see encode_map
        cudaFree(nullptr);
        r = encode();
    }
    return r == CUDA_SUCCESS;
}

bool make_ds_map(CUtensorMap* m, const void* ptr, long long tiles, bool bf16, int rows = 128) {
    const MapKey k{rows == 128 ? 1 : 3, ptr, tiles, 0, 0, bf16};
    if (g_maps.get(k, m)) {
        g_map_hits.fetch_add(1, std::memory_order_relaxed);
        return true;
    }
    g_map_misses.fetch_add(1, std::memory_order_relaxed);
    if (!encode_ds_map(m, ptr, tiles, bf16, rows)) return false;
    g_maps.put(k, *m);
    return true;
}

// sm_100 check, cached per device.
int check_device() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return fail(VATTN_ECUDA, "no CUDA device");
    static int cached[64];
    static std::once_flag flags[64];
    if (dev < 0 || dev >= 64) return fail(VATTN_ECUDA, "device index out of range");
    std::call_once(flags[dev], [dev] {
        int major = 0, minor = 0;
        cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
        cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
        cached[dev] = major * 10 + minor;
    });
    if (cached[dev] != 100)
        return fail(VATTN_ECUDA, "vattn_b200 kernels are built for sm_100a (B200); device is sm_" +
                                     std::to_string(cached[dev]));
    return VATTN_OK;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int validate(const vattn_config* c) {
    if (!c) return fail(VATTN_EINVAL, "vattn_config: null");
    if (c->batch < 1 || c->heads < 1)
        return fail(VATTN_EINVAL, "AttnConfig: batch and heads must be positive");
    if (c->seq_len < 1 || c->head_dim < 1)
        return fail(VATTN_EINVAL, "AttnConfig: seq_len and head_dim must be positive");
    if (c->dtype != VATTN_F16 && c->dtype != VATTN_BF16)
        return fail(VATTN_EINVAL, "vattn_config: dtype must be VATTN_F16 or VATTN_BF16");
    if (c->causal != 0 && c->causal != 1) return fail(VATTN_EINVAL, "vattn_config: causal must be 0/1");
    if (!std::isfinite(c->softmax_scale)) return fail(VATTN_EINVAL, "vattn_config: softmax_scale not finite");
    if (!(c->dropout_p >= 0.0f && c->dropout_p < 1.0f))
        return fail(VATTN_EINVAL, "AttnConfig: dropout_p must be in [0, 1)");
    if (c->head_dim != 64 && c->head_dim != 128)
        return fail(VATTN_EUNSUPPORTED, "head_dim must be 64 or 128 at the C ABI (pad in the caller)");
    const long long bh_all = static_cast<long long>(c->batch) * c->heads;
    if (c->bh_count < 0 || c->bh_offset < 0)
        return fail(VATTN_EINVAL, "vattn_config: bh_offset / bh_count must be >= 0");
    if (c->bh_count == 0 && c->bh_offset != 0)
        return fail(VATTN_EINVAL, "vattn_config: bh_offset without bh_count");
    if (static_cast<long long>(c->bh_offset) + c->bh_count > bh_all)
        return fail(VATTN_EINVAL, "vattn_config: (b, h) slab [bh_offset, bh_offset + bh_count) exceeds batch * heads");
    const long long bh = c->bh_count ? c->bh_count : bh_all;
    if (bh > 65535) return fail(VATTN_EUNSUPPORTED, "batch * heads (per call) must be <= 65535");
    if (bh * c->seq_len > (1ll << 31) - 1)
        return fail(VATTN_EUNSUPPORTED, "batch * heads * seq_len must fit in int32");
    return VATTN_OK;
}

// (b, h) units this call runs (the slab, or the whole problem).
int units(const vattn_config* c) { return c->bh_count ? c->bh_count : c->batch * c->heads; }

float eff_scale(const vattn_config* c) {
    // AttnConfig::scale(), proj/src/attention_forward.cpp:42-45
    return c->softmax_scale > 0.0f ? c->softmax_scale
                                   : 1.0f / std::sqrt(static_cast<float>(c->head_dim));
}

constexpr float kLog2e = 1.4426950408889634f;

// Dropout constants: keep iff bits_to_unit(hash) >= p  <=>  (hash >> 11) >= ceil(p * 2^53)
// (exact: bits_to_unit is (hash >> 11) * 2^-53 in binary64, rng.cpp:19-21, 46-49).
void set_dropout(const vattn_config* c, int* H, int* bh_off, float* inv_keep, uint64_t* seed, uint64_t* thresh) {
    *H = c->heads;
    *bh_off = c->bh_offset;
    *inv_keep = 1.0f / (1.0f - c->dropout_p);  // binary32, attention_forward.cpp:83 / attention_backward.cpp:81
    *seed = c->seed;
    *thresh = static_cast<uint64_t>(std::ceil(static_cast<double>(c->dropout_p) * 9007199254740992.0));
}

// (b,h) units per dispatch group (see grid_bh): the largest divisor of BH whose
// shared per-unit streams fit the kernel's L2 budget.  Causal forward: 64 MB (the
// longest query blocks of a group start first, so the per-SM tail shrinks from ~70 us
// to ~5 us at C3: +3 % standalone, +12 % at B = 2); non-causal items are all the same
// length, so the forward stays unit-major there (grouping measured -2..4 %).  Backward: unit-major (G = 1): every
// key tile of one unit reads the same Q/dO stream at once, which groups only dilute
// (measured: dK/dV CTAs 3 % slower, dQ GEMM 10 % slower, tails shrink but spans do not).
// Tuning overrides: VATTN_L2_GROUP_MB_FWD / VATTN_L2_GROUP_MB_BWD (0 = unit-major).
int bh_group(int BH, long long per_unit_bytes, bool fwd) {
    static const long long budget_f = [] {
        const char* e = getenv("VATTN_L2_GROUP_MB_FWD");
        return (e ? atoll(e) : 64ll) << 20;
    }();
    static const long long budget_b = [] {
        const char* e = getenv("VATTN_L2_GROUP_MB_BWD");
        return (e ? atoll(e) : 0ll) << 20;
    }();
    const long long budget = fwd ? budget_f : budget_b;
    int G = 1;
    for (int g = 1; g <= BH; ++g)
        if (BH % g == 0 && static_cast<long long>(g) * per_unit_bytes <= budget) G = g;
    return G;
}

// dK/dV dispatch (grid_item_tail): causal key tiles differ in length up to n_q-fold,
// so the units of the last ~3.5 waves go longest-first (their heaviest tiles would
// otherwise start in the final wave and leave a ~60 us per-SM tail at C3).  The rest
// stays unit-major: all key tiles of one unit share its Q/dO stream in L2 (a fully
// grouped order measured 3 % slower per CTA).  VATTN_DKDV_TAIL_WAVES overrides (0 = off).
// SM count of the current device (cached per device; racing writers store the same value).
int sm_count_cached() {
    static std::atomic<int> sm_count[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
    int sms = sm_count[dev].load(std::memory_order_relaxed);
    if (!sms) {
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = 148;
        sm_count[dev].store(sms, std::memory_order_relaxed);
    }
    return sms;
}

int dkdv_tail_units(int BH, int n_q, int ctas_per_item = 1) {
    static const double waves = [] {
        const char* e = getenv("VATTN_DKDV_TAIL_WAVES");
        return e ? atof(e) : 3.5;
    }();
    const int sms = sm_count_cached();
    const int T = static_cast<int>((waves * (sms / ctas_per_item) + n_q - 1) / n_q);
    return T < 0 ? 0 : (T > BH ? BH : T);
}

int current_device() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
    return dev;
}

// One cudaFuncSetAttribute per (kernel instantiation, device): function attributes
// are per-context state, so a process that drives several GPUs opts in on each.
// Keyed on the kernel itself (different instantiations share a function-pointer type).
template <auto kKernel>
cudaError_t set_smem_once(int bytes) {
    static std::once_flag once[64];
    static cudaError_t err[64];
    const int dev = current_device();
    std::call_once(once[dev], [&] { err[dev] = cudaFuncSetAttribute(kKernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes); });
    return err[dev];
}

// Launch with programmatic stream serialisation (see griddep_* in sm100_ptx.cuh):
// the kernel's CTAs may start their prologue while the previous kernel drains.
template <typename... Params, typename... Args>
cudaError_t launch_pdl(void (*kernel)(Params...), dim3 grid, dim3 block, int smem, cudaStream_t stream,
                       Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = static_cast<size_t>(smem);
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
    if (e != cudaSuccess) g_launch_err = e;  // reported by the call's final error check
    return e;
}
// The same with (2,1,1) clusters (CTA pairs: cta_group::2 kernels).
template <typename... Params, typename... Args>
cudaError_t launch_pdl_pair(void (*kernel)(Params...), dim3 grid, dim3 block, int smem, cudaStream_t stream,
                            Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = static_cast<size_t>(smem);
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = 2;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
    if (e != cudaSuccess) g_launch_err = e;
    return e;
}


// Both keep-bit copies of `c` (query-major, then key-major; mha_dropmask_kernel).
void launch_dropmask(const vattn_config* c, uint32_t* mask, cudaStream_t stream) {
    int H, bh_off;
    float inv_keep;
    uint64_t seed, thresh;
    set_dropout(c, &H, &bh_off, &inv_keep, &seed, &thresh);
    const int nt = (c->seq_len + 127) / 128;
    const unsigned pairs = c->causal ? static_cast<unsigned>(nt) * (nt + 1) / 2 : static_cast<unsigned>(nt) * nt;
    ProfScope prof(stream, 4);
    launch_pdl(mha_dropmask_kernel, dim3(pairs, static_cast<unsigned>(units(c))), dim3(256), 0, stream, mask, nt * 128,
               H, bh_off, seed, thresh, c->causal);
}

template <int kD, bool kBF16, bool kDrop>
int launch_forward(const vattn_config* c, const void* q, const void* k, const void* v, void* o,
                   float* lse, uint32_t* drop_mask, unsigned int* status, cudaStream_t stream) {
    const int BH = units(c), N = c->seq_len;
    CUtensorMap mq, mk, mv, mo;
    if (!make_map(&mq, q, BH, N, kD, kBF16) || !make_map(&mk, k, BH, N, kD, kBF16) ||
        !make_map(&mv, v, BH, N, kD, kBF16) || !make_map(&mo, o, BH, N, kD, kBF16))
        return fail(VATTN_ECUDA, g_err.empty() ? "cuTensorMapEncodeTiled failed" : g_err);
    constexpr int smem = FwdCfg<kD>::kSmemBytes;
    FwdParams p;
    p.lse = lse;
    p.N = N;
    p.n_kv = (N + 127) / 128;
    p.causal = c->causal;
    p.scale_log2 = eff_scale(c) * kLog2e;
    set_dropout(c, &p.H, &p.bh_off, &p.inv_keep, &p.drop_seed, &p.drop_thresh);
    p.drop_mask = drop_mask;
    p.mask_words = (N + 127) / 128 * 4;
    p.status = status;
    if (kDrop && drop_mask) launch_dropmask(c, drop_mask, stream);
    const int nqb = (N + 255) / 256;
    p.group = c->causal ? bh_group(BH, 2ll * N * kD * 2, true) : 1;  // K, V
    p.items = nqb * BH;
    // Persistent forward (one CTA per SM looping over the (unit, query block) items in
    // the same order, static round robin) for short heads, N <= 1024 -- the same rule and
    // reason as the dK/dV kernel; VATTN_FWD_PERSIST=0 / 1 forces either.
    static const int fwd_persist_env = [] {
        const char* e = getenv("VATTN_FWD_PERSIST");
        return e ? atoi(e) : -1;
    }();
    const int sms = sm_count_cached();
    // (the in-softmax hash variant, dropout without a mask buffer, is one-item-per-CTA only)
    const bool persist = (fwd_persist_env >= 0 ? fwd_persist_env == 1 : N <= 1024) && p.items > sms && !(kDrop && !drop_mask);
    p.stride = persist ? sms : p.items;
    const dim3 grid = persist ? dim3(static_cast<unsigned>(sms)) : tile_grid(nqb, BH, p.group);
    {
        ProfScope prof(stream, 0);
        constexpr int kMode = kDrop ? 1 : 0;  // dropout with a mask buffer / none
        if (kDrop && !drop_mask) {
            const cudaError_t attr_err = set_smem_once<mha_fwd_sm100_kernel<kD, kBF16, 2, false>>(smem);
            if (attr_err != cudaSuccess) return fail(VATTN_ECUDA, cudaGetErrorString(attr_err));
            launch_pdl(mha_fwd_sm100_kernel<kD, kBF16, 2, false>, grid, dim3(FwdCfg<kD>::kThreads), smem, stream, mq, mk, mv,
                       mo, p);
        } else {
            const cudaError_t attr_err = persist ? set_smem_once<mha_fwd_sm100_kernel<kD, kBF16, kMode, true>>(smem)
                                                 : set_smem_once<mha_fwd_sm100_kernel<kD, kBF16, kMode, false>>(smem);
            if (attr_err != cudaSuccess) return fail(VATTN_ECUDA, cudaGetErrorString(attr_err));
            if (persist)
                launch_pdl(mha_fwd_sm100_kernel<kD, kBF16, kMode, true>, grid, dim3(FwdCfg<kD>::kThreads), smem, stream, mq, mk,
                           mv, mo, p);
            else
                launch_pdl(mha_fwd_sm100_kernel<kD, kBF16, kMode, false>, grid, dim3(FwdCfg<kD>::kThreads), smem, stream, mq, mk,
                           mv, mo, p);
        }
    }
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = g_launch_err;
    g_launch_err = cudaSuccess;
    if (e != cudaSuccess) return fail(VATTN_ECUDA, std::string("mha_fwd launch: ") + cudaGetErrorString(e));
    g_launches = (kDrop && drop_mask) ? 2 : 1;
    return VATTN_OK;
}

struct BwdLayout {
    size_t lse2, dsum, ds, sync, mask, total;
    bool drop_mask;          // dropout keep bits hashed once into the workspace
    int n_q, Npad;
    bool materialize_ds;     // dQ as a GEMM over materialised dS (else recompute S, dP)
    long long ds_tiles_per_bh;
};

// dS materialisation costs 32 KiB of workspace per (query tile, key tile) pair
// (C3: 4.4 GB of a B200's 180 GB).  It is used at d = 128 while that stays under 40 %
// of the device's TOTAL memory (a property of the device, so the workspace size query
// and the launch always agree): C5 on one GPU needs 69 GB and is 8 % faster with it
// (57.8 vs 62.6 ms); on 8 GPUs each shard needs 8.6 GB.  VATTN_DQ_MODE=0/1 forces a
// mode (tuning and tests).
size_t ds_cap_bytes() {
    static std::atomic<size_t> cap[64] = {};  // per device; racing writers store the same value
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
    size_t c = cap[dev].load(std::memory_order_relaxed);
    if (!c) {
        size_t free_b = 0, total_b = 0;
        c = cudaMemGetInfo(&free_b, &total_b) == cudaSuccess ? total_b / 5 * 2 : (32ull << 30);
        cap[dev].store(c, std::memory_order_relaxed);
    }
    return c;
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// VATTN_DROP_MASK=0: no keep-bit masks at all (both backward kernels hash in place).
bool drop_mask_enabled() {
    static const bool on = [] {
        const char* e = getenv("VATTN_DROP_MASK");
        return !(e && atoi(e) == 0);
    }();
    return on;
}

BwdLayout bwd_layout(const vattn_config* c) {
    BwdLayout L{};
    const size_t BH = static_cast<size_t>(units(c));
    L.n_q = (c->seq_len + 127) / 128;
    L.Npad = L.n_q * 128;
    L.lse2 = 0;
    L.dsum = align256(BH * L.Npad * 4);
    L.ds = L.dsum + align256(BH * L.Npad * 4);
    const long long nq = L.n_q;
    L.ds_tiles_per_bh = c->causal ? nq * (nq + 1) / 2 : nq * nq;
    const size_t ds_bytes = BH * static_cast<size_t>(L.ds_tiles_per_bh) * 32768;
    static const int mode_env = [] {
        const char* e = getenv("VATTN_DQ_MODE");
        return e ? atoi(e) : -1;
    }();
    // (the dK/dV kernel's dS^T staging overlaps its dropout row-hash buffer, used only
    // when the keep bits are hashed in place)
    // d = 64 materialises only for N <= 1024: there the recompute kernel's short
    // per-CTA loops dominate (N = 512 / 1024: +8 % / +6 %, causal or not); at long N
    // the shorter dK/dV iterations pay more for the staging than the dQ GEMM saves
    // (N = 4k / 8k / 16k: -5 / -4 / -7 %).  d = 128: C3 +8 %.
    // Dropout: both backward kernels read the keep bits from a query-major bit mask
    // (BH * Npad^2 / 8 bytes) -- the forward's own (mha_forward_dropout_mask) or one
    // hashed here once -- instead of hashing every position twice.  That also frees the
    // dK/dV kernel's row-hash buffer for the dS^T staging box, so dropout takes the dQ
    // GEMM path.  VATTN_DROP_MASK=0: hash in place (and recompute dQ).
    const bool mask_env = drop_mask_enabled();
    const size_t mask_bytes = 2 * BH * static_cast<size_t>(L.Npad) * (L.Npad / 8);  // query- + key-major
    L.drop_mask = c->dropout_p > 0.0f && mask_env;
    L.materialize_ds = c->dropout_p > 0.0f && !L.drop_mask
                           ? false
                           : (mode_env >= 0 ? mode_env == 1 : ((c->head_dim == 128 || c->seq_len <= 1024) && ds_bytes <= ds_cap_bytes()));
    L.sync = L.ds + (L.materialize_ds ? align256(ds_bytes) : 0);  // dQ hand-off words (BwdParams::dq_sync)
    L.mask = L.sync + (L.materialize_ds ? align256((2 + BH) * sizeof(int)) : 0);
    L.total = L.mask + (L.drop_mask ? align256(mask_bytes) : 0);
    return L;
}

template <int kD, bool kBF16, bool kDrop>
int launch_backward(const vattn_config* c, const void* q, const void* k, const void* v,
                    const void* o, const void* dout, const float* lse, void* dq, void* dk,
                    void* dv, void* ws, const uint32_t* ext_mask, cudaStream_t stream) {
    const int BH = units(c), N = c->seq_len;
    const BwdLayout L = bwd_layout(c);
    uint8_t* w = static_cast<uint8_t*>(ws);
    float* lse2 = reinterpret_cast<float*>(w + L.lse2);
    float* dsum = reinterpret_cast<float*>(w + L.dsum);

    CUtensorMap mq, mk, mv, mdo, mdq;
    if (!make_map(&mq, q, BH, N, kD, kBF16) || !make_map(&mk, k, BH, N, kD, kBF16) ||
        !make_map(&mv, v, BH, N, kD, kBF16) || !make_map(&mdo, dout, BH, N, kD, kBF16) ||
        !make_map(&mdq, dq, BH, N, kD, kBF16))
        return fail(VATTN_ECUDA, g_err.empty() ? "cuTensorMapEncodeTiled failed" : g_err);

    // 1) D = rowsum(dO o O), lse2 = lse * log2(e)
    {
        const long long rows = static_cast<long long>(BH) * L.Npad;
        // one wave (8 x 256-thread blocks per SM), each warp 4 x (32 / (d / 8)) rows per pass
        const long long rows_per_block = 8ll * 4 * (256 / kD);
        long long blocks = (rows + rows_per_block - 1) / rows_per_block;
        if (blocks > 148 * 8) blocks = 148 * 8;
        ProfScope prof(stream, 3);
        launch_pdl(mha_bwd_preprocess_kernel<kD, kBF16>, dim3(static_cast<unsigned>(blocks)), dim3(256), 0, stream,
                   o, dout, lse, lse2, dsum, N, L.Npad, BH, L.materialize_ds ? reinterpret_cast<int*>(w + L.sync) : nullptr,
                   L.materialize_ds ? 2 + BH : 0);
    }
    BwdParams p;
    p.lse2 = lse2;
    p.dsum = dsum;
    p.N = N;
    p.Npad = L.Npad;
    p.n_q = L.n_q;
    p.causal = c->causal;
    p.scale = eff_scale(c);
    p.scale_log2 = p.scale * kLog2e;
    set_dropout(c, &p.H, &p.bh_off, &p.inv_keep, &p.drop_seed, &p.drop_thresh);
    p.ds_out = L.materialize_ds ? reinterpret_cast<uint16_t*>(w + L.ds) : nullptr;
    p.ds_tiles_per_bh = L.ds_tiles_per_bh;
    // d = 128, VATTN_DKDV_PAIR=1: CTA pairs (cta_group::2 M = 256 MMAs, half the B-operand
    // shared-memory reads).  Off by default: measured 1-3 % slower than one CTA per key
    // tile at C3 / C5 (DESIGN 2.2 -- the step is bound by the P pass -> dV -> S chain, which
    // the pair does not shorten, not by shared-memory bandwidth).
    static const bool pair_env = [] {
        const char* e = getenv("VATTN_DKDV_PAIR");
        return e && atoi(e) == 1;
    }();
    const bool pair = kD == 128 && pair_env;
    const int n_pairs = (L.n_q + 1) / 2;
    // VATTN_DQ_WORKERS=W > 0: dQ overlapped with dK/dV (dS materialised, one CTA per key
    // tile): the first W CTAs of the dK/dV grid are persistent dQ workers (mha_bwd_sm100.cuh
    // dq_worker) taking units as their dS^T tiles complete; a full-width tail launch
    // finishes the rest.  Bitwise identical; measured neutral (C3 step 3.87 ms for W = 0,
    // 8, 16, 24: a dQ worker moves ~45 GB/s whether 24 or 148 SMs run it, so the dQ work
    // hidden equals the dK/dV work displaced -- profiles/r2_experiments.md).  Default 0:
    // the separate dQ GEMM launch.
    static const int workers_env = [] {
        const char* e = getenv("VATTN_DQ_WORKERS");
        return e ? atoi(e) : 0;
    }();
    const int sms = sm_count_cached();
    int W = workers_env;
    if (!L.materialize_ds || pair) W = 0;
    if (W > sms / 2) W = sms / 2;
    p.dq_sync = W > 0 ? reinterpret_cast<int*>(w + L.sync) : nullptr;
    p.dq_workers = W;
    p.dkdv_ctas = L.n_q * BH;
    p.n_units = BH;
    p.ds_signals = (kDsWarpStore<kD> ? 4 : 1) * DkdvCfg<kD>::kWG * L.n_q;
    p.dkdv_items = L.n_q * BH;
    // Persistent dK/dV (one CTA per SM looping over the (unit, key tile) items, static
    // round robin; the next item's K / V / Q / dO loads and first S / dP MMAs overlap the
    // current item's epilogue) for short heads, N <= 1024: C2 N = 512 -10 %, N = 1k -7 %,
    // C4 -3.4 % per step.  At long causal N the static assignment loses the longest-first
    // balance of one CTA per item (C3 +7.5 %), so those keep one CTA per item.
    // VATTN_DKDV_PERSIST=0 / 1 forces either.  Not with the overlapped dQ workers, which
    // count finished items per CTA.
    static const int dkdv_persist_env = [] {
        const char* e = getenv("VATTN_DKDV_PERSIST");
        return e ? atoi(e) : -1;
    }();
    const bool dkdv_persist = dkdv_persist_env >= 0 ? dkdv_persist_env == 1 : L.n_q <= 8;
    const int dkdv_ctas = (dkdv_persist && W == 0 && p.dkdv_items > sms) ? sms : p.dkdv_items;
    p.tail_units = c->causal ? (pair ? dkdv_tail_units(BH, n_pairs, 2) : dkdv_tail_units(BH, L.n_q)) : 0;
    p.drop_mask = nullptr;
    p.drop_mask_k = nullptr;
    bool mask_kernel = false;
    if (L.drop_mask) {
        if (ext_mask) {  // the forward's keep bits (mha_forward_dropout_mask)
            p.drop_mask = ext_mask;
        } else {
            uint32_t* m = reinterpret_cast<uint32_t*>(w + L.mask);
            p.drop_mask = m;
            mask_kernel = true;
            launch_dropmask(c, m, stream);
        }
        p.drop_mask_k = p.drop_mask + static_cast<size_t>(BH) * L.Npad * (L.Npad / 32);
    }
    CUtensorMap mds;
    if (L.materialize_ds && !make_ds_map(&mds, p.ds_out, static_cast<long long>(BH) * L.ds_tiles_per_bh, kBF16))
        return fail(VATTN_ECUDA, "cuTensorMapEncodeTiled (dS) failed");
    // per-warp dS^T stores (kDsWarpStore): 32-key boxes, passed in the non-pair kernel's
    // (otherwise unused) 64-row Q map slot
    CUtensorMap mds32 = mq;
    if (kDsWarpStore<kD> && L.materialize_ds &&
        !make_ds_map(&mds32, p.ds_out, static_cast<long long>(BH) * L.ds_tiles_per_bh, kBF16, 32))
        return fail(VATTN_ECUDA, "cuTensorMapEncodeTiled (dS, 32-key boxes) failed");
    // 2) dK, dV (key-major)
    bool dkdv_launched = false;
    if constexpr (kD == 128) {
      if (pair) {
        CUtensorMap mq64, mdo64;
        if (!make_map(&mq64, q, BH, N, kD, kBF16, 64) || !make_map(&mdo64, dout, BH, N, kD, kBF16, 64))
            return fail(VATTN_ECUDA, g_err.empty() ? "cuTensorMapEncodeTiled failed" : g_err);
        auto kern = mha_bwd_dkdv_kernel<kD, kBF16, kDrop, true>;
        constexpr int smem = DkdvCfg<kD>::kSmemBytes;
        const cudaError_t ae = set_smem_once<mha_bwd_dkdv_kernel<kD, kBF16, kDrop, true>>(smem);
        if (ae != cudaSuccess) return fail(VATTN_ECUDA, cudaGetErrorString(ae));
        ProfScope prof(stream, 1);
        launch_pdl_pair(kern, dim3(2 * n_pairs * BH), dim3(DkdvCfg<kD>::kThreads), smem, stream, mq, mk, mv, mdo,
                        L.materialize_ds ? mds : mq, mq64, mdo64, mdq, dk, dv, p);
        dkdv_launched = true;
      }
    }
    if (!dkdv_launched) {
        // (the dQ workers' layout may be the larger one)
        constexpr int smem = DkdvCfg<kD>::kSmemBytes > DqGemmCfg<kD>::kSmemBytes ? DkdvCfg<kD>::kSmemBytes
                                                                                 : DqGemmCfg<kD>::kSmemBytes;
        const bool multi = dkdv_ctas < p.dkdv_items;
        const cudaError_t ae = multi ? set_smem_once<mha_bwd_dkdv_kernel<kD, kBF16, kDrop, false, true>>(smem)
                                     : set_smem_once<mha_bwd_dkdv_kernel<kD, kBF16, kDrop, false, false>>(smem);
        if (ae != cudaSuccess) return fail(VATTN_ECUDA, cudaGetErrorString(ae));
        ProfScope prof(stream, 1);
        if (multi)
            launch_pdl(mha_bwd_dkdv_kernel<kD, kBF16, kDrop, false, true>, dim3(dkdv_ctas + W), dim3(DkdvCfg<kD>::kThreads),
                       smem, stream, mq, mk, mv, mdo, L.materialize_ds ? mds : mq, mds32, mdo, mdq, dk, dv, p);
        else
            launch_pdl(mha_bwd_dkdv_kernel<kD, kBF16, kDrop, false, false>, dim3(dkdv_ctas + W), dim3(DkdvCfg<kD>::kThreads),
                       smem, stream, mq, mk, mv, mdo, L.materialize_ds ? mds : mq, mds32, mdo, mdq, dk, dv, p);
    }
    // 3) dQ (query-major, fixed-order accumulation in TMEM)
    // The dQ GEMM runs as the persistent worker kernel (one CTA per SM looping over the
    // (unit, query tile) items; bitwise the same as one CTA per tile): C2 N = 512 / 1k and
    // C4 steps -3 / -1 / -1 %, C3 neutral.  VATTN_DQ_PERSIST=0: one CTA per query tile.
    static const bool persist_env = [] {
        const char* e = getenv("VATTN_DQ_PERSIST");
        return !(e && atoi(e) == 0);
    }();
    if (W > 0 || (persist_env && L.materialize_ds && !pair)) {  // full width (after the workers, if any)
        auto kern = mha_bwd_dq_tail_kernel<kD, kBF16>;
        constexpr int smem = DqGemmCfg<kD>::kSmemBytes;
        const cudaError_t ae = set_smem_once<mha_bwd_dq_tail_kernel<kD, kBF16>>(smem);
        if (ae != cudaSuccess) return fail(VATTN_ECUDA, cudaGetErrorString(ae));
        ProfScope prof(stream, 2);
        const int items = L.n_q * BH;
        BwdParams pt = p;
        pt.dq_sync = reinterpret_cast<int*>(w + L.sync);  // [0]: the item counter
        launch_pdl(kern, dim3(items < sms ? items : sms), dim3(256), smem, stream, mds, mk, mdq, pt);
    } else if (L.materialize_ds) {
        auto kern = mha_bwd_dq_gemm_kernel<kD, kBF16>;
        constexpr int smem = DqGemmCfg<kD>::kSmemBytes;
        const cudaError_t ae = set_smem_once<mha_bwd_dq_gemm_kernel<kD, kBF16>>(smem);
        if (ae != cudaSuccess) return fail(VATTN_ECUDA, cudaGetErrorString(ae));
        ProfScope prof(stream, 2);
        launch_pdl(kern, dim3(L.n_q * BH), dim3(256), smem, stream, mds, mk, mdq, p);
    } else {
        auto kern = mha_bwd_dq_kernel<kD, kBF16, kDrop>;
        constexpr int smem = DqCfg<kD>::kSmemBytes;
        const cudaError_t ae = set_smem_once<mha_bwd_dq_kernel<kD, kBF16, kDrop>>(smem);
        if (ae != cudaSuccess) return fail(VATTN_ECUDA, cudaGetErrorString(ae));
        ProfScope prof(stream, 2);
        launch_pdl(kern, tile_grid(L.n_q, BH, bh_group(BH, 2ll * N * kD * 2, false)), dim3(384), smem, stream, mq, mk, mv,
                   mdo, mdq, p);  // K, V
    }
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = g_launch_err;
    g_launch_err = cudaSuccess;
    if (e != cudaSuccess) return fail(VATTN_ECUDA, std::string("mha_bwd launch: ") + cudaGetErrorString(e));
    g_launches = mask_kernel ? 4 : 3;
    return VATTN_OK;
}

}  // namespace

extern "C" {

#ifdef VATTN_TRACE
// Debug-only: select the backward work item to trace / read its timeline.
int vattn_trace_select(int kid, int item) {
    cudaMemcpyToSymbol(g_vattn_trace_kid, &kid, sizeof(int));
    cudaMemcpyToSymbol(g_vattn_trace_block, &item, sizeof(int));
    long long z[4096] = {0};
    cudaMemcpyToSymbol(g_vattn_trace, z, sizeof(z));
    return 0;
}
int vattn_cta_read(unsigned long long* out, int n_blocks) {  // [block][start_ns, end_ns, smid]
    static unsigned long long z[16384][3];
    const int n = n_blocks < 16384 ? n_blocks : 16384;
    if (cudaMemcpyFromSymbol(out, g_vattn_cta, sizeof(unsigned long long) * 3 * n) != cudaSuccess) return 1;
    return cudaMemcpyToSymbol(g_vattn_cta, z, sizeof(z)) == cudaSuccess ? 0 : 1;
}
int vattn_trace_read(long long* out, int n) {
    return cudaMemcpyFromSymbol(out, g_vattn_trace, sizeof(long long) * (n < 4096 ? n : 4096)) ==
                   cudaSuccess
               ? 0
               : 1;
}
#endif

int vattn_abi_version(void) { return VATTN_B200_ABI_VERSION; }

const char* vattn_last_error(void) { return g_err.c_str(); }

// internal (capi_host.cu): report a host-pipeline failure through vattn_last_error,
// and validate a config with the device entry points' own rules.
void vattn_set_error_(const char* msg) { g_err = msg ? msg : ""; }
int vattn_validate_(const vattn_config* cfg) { return validate(cfg); }

int vattn_last_launch_count(void) { return g_launches; }

void vattn_map_cache_stats(long long* hits, long long* misses) {
    if (hits) *hits = g_map_hits.load();
    if (misses) *misses = g_map_misses.load();
}


void vattn_profile_enable(int on) {
    std::lock_guard<std::mutex> l(g_prof_mu);
    for (auto& e : g_prof) {
        cudaEventDestroy(e.a);
        cudaEventDestroy(e.b);
    }
    g_prof.clear();
    g_prof_on = on != 0;
}

int vattn_profile_read(int kind, double* ms_total, int* launches) {
    std::lock_guard<std::mutex> l(g_prof_mu);
    double t = 0;
    int n = 0;
    for (auto& e : g_prof) {
        if (e.kind != kind) continue;
        if (cudaEventSynchronize(e.b) != cudaSuccess) return fail(VATTN_ECUDA, "profile event sync");
        float ms = 0;
        cudaEventElapsedTime(&ms, e.a, e.b);
        t += ms;
        ++n;
    }
    if (ms_total) *ms_total = t;
    if (launches) *launches = n;
    return VATTN_OK;
}

static int forward_impl(const vattn_config* cfg, const void* q, const void* k, const void* v, void* o, float* lse,
                        uint32_t* mask, unsigned int* status, void* stream) {
    g_launches = 0;
    int rc = validate(cfg);
    if (rc) return rc;
    if (!q || !k || !v || !o || !lse) return fail(VATTN_EINVAL, "mha_forward: null tensor pointer");
    if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(o))
        return fail(VATTN_EINVAL, "mha_forward: tensors must be 16-byte aligned");
    if ((rc = check_device())) return rc;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int sel = (cfg->head_dim == 128 ? 4 : 0) | (cfg->dtype == VATTN_BF16 ? 2 : 0) | (cfg->dropout_p > 0.0f ? 1 : 0);
    switch (sel) {
        case 0: return launch_forward<64, false, false>(cfg, q, k, v, o, lse, mask, status, s);
        case 1: return launch_forward<64, false, true>(cfg, q, k, v, o, lse, mask, status, s);
        case 2: return launch_forward<64, true, false>(cfg, q, k, v, o, lse, mask, status, s);
        case 3: return launch_forward<64, true, true>(cfg, q, k, v, o, lse, mask, status, s);
        case 4: return launch_forward<128, false, false>(cfg, q, k, v, o, lse, mask, status, s);
        case 5: return launch_forward<128, false, true>(cfg, q, k, v, o, lse, mask, status, s);
        case 6: return launch_forward<128, true, false>(cfg, q, k, v, o, lse, mask, status, s);
        default: return launch_forward<128, true, true>(cfg, q, k, v, o, lse, mask, status, s);
    }
}

int mha_forward(const vattn_config* cfg, const void* q, const void* k, const void* v, void* o,
                float* lse, void* stream) {
    return forward_impl(cfg, q, k, v, o, lse, nullptr, nullptr, stream);
}

// internal (capi_host.cu): forward of one slab with the domain-error word
int vattn_forward_status_(const vattn_config* cfg, const void* q, const void* k, const void* v, void* o, float* lse,
                          unsigned int* status, void* stream) {
    return forward_impl(cfg, q, k, v, o, lse, nullptr, status, stream);
}

int mha_forward_ex(const vattn_config* cfg, const void* q, const void* k, const void* v, void* o, float* lse,
                   void* drop_mask, unsigned int* status, void* stream) {
    g_launches = 0;
    int rc = validate(cfg);
    if (rc) return rc;
    if (drop_mask) {
        if (cfg->dropout_p <= 0.0f) return fail(VATTN_EINVAL, "mha_forward_ex: drop_mask needs dropout_p > 0");
        if (!drop_mask_enabled()) return fail(VATTN_EINVAL, "mha_forward_ex: keep-bit masks are disabled (VATTN_DROP_MASK=0)");
        if ((reinterpret_cast<uintptr_t>(drop_mask) & 255u) != 0)
            return fail(VATTN_EINVAL, "mha_forward_ex: mask must be 256-byte aligned");
    }
    if (status && (reinterpret_cast<uintptr_t>(status) & 3u) != 0)
        return fail(VATTN_EINVAL, "mha_forward_ex: status word must be 4-byte aligned");
    return forward_impl(cfg, q, k, v, o, lse, static_cast<uint32_t*>(drop_mask), status, stream);
}

size_t mha_dropout_mask_bytes(const vattn_config* cfg) {
    if (validate(cfg) || cfg->dropout_p <= 0.0f || !drop_mask_enabled()) return 0;
    const size_t Npad = static_cast<size_t>((cfg->seq_len + 127) / 128) * 128;
    return 2 * static_cast<size_t>(units(cfg)) * Npad * (Npad / 8);  // query-major + key-major copies
}

int mha_forward_dropout_mask(const vattn_config* cfg, const void* q, const void* k, const void* v, void* o, float* lse,
                             void* drop_mask, void* stream) {
    g_launches = 0;
    int rc = validate(cfg);
    if (rc) return rc;
    if (cfg->dropout_p <= 0.0f) return fail(VATTN_EINVAL, "mha_forward_dropout_mask: dropout_p must be > 0");
    if (!drop_mask || (reinterpret_cast<uintptr_t>(drop_mask) & 255u) != 0)
        return fail(VATTN_EINVAL, "mha_forward_dropout_mask: mask must be non-null and 256-byte aligned");
    if (!drop_mask_enabled()) return fail(VATTN_EINVAL, "mha_forward_dropout_mask: keep-bit masks are disabled (VATTN_DROP_MASK=0)");
    return forward_impl(cfg, q, k, v, o, lse, static_cast<uint32_t*>(drop_mask), nullptr, stream);
}

int mha_dpsum(const vattn_config* cfg, const void* o, const void* dout, float* d_rows, void* stream) {
    g_launches = 0;
    int rc = validate(cfg);
    if (rc) return rc;
    if (!o || !dout || !d_rows) return fail(VATTN_EINVAL, "mha_dpsum: null pointer");
    if (!aligned16(o) || !aligned16(dout)) return fail(VATTN_EINVAL, "mha_dpsum: tensors must be 16-byte aligned");
    if ((rc = check_device())) return rc;
    const int BH = units(cfg), N = cfg->seq_len;
    const long long rows = static_cast<long long>(BH) * N;
    long long blocks = (rows + 15) / 16;
    if (blocks > 148 * 16) blocks = 148 * 16;
    const dim3 grid(static_cast<unsigned>(blocks));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // the backward's preprocess kernel with no padding and no lse2 output
    if (cfg->head_dim == 128) {
        if (cfg->dtype == VATTN_BF16)
            launch_pdl(mha_bwd_preprocess_kernel<128, true>, grid, dim3(256), 0, s, o, dout, (const float*)nullptr,
                       (float*)nullptr, d_rows, N, N, BH, (int*)nullptr, 0);
        else
            launch_pdl(mha_bwd_preprocess_kernel<128, false>, grid, dim3(256), 0, s, o, dout, (const float*)nullptr,
                       (float*)nullptr, d_rows, N, N, BH, (int*)nullptr, 0);
    } else {
        if (cfg->dtype == VATTN_BF16)
            launch_pdl(mha_bwd_preprocess_kernel<64, true>, grid, dim3(256), 0, s, o, dout, (const float*)nullptr,
                       (float*)nullptr, d_rows, N, N, BH, (int*)nullptr, 0);
        else
            launch_pdl(mha_bwd_preprocess_kernel<64, false>, grid, dim3(256), 0, s, o, dout, (const float*)nullptr,
                       (float*)nullptr, d_rows, N, N, BH, (int*)nullptr, 0);
    }
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = g_launch_err;
    g_launch_err = cudaSuccess;
    if (e != cudaSuccess) return fail(VATTN_ECUDA, std::string("mha_dpsum launch: ") + cudaGetErrorString(e));
    g_launches = 1;
    return VATTN_OK;
}

int vattn_dropout_digest(const vattn_config* cfg, int tile_rows, int tile_cols, unsigned long long* digest,
                         void* stream) {
    g_launches = 0;
    int rc = validate(cfg);
    if (rc) return rc;
    if (!digest) return fail(VATTN_EINVAL, "vattn_dropout_digest: null pointer");
    if (tile_rows < 1 || tile_cols < 1) return fail(VATTN_EINVAL, "vattn_dropout_digest: tiles must be positive");
    if ((rc = check_device())) return rc;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (cudaMemsetAsync(digest, 0, sizeof(unsigned long long), s) != cudaSuccess)
        return fail(VATTN_ECUDA, "vattn_dropout_digest: memset");
    if (cfg->dropout_p <= 0.0f) return VATTN_OK;  // no mask consumed: digest 0 (as the reference)
    int H, bh_off;
    float inv_keep;
    uint64_t seed, thresh;
    set_dropout(cfg, &H, &bh_off, &inv_keep, &seed, &thresh);
    const int N = cfg->seq_len;
    const dim3 grid((N + tile_rows - 1) / tile_rows, units(cfg));
    dropout_digest_kernel<<<grid, 256, 0, s>>>(digest, seed, H, bh_off, N, tile_rows, tile_cols, cfg->causal, thresh);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(VATTN_ECUDA, std::string("vattn_dropout_digest: ") + cudaGetErrorString(e));
    g_launches = 1;
    return VATTN_OK;
}

size_t mha_backward_workspace_bytes(const vattn_config* cfg) {
    if (validate(cfg)) return 0;
    return bwd_layout(cfg).total;
}

size_t mha_backward_workspace_bytes_mask(const vattn_config* cfg) {
    if (validate(cfg)) return 0;
    const BwdLayout L = bwd_layout(cfg);
    return L.drop_mask ? L.mask : L.total;  // the caller's mask replaces the workspace's own
}

static int backward_impl(const vattn_config* cfg, const void* q, const void* k, const void* v, const void* o,
                         const void* dout, const float* lse, void* dq, void* dk, void* dv, void* workspace,
                         size_t workspace_bytes, const uint32_t* mask, void* stream) {
    g_launches = 0;
    int rc = validate(cfg);
    if (rc) return rc;
    if (!q || !k || !v || !o || !dout || !lse || !dq || !dk || !dv || !workspace)
        return fail(VATTN_EINVAL, "mha_backward: null pointer");
    if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(o) || !aligned16(dout) ||
        !aligned16(dq) || !aligned16(dk) || !aligned16(dv))
        return fail(VATTN_EINVAL, "mha_backward: tensors must be 16-byte aligned");
    if ((reinterpret_cast<uintptr_t>(workspace) & 255u) != 0)
        return fail(VATTN_EINVAL, "mha_backward: workspace must be 256-byte aligned");
    {
        const BwdLayout L = bwd_layout(cfg);
        // with the forward's keep bits (mask) the workspace needs no mask region of its own
        if (workspace_bytes < ((mask && L.drop_mask) ? L.mask : L.total))
            return fail(VATTN_EINVAL, "mha_backward: workspace too small (see mha_backward_workspace_bytes)");
    }
    if ((rc = check_device())) return rc;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int sel = (cfg->head_dim == 128 ? 4 : 0) | (cfg->dtype == VATTN_BF16 ? 2 : 0) | (cfg->dropout_p > 0.0f ? 1 : 0);
#define VATTN_BWD(D, BF, DR) launch_backward<D, BF, DR>(cfg, q, k, v, o, dout, lse, dq, dk, dv, workspace, mask, s)
    switch (sel) {
        case 0: return VATTN_BWD(64, false, false);
        case 1: return VATTN_BWD(64, false, true);
        case 2: return VATTN_BWD(64, true, false);
        case 3: return VATTN_BWD(64, true, true);
        case 4: return VATTN_BWD(128, false, false);
        case 5: return VATTN_BWD(128, false, true);
        case 6: return VATTN_BWD(128, true, false);
        default: return VATTN_BWD(128, true, true);
    }
#undef VATTN_BWD
}

int mha_backward(const vattn_config* cfg, const void* q, const void* k, const void* v,
                 const void* o, const void* dout, const float* lse, void* dq, void* dk, void* dv,
                 void* workspace, size_t workspace_bytes, void* stream) {
    return backward_impl(cfg, q, k, v, o, dout, lse, dq, dk, dv, workspace, workspace_bytes, nullptr, stream);
}

// internal (capi_host.cu): forward + backward of one slab on device buffers.  With
// dropout the forward keeps its keep bits in the workspace's mask region and the
// backward reads them (no second hash pass).
int vattn_step_device_(const vattn_config* cfg, const void* q, const void* k, const void* v, const void* dout, void* o,
                       float* lse, void* dq, void* dk, void* dv, void* workspace, size_t workspace_bytes,
                       unsigned int* status, void* stream) {
    int rc = validate(cfg);
    if (rc) return rc;
    uint32_t* mask = nullptr;
    if (cfg->dropout_p > 0.0f) {
        const BwdLayout L = bwd_layout(cfg);
        if (L.drop_mask && workspace && workspace_bytes >= L.total)
            mask = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(workspace) + L.mask);
    }
    rc = forward_impl(cfg, q, k, v, o, lse, mask, status, stream);
    if (rc) return rc;
    return backward_impl(cfg, q, k, v, o, dout, lse, dq, dk, dv, workspace, workspace_bytes, mask, stream);
}

int mha_backward_dropout_mask(const vattn_config* cfg, const void* q, const void* k, const void* v, const void* o,
                              const void* dout, const float* lse, const void* drop_mask, void* dq, void* dk, void* dv,
                              void* workspace, size_t workspace_bytes, void* stream) {
    g_launches = 0;
    int rc = validate(cfg);
    if (rc) return rc;
    if (cfg->dropout_p <= 0.0f) return fail(VATTN_EINVAL, "mha_backward_dropout_mask: dropout_p must be > 0");
    if (!drop_mask || (reinterpret_cast<uintptr_t>(drop_mask) & 255u) != 0)
        return fail(VATTN_EINVAL, "mha_backward_dropout_mask: mask must be non-null and 256-byte aligned");
    return backward_impl(cfg, q, k, v, o, dout, lse, dq, dk, dv, workspace, workspace_bytes,
                         static_cast<const uint32_t*>(drop_mask), stream);
}

}  // extern "C"
