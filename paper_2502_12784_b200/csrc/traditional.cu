// traditional.cu -- the unfused three-pass attention forward (comparator only),
// include/vattn_b200_traditional.h.  Mirrors vattn::forward_traditional
// (reference proj/src/attention_forward.cpp:229-310): S = Q K^T materialised in
// binary32, a full-row softmax pass (scale, causal mask, natural exp, P = f16(w/l),
// dropout, lse = m + ln l), then O = P V.  The two GEMMs are cuBLAS strided-batched
// GEMMs (plain library GEMMs; the fused path in libvattn_b200.so never uses cuBLAS).
#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <cmath>
#include <string>

#include "../../include/vattn_b200_traditional.h"
#include "sm100_ptx.cuh"

using namespace vattn_sm100;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& m) {
    g_err = m;
    return code;
}

constexpr int kThreads = 256;

__device__ float block_reduce(float v, bool is_max, float* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float w = __shfl_xor_sync(0xffffffffu, v, o);
        v = is_max ? fmaxf(v, w) : v + w;
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();  // red[] free from the previous reduction
    if (lane == 0) red[warp] = v;
    __syncthreads();
    v = lane < kThreads / 32 ? red[lane] : (is_max ? -INFINITY : 0.0f);
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) {
        const float w = __shfl_xor_sync(0xffffffffu, v, o);
        v = is_max ? fmaxf(v, w) : v + w;
    }
    return __shfl_sync(0xffffffffu, v, 0);  // lanes >= 8 reduced only the identity
}

// One CTA per query row: three passes over the binary32 score row (max, sum, emit).
template <bool kBF16, bool kDrop>
__global__ void __launch_bounds__(kThreads) softmax_rows_kernel(const float* __restrict__ S, void* __restrict__ P,
                                                                float* __restrict__ lse, int N, float scale,
                                                                int causal, int H, int bh_off, float inv_keep,
                                                                uint64_t seed, uint64_t thresh) {
    using T16 = typename std::conditional<kBF16, __nv_bfloat16, __half>::type;
    __shared__ float red[kThreads / 32];
    const size_t row = blockIdx.x;
    const int i = static_cast<int>(row % N);
    const int bh = static_cast<int>(row / N);
    const float* s = S + row * N;
    T16* p = reinterpret_cast<T16*>(P) + row * N;
    const int lim = causal ? i + 1 : N;  // keys j < lim are visible (attention_forward.cpp:262)
    float m = -INFINITY;
    for (int j = threadIdx.x; j < lim; j += kThreads) m = fmaxf(m, s[j] * scale);
    m = block_reduce(m, true, red);
    float l = 0.0f;
    for (int j = threadIdx.x; j < lim; j += kThreads) l += expf(s[j] * scale - m);
    l = block_reduce(l, false, red);
    const float inv_l = 1.0f / l;
    DropRow dr{};
    if constexpr (kDrop) dr = drop_row(drop_bh_base(seed, (bh + bh_off) / H, (bh + bh_off) % H), i);
    for (int j = threadIdx.x; j < N; j += kThreads) {
        float pj = j < lim ? expf(s[j] * scale - m) * inv_l : 0.0f;  // w / l (:283)
        if constexpr (kDrop) pj = drop_keep(dr, j, thresh) ? pj * inv_keep : 0.0f;
        p[j] = static_cast<T16>(pj);
    }
    if (threadIdx.x == 0) lse[row] = m + logf(l);  // (:288)
}

cublasHandle_t handle() {
    thread_local cublasHandle_t h[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return nullptr;
    if (!h[dev] && cublasCreate(&h[dev]) != CUBLAS_STATUS_SUCCESS) h[dev] = nullptr;
    return h[dev];
}

size_t al(size_t x) { return (x + 255) & ~size_t(255); }

int units(const vattn_config* c) { return c->bh_count ? c->bh_count : c->batch * c->heads; }

int check(const vattn_config* c) {
    if (!c) return fail(VATTN_EINVAL, "vattn_config: null");
    if (c->batch < 1 || c->heads < 1 || c->seq_len < 1 || c->head_dim < 1)
        return fail(VATTN_EINVAL, "AttnConfig: sizes must be positive");
    if (c->head_dim % 4 != 0) return fail(VATTN_EINVAL, "AttnConfig: head_dim must be a multiple of 4");
    if (c->dtype != VATTN_F16 && c->dtype != VATTN_BF16) return fail(VATTN_EINVAL, "vattn_config: dtype");
    if (!(c->dropout_p >= 0.0f && c->dropout_p < 1.0f))
        return fail(VATTN_EINVAL, "AttnConfig: dropout_p must be in [0, 1)");
    if (c->bh_count < 0 || c->bh_offset < 0 ||
        static_cast<long long>(c->bh_offset) + c->bh_count > static_cast<long long>(c->batch) * c->heads ||
        (c->bh_count == 0 && c->bh_offset != 0))
        return fail(VATTN_EINVAL, "vattn_config: bad (b, h) slab");
    if (static_cast<long long>(units(c)) * c->seq_len > (1ll << 31) - 1)
        return fail(VATTN_EUNSUPPORTED, "traditional: B*H*N rows must fit in int32");
    return VATTN_OK;
}

}  // namespace

extern "C" {

const char* vattn_traditional_last_error(void) { return g_err.c_str(); }

size_t mha_forward_traditional_workspace_bytes(const vattn_config* c) {
    if (check(c)) return 0;
    const size_t nn = static_cast<size_t>(units(c)) * c->seq_len * c->seq_len;
    return al(nn * 4) + al(nn * 2);
}

int mha_forward_traditional(const vattn_config* c, const void* q, const void* k, const void* v, void* o,
                            float* lse, void* ws, size_t ws_bytes, void* stream) {
    int rc = check(c);
    if (rc) return rc;
    if (!q || !k || !v || !o || !lse || !ws) return fail(VATTN_EINVAL, "mha_forward_traditional: null pointer");
    if (ws_bytes < mha_forward_traditional_workspace_bytes(c))
        return fail(VATTN_EINVAL, "mha_forward_traditional: workspace too small");
    cublasHandle_t h = handle();
    if (!h) return fail(VATTN_ECUDA, "cublasCreate failed");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cublasSetStream(h, s);
    const int BH = units(c), N = c->seq_len, d = c->head_dim;
    const long long nn = static_cast<long long>(N) * N, nd = static_cast<long long>(N) * d;
    float* S = static_cast<float*>(ws);
    void* P = static_cast<uint8_t*>(ws) + al(static_cast<size_t>(BH) * nn * 4);
    const cudaDataType_t t16 = c->dtype == VATTN_BF16 ? CUDA_R_16BF : CUDA_R_16F;
    const float one = 1.0f, zero = 0.0f;
    // Pass 1: row-major S = Q K^T  <=>  column-major S^T = K Q^T  (m = n = N, k = d)
    cublasStatus_t st = cublasGemmStridedBatchedEx(h, CUBLAS_OP_T, CUBLAS_OP_N, N, N, d, &one, k, t16, d, nd, q, t16,
                                                   d, nd, &zero, S, CUDA_R_32F, N, nn, BH, CUBLAS_COMPUTE_32F,
                                                   CUBLAS_GEMM_DEFAULT);
    if (st != CUBLAS_STATUS_SUCCESS) return fail(VATTN_ECUDA, "cuBLAS S = Q K^T failed");
    // Pass 2: full-row softmax (+ dropout), P and lse written out
    const float scale = c->softmax_scale > 0.0f ? c->softmax_scale : 1.0f / std::sqrt(static_cast<float>(d));
    const float inv_keep = 1.0f / (1.0f - c->dropout_p);
    const uint64_t thresh = static_cast<uint64_t>(std::ceil(static_cast<double>(c->dropout_p) * 9007199254740992.0));
    const unsigned rows = static_cast<unsigned>(static_cast<long long>(BH) * N);
    const bool bf = c->dtype == VATTN_BF16, drop = c->dropout_p > 0.0f;
#define VATTN_SOFTMAX(BF, DR)                                                                              \
    softmax_rows_kernel<BF, DR><<<rows, kThreads, 0, s>>>(S, P, lse, N, scale, c->causal, c->heads,       \
                                                        c->bh_offset, inv_keep, c->seed, thresh)
    if (bf) {
        if (drop) VATTN_SOFTMAX(true, true); else VATTN_SOFTMAX(true, false);
    } else {
        if (drop) VATTN_SOFTMAX(false, true); else VATTN_SOFTMAX(false, false);
    }
#undef VATTN_SOFTMAX
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(VATTN_ECUDA, std::string("softmax launch: ") + cudaGetErrorString(e));
    // Pass 3: row-major O = P V  <=>  column-major O^T = V^T P^T  (m = d, n = N, k = N)
    st = cublasGemmStridedBatchedEx(h, CUBLAS_OP_N, CUBLAS_OP_N, d, N, N, &one, v, t16, d, nd, P, t16, N, nn, &zero,
                                    o, t16, d, nd, BH, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
    if (st != CUBLAS_STATUS_SUCCESS) return fail(VATTN_ECUDA, "cuBLAS O = P V failed");
    return VATTN_OK;
}

}  // extern "C"
