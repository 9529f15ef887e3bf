// vattn_b200/mha.hpp -- C++ operator API of the B200 fused-MHA training path.
//
// Header-only layer over the C ABI (include/vattn_b200.h) that mirrors the
// reference's operator surface (arxiv 2502.12784, /root/reference/proj):
//
//   vattn_b200::AttnConfig      <- vattn::AttnConfig     (include/vattn/attention.hpp:11-26)
//   vattn_b200::ForwardOutput   <- vattn::ForwardOutput  (attention.hpp:28-33)
//   vattn_b200::GradOutputs     <- vattn::GradOutputs    (include/vattn/backward.hpp:10-14)
//   vattn_b200::forward_fused   <- vattn::forward_fused  (attention.hpp:51-52)
//   vattn_b200::backward_fused  <- vattn::backward_fused (backward.hpp:56-59)
//
// Host tensors use the reference layout (dense row-major [B, H, N, d], binary16
// bit patterns; lse [B, H, N] binary32).  Each call allocates device buffers,
// copies in, runs the sm_100a kernels through the C ABI on `stream`, copies
// out and synchronizes -- the drop-in for the reference's synchronous CPU
// calls.  The *_device overloads take caller-owned device pointers and are
// asynchronous (what benchmarks and training loops use).  Errors are thrown as
// the reference throws them: std::invalid_argument for config/shape problems,
// std::domain_error for numerical-domain problems, std::runtime_error for CUDA
// failures (there is no CPU fallback).
//
// head_dim values other than 64/128 (any d <= 128 with d % 4 == 0, as the
// reference allows) are zero-padded on the device: padded Q/K columns add 0 to
// every dot product, padded V columns produce 0 output columns that are dropped.
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../vattn_b200.h"

namespace vattn_b200 {

// vattn::AccMode (attention.hpp:9).  Selects the reference's emulated softmax-stage
// datapath, so it only changes the reported event counters; the GPU accumulates in fp32.
enum class AccMode { FP16_ACC, FP32_ACC };

struct AttnConfig {
    int batch = 1;
    int heads = 1;
    int seq_len = 0;
    int head_dim = 0;
    int tile_rows = 64;  // validated like the reference; the GPU tiles are fixed at 128
    int tile_cols = 64;
    bool causal = false;
    float dropout_p = 0.0f;
    uint64_t seed = 0;
    float softmax_scale = 0.0f;  // <= 0 picks 1/sqrt(head_dim)
    vattn_dtype dtype = VATTN_F16;
    AccMode acc_mode = AccMode::FP32_ACC;

    // AttnConfig::validate (proj/src/attention_forward.cpp:31-40), minus the
    // N % tile requirement the GPU path does not need.
    void validate() const {
        auto req = [](bool ok, const char* m) {
            if (!ok) throw std::invalid_argument(m);
        };
        req(batch >= 1 && heads >= 1, "AttnConfig: batch and heads must be positive");
        req(seq_len > 0 && head_dim > 0, "AttnConfig: seq_len and head_dim must be positive");
        req(tile_rows > 0 && tile_rows % 8 == 0, "AttnConfig: tile_rows must be a positive multiple of 8");
        req(tile_cols > 0 && tile_cols % 8 == 0, "AttnConfig: tile_cols must be a positive multiple of 8");
        req(head_dim % 4 == 0, "AttnConfig: head_dim must be a multiple of 4");
        req(dropout_p >= 0.0f && dropout_p < 1.0f, "AttnConfig: dropout_p must be in [0, 1)");
    }
    // AttnConfig::scale (attention_forward.cpp:42-45)
    float scale() const {
        return softmax_scale > 0.0f ? softmax_scale : 1.0f / std::sqrt(static_cast<float>(head_dim));
    }
    size_t elems() const {
        return static_cast<size_t>(batch) * heads * seq_len * head_dim;
    }
    size_t rows() const { return static_cast<size_t>(batch) * heads * seq_len; }
};

// vattn::TrafficCounter (include/vattn/traffic.hpp:12-31).  The GPU path emulates
// nothing, so the reference's modeled-HBM counters are filled from closed forms of
// its own bookkeeping (traffic_* below; pinned to the reference library by
// tests/test_traffic_spat.py and tests/cpp/mha_cpp_parity.cpp).  The Volta
// datapath events (mma_invocations, shuffle_events, convert_events) are pure
// functions of the config too and are restated the same way (paper_2502_12784_b200/
// traffic.py documents each term); measured DRAM bytes are in profiles/.
struct TrafficCounter {
    uint64_t matrix_pass_reads = 0;
    uint64_t matrix_pass_writes = 0;
    uint64_t element_reads = 0;
    uint64_t element_writes = 0;
    uint64_t mma_invocations = 0;
    uint64_t shuffle_events = 0;
    uint64_t convert_events = 0;
};

struct ForwardOutput {
    std::vector<uint16_t> out;  // [B, H, N, d] 16-bit bit patterns
    std::vector<float> lse;     // [B, H, N]
    TrafficCounter traffic;     // closed forms of attention.hpp:40-50
    uint64_t mask_digest = 0;   // the reference's dropout digest over the visited tiles (vattn_dropout_digest)
};

struct GradOutputs {
    std::vector<uint16_t> dq, dk, dv;  // [B, H, N, d]
    TrafficCounter traffic;            // closed forms of attention_backward.cpp:59-219
    uint64_t mask_digest = 0;
};

// (query-tile, key-tile) pairs a reference fused pass visits per (b, h)
// (causal: key tile kt is visited by query tile qt iff kt*Bc <= qt*Br + Br - 1,
// attention_forward.cpp:128, attention_backward.cpp:125).
inline uint64_t visited_pairs(const AttnConfig& c) {
    const int nq = c.seq_len / c.tile_rows, nk = c.seq_len / c.tile_cols;
    if (!c.causal) return static_cast<uint64_t>(nq) * nk;
    uint64_t t = 0;
    for (int qt = 0; qt < nq; ++qt) {
        const int last = (qt * c.tile_rows + c.tile_rows - 1) / c.tile_cols + 1;
        t += static_cast<uint64_t>(last < nk ? last : nk);
    }
    return t;
}

// m8n8k4 invocations of one tile GEMM C[rows x cols] += A[rows x k] B[k x cols]
// (tile_pipeline.cpp:36-49): (k/4) k-steps x rows/8 bands x ceil(cols/32) chunks.
inline uint64_t mma_count(uint64_t rows, uint64_t cols, uint64_t k) {
    return (k / 4) * (rows / 8) * ((cols / 8 + 3) / 4);
}
inline uint64_t pad8(uint64_t d) { return (d + 7) / 8 * 8; }

// Per-(b,h) events of T visited forward pairs (attention_forward.cpp:126-173).
inline void forward_events(uint64_t br, uint64_t bc, uint64_t d, uint64_t T, bool fp16_acc, uint64_t& mma,
                           uint64_t& shf, uint64_t& cvt) {
    mma = T * (mma_count(br, bc, d) + mma_count(br, pad8(d), bc));
    shf = fp16_acc ? 0 : T * 2 * (br / 8);        // xor rounds for row max and row sum
    cvt = fp16_acc ? T * (2 * br * bc + 2 * br * d) : 0;  // S widened, O round trip, P narrowed
}

inline TrafficCounter traffic_forward_fused(const AttnConfig& c) {
    const uint64_t BH = static_cast<uint64_t>(c.batch) * c.heads, N = c.seq_len, d = c.head_dim;
    const uint64_t T = visited_pairs(c);
    TrafficCounter t;
    t.matrix_pass_reads = 3;  // Q, K, V
    t.matrix_pass_writes = 1;  // O
    t.element_reads = BH * (N * d + 2ull * c.tile_cols * d * T);
    t.element_writes = BH * (N * d + N);
    uint64_t mma, shf, cvt;
    forward_events(c.tile_rows, c.tile_cols, d, T, c.acc_mode == AccMode::FP16_ACC, mma, shf, cvt);
    t.mma_invocations = BH * mma;
    t.shuffle_events = BH * shf;
    t.convert_events = BH * cvt;
    return t;
}

// forward_traditional (attention_forward.cpp:229-310): S, P materialised, 5/3 passes.
inline TrafficCounter traffic_forward_traditional(const AttnConfig& c) {
    const uint64_t BH = static_cast<uint64_t>(c.batch) * c.heads, N = c.seq_len, d = c.head_dim;
    TrafficCounter t;
    t.matrix_pass_reads = 5;   // Q, K | S | P, V
    t.matrix_pass_writes = 3;  // S | P | O
    t.element_reads = BH * (3 * N * d + 2 * N * N);
    t.element_writes = BH * (2 * N * N + N * d + N);
    t.mma_invocations = BH * (mma_count(N, N, d) + mma_count(N, pad8(d), N));
    return t;
}

inline TrafficCounter traffic_backward_fused(const AttnConfig& c) {
    const uint64_t BH = static_cast<uint64_t>(c.batch) * c.heads, N = c.seq_len, d = c.head_dim;
    const uint64_t br = c.tile_rows, bc = c.tile_cols, T = visited_pairs(c), nk = N / bc, dp = pad8(d);
    TrafficCounter t;
    t.matrix_pass_reads = 10;  // pre-pass Q K V; Q K V dO lse D; dQ finalize read
    t.matrix_pass_writes = 5;  // D, dK, dV, dQ adds, dQ narrowing
    t.element_reads = BH * ((N * d + 2 * bc * d * T) + 2 * bc * d * nk + T * (2 * br * d + 2 * br) + N * d);
    t.element_writes = BH * (N + T * br * d + 2 * bc * d * nk + N * d);
    uint64_t mma, shf, cvt;
    forward_events(br, bc, d, T, true, mma, shf, cvt);  // FP16-ACC recompute pre-pass (attention_backward.cpp:93-103)
    // S, dV, dP, dQ, dK GEMMs and four Br x Bc conversions per visited pair (:132-199)
    t.mma_invocations = BH * (mma + T * (2 * mma_count(br, bc, d) + 2 * mma_count(bc, dp, br) + mma_count(br, dp, bc)));
    t.convert_events = BH * (cvt + T * 4 * br * bc);
    return t;
}

namespace detail {

inline void check(int rc, const char* where) {
    if (rc == VATTN_OK) return;
    const std::string msg = std::string(where) + ": " + vattn_last_error();
    if (rc == VATTN_EINVAL) throw std::invalid_argument(msg);
    if (rc == VATTN_EDOMAIN) throw std::domain_error(msg);
    if (rc == VATTN_EUNSUPPORTED) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

inline void cuda(cudaError_t e, const char* where) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(where) + ": " + cudaGetErrorString(e));
}

struct DevBuf {
    void* p = nullptr;
    explicit DevBuf(size_t bytes) { cuda(cudaMalloc(&p, bytes ? bytes : 16), "cudaMalloc"); }
    ~DevBuf() { cudaFree(p); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
};

// Device domain-error word of one call (mha_forward_ex): zeroed on creation;
// throw_if_set() -- after the stream synchronised -- throws std::domain_error where
// the reference does (online_softmax.cpp:33-34 NaN score, :81-82 l == 0).
struct DomainWord {
    DevBuf buf{sizeof(unsigned int)};
    explicit DomainWord(cudaStream_t s) { cuda(cudaMemsetAsync(buf.p, 0, sizeof(unsigned int), s), "memset"); }
    unsigned int* ptr() const { return static_cast<unsigned int*>(buf.p); }
    void throw_if_set(const char* where) const {
        unsigned int h = 0;
        cuda(cudaMemcpy(&h, buf.p, sizeof(h), cudaMemcpyDeviceToHost), "D2H status");
        if (h & VATTN_DOMAIN_ROW)
            throw std::domain_error(std::string(where) +
                                    ": softmax: NaN score or fully masked row (l == 0) in a query row");
    }
};

inline int native_dim(int d) {
    if (d <= 64) return 64;
    if (d <= 128) return 128;
    throw std::invalid_argument("head_dim > 128 is not supported on the B200 path");
}

// host [rows, d] -> device [rows, dn] zero padded
inline void upload_padded(void* dst, const uint16_t* src, size_t rows, int d, int dn, cudaStream_t s) {
    if (d == dn) {
        cuda(cudaMemcpyAsync(dst, src, rows * d * 2, cudaMemcpyHostToDevice, s), "H2D");
        return;
    }
    cuda(cudaMemsetAsync(dst, 0, rows * dn * 2, s), "memset");
    cuda(cudaMemcpy2DAsync(dst, dn * 2, src, d * 2, d * 2, rows, cudaMemcpyHostToDevice, s), "H2D 2D");
}

inline void download_padded(uint16_t* dst, const void* src, size_t rows, int d, int dn, cudaStream_t s) {
    cuda(cudaMemcpy2DAsync(dst, d * 2, src, dn * 2, d * 2, rows, cudaMemcpyDeviceToHost, s), "D2H");
}

inline vattn_config to_c(const AttnConfig& c, int dn) {
    vattn_config r{};  // bh_offset = bh_count = 0: the whole problem
    r.batch = c.batch;
    r.heads = c.heads;
    r.seq_len = c.seq_len;
    r.head_dim = dn;
    r.causal = c.causal ? 1 : 0;
    r.softmax_scale = c.scale();  // scale of the true head_dim, not the padded one
    r.dtype = c.dtype;
    r.dropout_p = c.dropout_p;
    r.seed = c.seed;
    return r;
}

// The reference's mask_digest for a pass with (tile_rows x tile_cols) tiles (0 when
// dropout_p == 0): C ABI vattn_dropout_digest, bit-identical to the reference.
inline uint64_t mask_digest(const vattn_config& c, int tile_rows, int tile_cols) {
    if (c.dropout_p <= 0.0f) return 0;
    unsigned long long* d = nullptr;
    cuda(cudaMalloc(reinterpret_cast<void**>(&d), sizeof(unsigned long long)), "cudaMalloc");
    const int rc = vattn_dropout_digest(&c, tile_rows, tile_cols, d, nullptr);
    unsigned long long h = 0;
    if (rc == VATTN_OK) cuda(cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost), "D2H digest");
    cudaFree(d);
    check(rc, "vattn_dropout_digest");
    return h;
}

}  // namespace detail

// ---------------------------------------------------------- device overloads

// `status` (optional): zeroed device word that receives VATTN_DOMAIN_ROW for the rows
// where the reference would throw std::domain_error (read it after synchronising).
inline void forward_fused_device(const AttnConfig& cfg, const void* q, const void* k, const void* v,
                                 void* out, float* lse, cudaStream_t stream = nullptr,
                                 unsigned int* status = nullptr) {
    cfg.validate();
    if (cfg.head_dim != 64 && cfg.head_dim != 128)
        throw std::invalid_argument("forward_fused_device: head_dim must be 64 or 128 (use the host overload to pad)");
    const vattn_config c = detail::to_c(cfg, cfg.head_dim);
    detail::check(mha_forward_ex(&c, q, k, v, out, lse, nullptr, status, stream), "mha_forward_ex");
}

inline void backward_fused_device(const AttnConfig& cfg, const void* q, const void* k,
                                  const void* v, const void* out, const void* d_out,
                                  const float* lse, void* dq, void* dk, void* dv, void* workspace,
                                  size_t workspace_bytes, cudaStream_t stream = nullptr) {
    cfg.validate();
    if (cfg.head_dim != 64 && cfg.head_dim != 128)
        throw std::invalid_argument("backward_fused_device: head_dim must be 64 or 128");
    const vattn_config c = detail::to_c(cfg, cfg.head_dim);
    detail::check(mha_backward(&c, q, k, v, out, d_out, lse, dq, dk, dv, workspace, workspace_bytes, stream),
                  "mha_backward");
}

// ------------------------------------------------------------ host overloads

// vattn::forward_fused: host [B,H,N,d] binary16 in, ForwardOutput out.  Native
// head dims go through mha_forward_host (PCIe copies pipelined against the
// kernels, slab by slab); other head dims are zero-padded on the device.
inline ForwardOutput forward_fused(const std::vector<uint16_t>& q, const std::vector<uint16_t>& k,
                                   const std::vector<uint16_t>& v, const AttnConfig& cfg) {
    cfg.validate();
    if (q.size() != cfg.elems() || k.size() != cfg.elems() || v.size() != cfg.elems())
        throw std::invalid_argument("forward_fused: Q/K/V shape mismatch");
    const int dn = detail::native_dim(cfg.head_dim);
    const size_t rows = cfg.rows();
    ForwardOutput r;
    r.out.resize(cfg.elems());
    r.lse.resize(rows);
    r.traffic = traffic_forward_fused(cfg);
    const vattn_config c = detail::to_c(cfg, dn);
    r.mask_digest = detail::mask_digest(c, cfg.tile_rows, cfg.tile_cols);
    if (dn == cfg.head_dim) {
        detail::check(mha_forward_host(&c, q.data(), k.data(), v.data(), r.out.data(), r.lse.data(), nullptr),
                      "mha_forward_host");
        return r;
    }
    cudaStream_t s = nullptr;
    detail::DevBuf dq(rows * dn * 2), dk(rows * dn * 2), dv(rows * dn * 2), dout(rows * dn * 2),
        dlse(rows * 4);
    detail::upload_padded(dq.p, q.data(), rows, cfg.head_dim, dn, s);
    detail::upload_padded(dk.p, k.data(), rows, cfg.head_dim, dn, s);
    detail::upload_padded(dv.p, v.data(), rows, cfg.head_dim, dn, s);
    detail::DomainWord dom(s);
    detail::check(mha_forward_ex(&c, dq.p, dk.p, dv.p, dout.p, static_cast<float*>(dlse.p), nullptr, dom.ptr(), s),
                  "mha_forward_ex");
    detail::download_padded(r.out.data(), dout.p, rows, cfg.head_dim, dn, s);
    detail::cuda(cudaMemcpyAsync(r.lse.data(), dlse.p, rows * 4, cudaMemcpyDeviceToHost, s), "D2H lse");
    detail::cuda(cudaStreamSynchronize(s), "sync");
    dom.throw_if_set("forward_fused");
    return r;
}

// vattn::backward_fused (6-argument form): the reference re-runs the forward to
// obtain O (attention_backward.cpp:91-104); so does this overload.
inline GradOutputs backward_fused(const std::vector<uint16_t>& q, const std::vector<uint16_t>& k,
                                  const std::vector<uint16_t>& v, const std::vector<uint16_t>& d_out,
                                  const std::vector<float>& lse, const AttnConfig& cfg) {
    cfg.validate();
    if (q.size() != cfg.elems() || k.size() != cfg.elems() || v.size() != cfg.elems() ||
        d_out.size() != cfg.elems())
        throw std::invalid_argument("backward_fused: input shape mismatch");
    if (lse.size() != cfg.rows()) throw std::invalid_argument("backward_fused: lse shape mismatch");
    const int dn = detail::native_dim(cfg.head_dim);
    const size_t rows = cfg.rows();
    cudaStream_t s = nullptr;
    const size_t tb = rows * dn * 2;
    detail::DevBuf bq(tb), bk(tb), bv(tb), bdo(tb), bo(tb), bdq(tb), bdk(tb), bdv(tb), blse(rows * 4),
        bjunk(rows * 4);
    detail::upload_padded(bq.p, q.data(), rows, cfg.head_dim, dn, s);
    detail::upload_padded(bk.p, k.data(), rows, cfg.head_dim, dn, s);
    detail::upload_padded(bv.p, v.data(), rows, cfg.head_dim, dn, s);
    detail::upload_padded(bdo.p, d_out.data(), rows, cfg.head_dim, dn, s);
    detail::cuda(cudaMemcpyAsync(blse.p, lse.data(), rows * 4, cudaMemcpyHostToDevice, s), "H2D lse");
    const vattn_config c = detail::to_c(cfg, dn);
    // the recomputed forward (as the reference's) raises the reference's domain errors
    detail::DomainWord dom(s);
    const size_t mask_bytes = cfg.dropout_p > 0.0f ? mha_dropout_mask_bytes(&c) : 0;
    if (mask_bytes) {
        // the recomputed forward keeps its dropout keep bits; the backward reads them
        // instead of hashing every position again (bit-identical results), so the
        // workspace needs no mask region of its own
        const size_t wsb = mha_backward_workspace_bytes_mask(&c);
        detail::DevBuf ws(wsb);
        detail::DevBuf mask(mask_bytes);
        detail::check(mha_forward_ex(&c, bq.p, bk.p, bv.p, bo.p, static_cast<float*>(bjunk.p), mask.p, dom.ptr(), s),
                      "mha_forward_ex");
        detail::check(mha_backward_dropout_mask(&c, bq.p, bk.p, bv.p, bo.p, bdo.p, static_cast<const float*>(blse.p),
                                                mask.p, bdq.p, bdk.p, bdv.p, ws.p, wsb, s),
                      "mha_backward_dropout_mask");
        detail::cuda(cudaStreamSynchronize(s), "sync");  // before `mask` is freed
    } else {
        const size_t wsb = mha_backward_workspace_bytes(&c);
        detail::DevBuf ws(wsb);
        detail::check(mha_forward_ex(&c, bq.p, bk.p, bv.p, bo.p, static_cast<float*>(bjunk.p), nullptr, dom.ptr(), s),
                      "mha_forward_ex");
        detail::check(mha_backward(&c, bq.p, bk.p, bv.p, bo.p, bdo.p, static_cast<const float*>(blse.p),
                                   bdq.p, bdk.p, bdv.p, ws.p, wsb, s),
                      "mha_backward");
        detail::cuda(cudaStreamSynchronize(s), "sync");  // before `ws` is freed
    }
    dom.throw_if_set("backward_fused");
    GradOutputs g;
    g.traffic = traffic_backward_fused(cfg);
    g.mask_digest = detail::mask_digest(c, cfg.tile_rows, cfg.tile_cols);
    g.dq.resize(cfg.elems());
    g.dk.resize(cfg.elems());
    g.dv.resize(cfg.elems());
    detail::download_padded(g.dq.data(), bdq.p, rows, cfg.head_dim, dn, s);
    detail::download_padded(g.dk.data(), bdk.p, rows, cfg.head_dim, dn, s);
    detail::download_padded(g.dv.data(), bdv.p, rows, cfg.head_dim, dn, s);
    detail::cuda(cudaStreamSynchronize(s), "sync");
    return g;
}

}  // namespace vattn_b200
