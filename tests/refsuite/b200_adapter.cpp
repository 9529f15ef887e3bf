// b200_adapter.cpp -- the reference's fused-path API implemented on the B200 library,
// so the reference's OWN unit tests (proj/tests/test_forward.cpp, test_backward.cpp,
// compiled unmodified) run against the GPU path.  Test infrastructure: it replaces
// exactly the two reference translation units that hold the path
// (proj/src/attention_forward.cpp, attention_backward.cpp); every other reference
// source (binary64 oracle, RNG, binary16, workload, tensor I/O) is the reference's own.
//
// Mapping:
//   vattn::forward_fused       -> vattn_b200::forward_fused (C ABI mha_forward_host)
//   vattn::backward_fused      -> vattn_b200::backward_fused (mha_forward + mha_backward; with dropout
//                                 the *_dropout_mask pair, the forward keeping its keep bits)
//   vattn::forward_traditional -> mha_forward_traditional (unfused comparator)
//   vattn::compute_dpsum       -> mha_dpsum
//   TrafficCounter             -> closed forms (vattn_b200::traffic_*)
// mask_digest comes from vattn_dropout_digest (bit-identical to the reference's).
// Documented divergences the reference's tests can observe: no
// ForwardTrace / DqContribution log / Volta datapath event counters (emulation hooks),
// outputs are not bit-identical to the emulated m8n8k4 pipeline, and the backward
// accepts FP32-ACC (the GPU always accumulates in fp32).
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "vattn/attention.hpp"
#include "vattn/backward.hpp"
#include "vattn/half.hpp"
#include "vattn_b200.h"
#include "vattn_b200/mha.hpp"
#include "vattn_b200_traditional.h"

namespace vattn {

namespace {

void require(bool ok, const char* msg) {
    if (!ok) throw std::invalid_argument(msg);
}

void require_bhnd(const Tensor<Half>& t, const AttnConfig& cfg, const char* what) {
    require(t.rank() == 4 && t.dims()[0] == static_cast<std::size_t>(cfg.batch) &&
                t.dims()[1] == static_cast<std::size_t>(cfg.heads) &&
                t.dims()[2] == static_cast<std::size_t>(cfg.seq_len) &&
                t.dims()[3] == static_cast<std::size_t>(cfg.head_dim),
            what);
}

vattn_b200::AttnConfig to_b200(const AttnConfig& c) {
    vattn_b200::AttnConfig b;
    b.batch = c.batch;
    b.heads = c.heads;
    b.seq_len = c.seq_len;
    b.head_dim = c.head_dim;
    b.tile_rows = c.tile_rows;
    b.tile_cols = c.tile_cols;
    b.causal = c.causal;
    b.dropout_p = c.dropout_p;
    b.seed = c.seed;
    b.softmax_scale = c.softmax_scale;
    b.dtype = VATTN_F16;
    b.acc_mode = c.acc_mode == AccMode::FP16_ACC ? vattn_b200::AccMode::FP16_ACC : vattn_b200::AccMode::FP32_ACC;
    return b;
}

std::vector<uint16_t> bits(const Tensor<Half>& t) {
    std::vector<uint16_t> v(t.size());
    for (std::size_t i = 0; i < t.size(); ++i) v[i] = t.data()[i].bits;
    return v;
}

Tensor<Half> from_bits(const std::vector<uint16_t>& v, const std::vector<std::size_t>& dims) {
    Tensor<Half> t(dims);
    for (std::size_t i = 0; i < t.size(); ++i) t.data()[i] = Half::from_bits(v[i]);
    return t;
}

TrafficCounter to_ref(const vattn_b200::TrafficCounter& b) {
    TrafficCounter t;
    t.matrix_pass_reads = b.matrix_pass_reads;
    t.matrix_pass_writes = b.matrix_pass_writes;
    t.element_reads = b.element_reads;
    t.element_writes = b.element_writes;
    t.mma_invocations = b.mma_invocations;
    t.shuffle_events = b.shuffle_events;
    t.convert_events = b.convert_events;
    return t;
}

void cuda_ok(cudaError_t e, const char* where) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(where) + ": " + cudaGetErrorString(e));
}

}  // namespace

// AttnConfig::validate / scale: the reference's rules (attention_forward.cpp:31-45)
void AttnConfig::validate() const {
    require(batch >= 1 && heads >= 1, "AttnConfig: batch and heads must be positive");
    require(seq_len > 0 && head_dim > 0, "AttnConfig: seq_len and head_dim must be positive");
    require(tile_rows > 0 && tile_rows % 8 == 0, "AttnConfig: tile_rows must be a positive multiple of 8");
    require(tile_cols > 0 && tile_cols % 8 == 0, "AttnConfig: tile_cols must be a positive multiple of 8");
    require(head_dim % 4 == 0, "AttnConfig: head_dim must be a multiple of 4");
    require(seq_len % tile_rows == 0, "AttnConfig: seq_len must be a multiple of tile_rows");
    require(seq_len % tile_cols == 0, "AttnConfig: seq_len must be a multiple of tile_cols");
    require(dropout_p >= 0.0f && dropout_p < 1.0f, "AttnConfig: dropout_p must be in [0, 1)");
}

float AttnConfig::scale() const {
    return softmax_scale > 0.0f ? softmax_scale : 1.0f / std::sqrt(static_cast<float>(head_dim));
}

ForwardOutput forward_fused(const Tensor<Half>& q, const Tensor<Half>& k, const Tensor<Half>& v,
                            const AttnConfig& cfg, ForwardTrace* trace) {
    cfg.validate();
    require_bhnd(q, cfg, "forward_fused: Q shape mismatch");
    require_bhnd(k, cfg, "forward_fused: K shape mismatch");
    require_bhnd(v, cfg, "forward_fused: V shape mismatch");
    if (trace) throw std::logic_error("forward_fused: ForwardTrace is an emulation hook, not produced on B200");
    const auto r = vattn_b200::forward_fused(bits(q), bits(k), bits(v), to_b200(cfg));
    ForwardOutput out;
    out.out = from_bits(r.out, q.dims());
    out.lse = Tensor<float>(std::vector<std::size_t>{q.dims()[0], q.dims()[1], q.dims()[2]});
    std::memcpy(out.lse.data(), r.lse.data(), r.lse.size() * sizeof(float));
    out.traffic = to_ref(r.traffic);
    out.mask_digest = r.mask_digest;
    return out;
}

ForwardOutput forward_traditional(const Tensor<Half>& q, const Tensor<Half>& k, const Tensor<Half>& v,
                                  const AttnConfig& cfg) {
    cfg.validate();
    require_bhnd(q, cfg, "forward_traditional: Q shape mismatch");
    require_bhnd(k, cfg, "forward_traditional: K shape mismatch");
    require_bhnd(v, cfg, "forward_traditional: V shape mismatch");
    vattn_config c{};
    c.batch = cfg.batch;
    c.heads = cfg.heads;
    c.seq_len = cfg.seq_len;
    c.head_dim = cfg.head_dim;
    c.causal = cfg.causal ? 1 : 0;
    c.softmax_scale = cfg.scale();
    c.dtype = VATTN_F16;
    c.dropout_p = cfg.dropout_p;
    c.seed = cfg.seed;
    const std::size_t bytes = q.size() * 2, rows = q.size() / cfg.head_dim;
    const std::size_t ws_bytes = mha_forward_traditional_workspace_bytes(&c);
    if (ws_bytes == 0) throw std::invalid_argument(vattn_traditional_last_error());
    void *dq, *dk, *dv, *dout, *dlse, *ws;
    cuda_ok(cudaMalloc(&dq, bytes), "cudaMalloc");
    cuda_ok(cudaMalloc(&dk, bytes), "cudaMalloc");
    cuda_ok(cudaMalloc(&dv, bytes), "cudaMalloc");
    cuda_ok(cudaMalloc(&dout, bytes), "cudaMalloc");
    cuda_ok(cudaMalloc(&dlse, rows * 4), "cudaMalloc");
    cuda_ok(cudaMalloc(&ws, ws_bytes), "cudaMalloc");
    cuda_ok(cudaMemcpy(dq, q.data(), bytes, cudaMemcpyHostToDevice), "H2D");
    cuda_ok(cudaMemcpy(dk, k.data(), bytes, cudaMemcpyHostToDevice), "H2D");
    cuda_ok(cudaMemcpy(dv, v.data(), bytes, cudaMemcpyHostToDevice), "H2D");
    const int rc = mha_forward_traditional(&c, dq, dk, dv, dout, static_cast<float*>(dlse), ws, ws_bytes, nullptr);
    ForwardOutput out;
    out.out = Tensor<Half>(q.dims());
    out.lse = Tensor<float>(std::vector<std::size_t>{q.dims()[0], q.dims()[1], q.dims()[2]});
    if (rc == VATTN_OK) {
        cuda_ok(cudaMemcpy(out.out.data(), dout, bytes, cudaMemcpyDeviceToHost), "D2H");
        cuda_ok(cudaMemcpy(out.lse.data(), dlse, rows * 4, cudaMemcpyDeviceToHost), "D2H");
    }
    for (void* p : {dq, dk, dv, dout, dlse, ws}) cudaFree(p);
    if (rc != VATTN_OK) throw std::invalid_argument(vattn_traditional_last_error());
    out.traffic = to_ref(vattn_b200::traffic_forward_traditional(to_b200(cfg)));
    vattn_config all = c;  // the traditional pass consumes every N x N position
    all.causal = 0;
    out.mask_digest = vattn_b200::detail::mask_digest(all, cfg.seq_len, cfg.seq_len);
    return out;
}

DqAccumulator::DqAccumulator(int batch, int heads, int n, int d)
    : buffer_(Tensor<float>::bhnd(batch, heads, n, d)) {}

Tensor<Half> DqAccumulator::finalize() const {
    Tensor<Half> out(buffer_.dims());
    for (std::size_t i = 0; i < buffer_.size(); ++i) out.data()[i] = f32_to_f16(buffer_.data()[i]);
    return out;
}

void dq_atomic_add(DqAccumulator& acc, const DqContribution& c) {
    const auto& dims = acc.buffer_.dims();
    require(c.delta.rows() == static_cast<int>(dims[2]) && c.delta.cols() == static_cast<int>(dims[3]),
            "dq_atomic_add: contribution shape mismatch");
    require(c.b >= 0 && c.b < static_cast<int>(dims[0]) && c.h >= 0 && c.h < static_cast<int>(dims[1]),
            "dq_atomic_add: batch/head out of range");
    for (int i = 0; i < c.delta.rows(); ++i)
        for (int j = 0; j < c.delta.cols(); ++j) acc.buffer_.at(c.b, c.h, i, j) += c.delta.at(i, j);
}

Tensor<float> compute_dpsum(const Tensor<Half>& d_out, const Tensor<Half>& out) {
    require(d_out.dims() == out.dims() && out.rank() == 4, "compute_dpsum: shape mismatch");
    const std::size_t B = out.dims()[0], H = out.dims()[1], N = out.dims()[2], d = out.dims()[3];
    Tensor<float> r(std::vector<std::size_t>{B, H, N});
    // the kernel reads 64/128-wide rows: zero-pad other head dims (zeros add nothing)
    const int dn = d <= 64 ? 64 : 128;
    require(d <= 128, "compute_dpsum: head_dim > 128 is not supported on the B200 path");
    std::vector<uint16_t> a(B * H * N * dn, 0), b(B * H * N * dn, 0);
    for (std::size_t row = 0; row < B * H * N; ++row)
        for (std::size_t j = 0; j < d; ++j) {
            a[row * dn + j] = out.data()[row * d + j].bits;
            b[row * dn + j] = d_out.data()[row * d + j].bits;
        }
    vattn_config c{};
    c.batch = static_cast<int>(B);
    c.heads = static_cast<int>(H);
    c.seq_len = static_cast<int>(N);
    c.head_dim = dn;
    c.dtype = VATTN_F16;
    void *da, *db, *dr;
    cuda_ok(cudaMalloc(&da, a.size() * 2), "cudaMalloc");
    cuda_ok(cudaMalloc(&db, b.size() * 2), "cudaMalloc");
    cuda_ok(cudaMalloc(&dr, r.size() * 4), "cudaMalloc");
    cuda_ok(cudaMemcpy(da, a.data(), a.size() * 2, cudaMemcpyHostToDevice), "H2D");
    cuda_ok(cudaMemcpy(db, b.data(), b.size() * 2, cudaMemcpyHostToDevice), "H2D");
    const int rc = mha_dpsum(&c, da, db, static_cast<float*>(dr), nullptr);
    if (rc == VATTN_OK) cuda_ok(cudaMemcpy(r.data(), dr, r.size() * 4, cudaMemcpyDeviceToHost), "D2H");
    cudaFree(da);
    cudaFree(db);
    cudaFree(dr);
    if (rc != VATTN_OK) throw std::invalid_argument(vattn_last_error());
    return r;
}

GradOutputs backward_fused(const Tensor<Half>& q, const Tensor<Half>& k, const Tensor<Half>& v,
                           const Tensor<Half>& d_out, const Tensor<float>& lse, const AttnConfig& cfg,
                           std::vector<DqContribution>* dq_log) {
    cfg.validate();
    require(q.dims() == k.dims() && q.dims() == v.dims() && q.dims() == d_out.dims(),
            "backward_fused: input shape mismatch");
    require_bhnd(q, cfg, "backward_fused: shapes do not match config");
    require(lse.rank() == 3 && lse.dims()[0] == static_cast<std::size_t>(cfg.batch) &&
                lse.dims()[1] == static_cast<std::size_t>(cfg.heads) &&
                lse.dims()[2] == static_cast<std::size_t>(cfg.seq_len),
            "backward_fused: lse shape mismatch");
    if (dq_log) throw std::logic_error("backward_fused: the DqContribution log is an emulation hook, not produced on B200");
    std::vector<float> l(lse.data(), lse.data() + lse.size());
    const auto g = vattn_b200::backward_fused(bits(q), bits(k), bits(v), bits(d_out), l, to_b200(cfg));
    GradOutputs r;
    r.dq = from_bits(g.dq, q.dims());
    r.dk = from_bits(g.dk, q.dims());
    r.dv = from_bits(g.dv, q.dims());
    r.traffic = to_ref(g.traffic);
    r.mask_digest = g.mask_digest;
    return r;
}

}  // namespace vattn
