// ref_shim.cpp -- extern "C" shim over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY (see vattn_oracle.c header).  Compiled together
// with the reference's own sources from /root/reference/proj/src by
// oracle/Makefile into oracle/_ref/libvattn_ref.so (never copied into this
// repo).  Used to (a) generate the golden fixtures under tests/golden/
// (oracle/gen_golden.py), (b) cross-check the C restatement, and (c) time the
// reference's CPU path as bench.py's cpu_baseline / `--impl reference` arm.
//
// Entry points wrap, one to one:
//   vr_forward_fused      -> vattn::forward_fused       include/vattn/attention.hpp:51-52
//   vr_backward_fused     -> vattn::backward_fused      include/vattn/backward.hpp:56-59
//   vr_compute_dpsum      -> vattn::compute_dpsum       include/vattn/backward.hpp:43
//   vr_attention_ref      -> vattn::attention_ref       include/vattn/reference.hpp:22-23
//   vr_attention_grad_ref -> vattn::attention_grad_ref  include/vattn/reference.hpp:31-34
//   vr_normal_tensor_f16  -> vattn::normal_tensor_f16   include/vattn/workload.hpp:10-17
//   vr_*_dropout          -> the same entry points with AttnConfig::dropout_p / seed set
//   vr_dropout_keep       -> vattn::dropout_keep                include/vattn/rng.hpp:22-26
//   vr_bench_units        -> forward_fused + backward_fused over (b,h) units on host threads
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "vattn/attention.hpp"
#include "vattn/backward.hpp"
#include "vattn/reference.hpp"
#include "vattn/tensor_io.hpp"
#include "vattn/workload.hpp"

using namespace vattn;

namespace {

thread_local std::string g_err;

std::vector<std::size_t> dims4(int B, int H, int N, int d) {
    return {static_cast<std::size_t>(B), static_cast<std::size_t>(H), static_cast<std::size_t>(N),
            static_cast<std::size_t>(d)};
}

Tensor<Half> from_bits(const uint16_t* p, int B, int H, int N, int d) {
    Tensor<Half> t(dims4(B, H, N, d));
    for (std::size_t i = 0; i < t.size(); ++i) t.data()[i] = Half::from_bits(p[i]);
    return t;
}

Tensor<double> from_f64(const double* p, int B, int H, int N, int d) {
    Tensor<double> t(dims4(B, H, N, d));
    std::memcpy(t.data(), p, t.size() * sizeof(double));
    return t;
}

AttnConfig make_cfg(int B, int H, int N, int d, int br, int bc, int causal, int acc_fp16,
                    float scale, float dropout_p = 0.0f, uint64_t seed = 0) {
    AttnConfig c;
    c.batch = B;
    c.heads = H;
    c.seq_len = N;
    c.head_dim = d;
    c.tile_rows = br;
    c.tile_cols = bc;
    c.causal = causal != 0;
    c.acc_mode = acc_fp16 ? AccMode::FP16_ACC : AccMode::FP32_ACC;
    c.softmax_scale = scale;
    c.dropout_p = dropout_p;
    c.seed = seed;
    return c;
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::domain_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}

}  // namespace

extern "C" {

const char* vr_last_error() { return g_err.c_str(); }

void vr_normal_tensor_f16(uint64_t seed, uint64_t stream, uint64_t count, uint16_t* out) {
    const Tensor<Half> t = normal_tensor_f16(seed, stream, {static_cast<std::size_t>(count)});
    for (std::size_t i = 0; i < t.size(); ++i) out[i] = t.data()[i].bits;
}

int vr_forward_fused(int B, int H, int N, int d, int br, int bc, int causal, int acc_fp16,
                     float scale, const uint16_t* q, const uint16_t* k, const uint16_t* v,
                     uint16_t* out, float* lse) {
    return guarded([&] {
        const AttnConfig cfg = make_cfg(B, H, N, d, br, bc, causal, acc_fp16, scale);
        const ForwardOutput r = forward_fused(from_bits(q, B, H, N, d), from_bits(k, B, H, N, d),
                                              from_bits(v, B, H, N, d), cfg);
        for (std::size_t i = 0; i < r.out.size(); ++i) out[i] = r.out.data()[i].bits;
        std::memcpy(lse, r.lse.data(), r.lse.size() * sizeof(float));
    });
}

int vr_backward_fused(int B, int H, int N, int d, int br, int bc, int causal, float scale,
                      const uint16_t* q, const uint16_t* k, const uint16_t* v,
                      const uint16_t* dout, const float* lse, uint16_t* dq, uint16_t* dk,
                      uint16_t* dv) {
    return guarded([&] {
        const AttnConfig cfg = make_cfg(B, H, N, d, br, bc, causal, /*acc_fp16=*/1, scale);
        Tensor<float> l(std::vector<std::size_t>{static_cast<std::size_t>(B),
                                                 static_cast<std::size_t>(H),
                                                 static_cast<std::size_t>(N)});
        std::memcpy(l.data(), lse, l.size() * sizeof(float));
        const GradOutputs g =
            backward_fused(from_bits(q, B, H, N, d), from_bits(k, B, H, N, d),
                           from_bits(v, B, H, N, d), from_bits(dout, B, H, N, d), l, cfg);
        for (std::size_t i = 0; i < g.dq.size(); ++i) {
            dq[i] = g.dq.data()[i].bits;
            dk[i] = g.dk.data()[i].bits;
            dv[i] = g.dv.data()[i].bits;
        }
    });
}

int vr_compute_dpsum(int B, int H, int N, int d, const uint16_t* dout, const uint16_t* o,
                     float* dpsum) {
    return guarded([&] {
        const Tensor<float> r =
            compute_dpsum(from_bits(dout, B, H, N, d), from_bits(o, B, H, N, d));
        std::memcpy(dpsum, r.data(), r.size() * sizeof(float));
    });
}

int vr_attention_ref(int B, int H, int N, int d, int causal, float scale, const double* q,
                     const double* k, const double* v, double* out, double* lse) {
    return guarded([&] {
        const AttnConfig cfg = make_cfg(B, H, N, d, 8, 8, causal, 0, scale);
        const RefForward r = attention_ref(from_f64(q, B, H, N, d), from_f64(k, B, H, N, d),
                                           from_f64(v, B, H, N, d), cfg);
        std::memcpy(out, r.out.data(), r.out.size() * sizeof(double));
        std::memcpy(lse, r.lse.data(), r.lse.size() * sizeof(double));
    });
}

int vr_attention_grad_ref(int B, int H, int N, int d, int causal, float scale, const double* q,
                          const double* k, const double* v, const double* dout, double* dq,
                          double* dk, double* dv) {
    return guarded([&] {
        const AttnConfig cfg = make_cfg(B, H, N, d, 8, 8, causal, 0, scale);
        const RefGrads g =
            attention_grad_ref(from_f64(q, B, H, N, d), from_f64(k, B, H, N, d),
                               from_f64(v, B, H, N, d), from_f64(dout, B, H, N, d), cfg);
        std::memcpy(dq, g.dq.data(), g.dq.size() * sizeof(double));
        std::memcpy(dk, g.dk.data(), g.dk.size() * sizeof(double));
        std::memcpy(dv, g.dv.data(), g.dv.size() * sizeof(double));
    });
}

// Dropout variants (rng.cpp:35-54; attention_forward.cpp:77-106; attention_backward.cpp:145-160;
// reference.cpp:66-69, 118-121).  mask_digest is returned for completeness.
int vr_dropout_keep(uint64_t seed, uint64_t b, uint64_t h, uint64_t row, uint64_t col, float p) {
    return dropout_keep(seed, b, h, row, col, p) ? 1 : 0;
}

int vr_forward_fused_dropout(int B, int H, int N, int d, int br, int bc, int causal, int acc_fp16,
                             float scale, float dropout_p, uint64_t seed, const uint16_t* q,
                             const uint16_t* k, const uint16_t* v, uint16_t* out, float* lse,
                             uint64_t* digest) {
    return guarded([&] {
        const AttnConfig cfg = make_cfg(B, H, N, d, br, bc, causal, acc_fp16, scale, dropout_p, seed);
        const ForwardOutput r = forward_fused(from_bits(q, B, H, N, d), from_bits(k, B, H, N, d),
                                              from_bits(v, B, H, N, d), cfg);
        for (std::size_t i = 0; i < r.out.size(); ++i) out[i] = r.out.data()[i].bits;
        std::memcpy(lse, r.lse.data(), r.lse.size() * sizeof(float));
        *digest = r.mask_digest;
    });
}

int vr_backward_fused_dropout(int B, int H, int N, int d, int br, int bc, int causal, float scale,
                              float dropout_p, uint64_t seed, const uint16_t* q, const uint16_t* k,
                              const uint16_t* v, const uint16_t* dout, const float* lse,
                              uint16_t* dq, uint16_t* dk, uint16_t* dv, uint64_t* digest) {
    return guarded([&] {
        const AttnConfig cfg = make_cfg(B, H, N, d, br, bc, causal, 1, scale, dropout_p, seed);
        Tensor<float> l(std::vector<std::size_t>{static_cast<std::size_t>(B),
                                                 static_cast<std::size_t>(H),
                                                 static_cast<std::size_t>(N)});
        std::memcpy(l.data(), lse, l.size() * sizeof(float));
        const GradOutputs g =
            backward_fused(from_bits(q, B, H, N, d), from_bits(k, B, H, N, d),
                           from_bits(v, B, H, N, d), from_bits(dout, B, H, N, d), l, cfg);
        for (std::size_t i = 0; i < g.dq.size(); ++i) {
            dq[i] = g.dq.data()[i].bits;
            dk[i] = g.dk.data()[i].bits;
            dv[i] = g.dv.data()[i].bits;
        }
        *digest = g.mask_digest;
    });
}

int vr_attention_ref_dropout(int B, int H, int N, int d, int causal, float scale, float dropout_p,
                             uint64_t seed, const double* q, const double* k, const double* v,
                             double* out, double* lse) {
    return guarded([&] {
        const AttnConfig cfg = make_cfg(B, H, N, d, 8, 8, causal, 0, scale, dropout_p, seed);
        const RefForward r = attention_ref(from_f64(q, B, H, N, d), from_f64(k, B, H, N, d),
                                           from_f64(v, B, H, N, d), cfg);
        std::memcpy(out, r.out.data(), r.out.size() * sizeof(double));
        std::memcpy(lse, r.lse.data(), r.lse.size() * sizeof(double));
    });
}

int vr_attention_grad_ref_dropout(int B, int H, int N, int d, int causal, float scale,
                                  float dropout_p, uint64_t seed, const double* q, const double* k,
                                  const double* v, const double* dout, double* dq, double* dk,
                                  double* dv) {
    return guarded([&] {
        const AttnConfig cfg = make_cfg(B, H, N, d, 8, 8, causal, 0, scale, dropout_p, seed);
        const RefGrads g =
            attention_grad_ref(from_f64(q, B, H, N, d), from_f64(k, B, H, N, d),
                               from_f64(v, B, H, N, d), from_f64(dout, B, H, N, d), cfg);
        std::memcpy(dq, g.dq.data(), g.dq.size() * sizeof(double));
        std::memcpy(dk, g.dk.data(), g.dk.size() * sizeof(double));
        std::memcpy(dv, g.dv.data(), g.dv.size() * sizeof(double));
    });
}

// CPU baseline: `units` independent (b,h) slices [1,1,N,d], each running
// forward_fused (FP32-ACC, 64x64 tiles) then backward_fused (FP16-ACC, its only
// mode), spread over `threads` host threads (the reference API is reentrant,
// SURVEY 8b).  Inputs are generated before the clock starts.  Returns the wall
// seconds of the timed region, or a negative value on error.
double vr_bench_units(int N, int d, int causal, int units, int threads) {
    const int tile = N < 64 ? N : 64;
    const AttnConfig fcfg = make_cfg(1, 1, N, d, tile, tile, causal, 0, 0.0f);
    const AttnConfig bcfg = make_cfg(1, 1, N, d, tile, tile, causal, 1, 0.0f);
    struct Unit {
        Tensor<Half> q, k, v, dout;
    };
    std::vector<Unit> work;
    work.reserve(static_cast<std::size_t>(units));
    for (int u = 0; u < units; ++u) {
        const auto dims = dims4(1, 1, N, d);
        const uint64_t seed = 1000 + static_cast<uint64_t>(u);
        work.push_back({normal_tensor_f16(seed, 1, dims), normal_tensor_f16(seed, 2, dims),
                        normal_tensor_f16(seed, 3, dims), normal_tensor_f16(seed, 4, dims)});
    }
    std::atomic<int> next{0};
    std::atomic<int> failed{0};
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int t = 0; t < (threads < 1 ? 1 : threads); ++t) {
        pool.emplace_back([&] {
            for (int u = next.fetch_add(1); u < units; u = next.fetch_add(1)) {
                try {
                    const Unit& w = work[static_cast<std::size_t>(u)];
                    const ForwardOutput f = forward_fused(w.q, w.k, w.v, fcfg);
                    const GradOutputs g = backward_fused(w.q, w.k, w.v, w.dout, f.lse, bcfg);
                    if (g.dq.size() == 0) failed.store(1);
                } catch (...) {
                    failed.store(1);
                }
            }
        });
    }
    for (auto& th : pool) th.join();
    const double secs =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return failed.load() ? -1.0 : secs;
}

// ---- TrafficCounter of the reference's own passes (pins the closed forms in
// paper_2502_12784_b200/traffic.py).  out[7] = matrix_pass_reads, matrix_pass_writes,
// element_reads, element_writes, mma_invocations, shuffle_events, convert_events.
static void put_traffic(const TrafficCounter& t, uint64_t* out) {
    out[0] = t.matrix_pass_reads;
    out[1] = t.matrix_pass_writes;
    out[2] = t.element_reads;
    out[3] = t.element_writes;
    out[4] = t.mma_invocations;
    out[5] = t.shuffle_events;
    out[6] = t.convert_events;
}

int vr_traffic(int which, int B, int H, int N, int d, int br, int bc, int causal, uint64_t* out) {
    return guarded([&] {
        const auto dims = dims4(B, H, N, d);
        const Tensor<Half> q = normal_tensor_f16(1, 1, dims), k = normal_tensor_f16(1, 2, dims),
                           v = normal_tensor_f16(1, 3, dims), dout = normal_tensor_f16(1, 4, dims);
        // which: 0 forward_fused FP32-ACC, 1 forward_traditional FP32-ACC, 2 backward_fused,
        //        3 forward_fused FP16-ACC, 4 forward_traditional FP16-ACC
        if (which == 0 || which == 3) {
            put_traffic(forward_fused(q, k, v, make_cfg(B, H, N, d, br, bc, causal, which == 3, 0.0f)).traffic, out);
        } else if (which == 1 || which == 4) {
            put_traffic(forward_traditional(q, k, v, make_cfg(B, H, N, d, br, bc, causal, which == 4, 0.0f)).traffic,
                        out);
        } else {  // backward_fused (FP16-ACC, its only mode)
            const AttnConfig c = make_cfg(B, H, N, d, br, bc, causal, 1, 0.0f);
            const ForwardOutput f = forward_fused(q, k, v, c);
            put_traffic(backward_fused(q, k, v, dout, f.lse, c).traffic, out);
        }
    });
}

// ---- SPAT container round trips through the reference's tensor_io.cpp
int vr_write_spat_f16(const char* path, int rank, const uint64_t* dims, const uint16_t* bits) {
    return guarded([&] {
        std::vector<std::size_t> dv(dims, dims + rank);
        Tensor<Half> t(dv);
        for (std::size_t i = 0; i < t.size(); ++i) t.data()[i] = Half::from_bits(bits[i]);
        write_spat(path, t);
    });
}
int vr_write_spat_f32(const char* path, int rank, const uint64_t* dims, const float* vals) {
    return guarded([&] {
        std::vector<std::size_t> dv(dims, dims + rank);
        Tensor<float> t(dv);
        std::memcpy(t.data(), vals, t.size() * sizeof(float));
        write_spat(path, t);
    });
}
int vr_read_spat_check(const char* path) {  // 0 = reads cleanly, else the error class
    return guarded([&] { (void)read_spat(path); });
}

}  // extern "C"
