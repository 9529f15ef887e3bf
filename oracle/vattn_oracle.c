/*
 * vattn_oracle.c -- CPU restatement of the reference's fused-MHA training path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the sm_100a
 * kernels in paper_2502_12784_b200/csrc.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The product
 * path never links or calls it; the CUDA library fails loudly when its own
 * kernels are missing instead of falling back here.
 *
 * Every function restates a reference function (paths relative to
 * /root/reference/proj) and is pinned against golden vectors produced by the
 * reference itself (oracle/gen_golden.cpp linked against the reference sources
 * compiled by oracle/Makefile into oracle/_ref/; fixtures in tests/golden/).
 *
 *   vo_mix64 / vo_hash_combine / vo_bits_to_unit / vo_normal_at
 *        src/rng.cpp:8-31                     (bit-exact)
 *   vo_f32_to_f16 / vo_f16_to_f32            src/half.cpp:5-65 (bit-exact)
 *   vo_f32_to_bf16 / vo_bf16_to_f32          RNE bf16 (no reference counterpart)
 *   vo_normal_tensor_f16                     include/vattn/workload.hpp:10-17 (bit-exact)
 *   vo_position_hash / vo_dropout_keep       src/rng.cpp:35-49 (bit-exact)
 *   vo_attention_ref[_dropout]               src/reference.cpp:26-80 (bit-exact)
 *   vo_attention_grad_ref[_dropout]          src/reference.cpp:82-167 (bit-exact)
 *   vo_forward_fused_fp32acc[_dropout]       src/attention_forward.cpp:110-227 with the
 *        FP32-ACC dot4 contract of src/half.cpp:67-77, the tile loop order of
 *        src/tile_pipeline.cpp:33-49, online softmax src/online_softmax.cpp:21-87
 *        and apply_dropout (:77-106) (bit-exact)
 *   vo_compute_dpsum                         src/attention_backward.cpp:44-57 (bit-exact)
 *   vo_error_metrics / vo_frobenius_rel      src/reference.cpp:186-222
 *
 * Layout everywhere: dense row-major [B, H, N, d] (include/vattn/tensor.hpp:45-50),
 * per-row scalars [B, H, N] (tensor.hpp:53-58).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define VO_EXPORT __attribute__((visibility("default")))

/* ---------------------------------------------------------------- rng ---- */

/* src/rng.cpp:8-13 (SplitMix64 finalizer). */
VO_EXPORT uint64_t vo_mix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

/* src/rng.cpp:15-17 */
VO_EXPORT uint64_t vo_hash_combine(uint64_t state, uint64_t v) {
    return vo_mix64(state ^ (v + 0x9e3779b97f4a7c15ull + (state << 6) + (state >> 2)));
}

/* src/rng.cpp:19-21 */
VO_EXPORT double vo_bits_to_unit(uint64_t bits) { return (double)(bits >> 11) * 0x1.0p-53; }

/* src/rng.cpp:23-31: Box-Muller over two counter draws. */
VO_EXPORT float vo_normal_at(uint64_t seed, uint64_t index) {
    const uint64_t a = vo_mix64(vo_hash_combine(seed, 2 * index));
    const uint64_t b = vo_mix64(vo_hash_combine(seed, 2 * index + 1));
    const double u1 = 1.0 - vo_bits_to_unit(a);
    const double u2 = vo_bits_to_unit(b);
    return (float)(sqrt(-2.0 * log(u1)) * cos(2.0 * 3.141592653589793238462643383279502884 * u2));
}

/* src/rng.cpp:35-42 position hash and :46-49 dropout_keep (keep iff u >= p). */
VO_EXPORT uint64_t vo_position_hash(uint64_t seed, uint64_t b, uint64_t h, uint64_t row, uint64_t col) {
    uint64_t s = vo_hash_combine(seed, 0x64726f70ull); /* "drop" stream tag */
    s = vo_hash_combine(s, b);
    s = vo_hash_combine(s, h);
    s = vo_hash_combine(s, row);
    s = vo_hash_combine(s, col);
    return s;
}

VO_EXPORT int vo_dropout_keep(uint64_t seed, uint64_t b, uint64_t h, uint64_t row, uint64_t col, float p) {
    if (p <= 0.0f) return 1;
    return vo_bits_to_unit(vo_position_hash(seed, b, h, row, col)) >= (double)p;
}

/* ------------------------------------------------------------- binary16 -- */

static inline uint32_t f2u(float x) { uint32_t u; memcpy(&u, &x, 4); return u; }
static inline float u2f(uint32_t u) { float x; memcpy(&x, &u, 4); return x; }

/* src/half.cpp:5-44: RNE narrowing, overflow -> inf, subnormals kept, NaN payload kept. */
VO_EXPORT uint16_t vo_f32_to_f16(float x) {
    const uint32_t f = f2u(x);
    const uint16_t sign = (uint16_t)((f >> 16) & 0x8000u);
    const uint32_t exp = (f >> 23) & 0xffu;
    const uint32_t mant = f & 0x007fffffu;
    if (exp == 0xffu) {
        if (mant == 0) return (uint16_t)(sign | 0x7c00u);
        uint32_t payload = mant >> 13;
        if (payload == 0) payload = 0x200u;
        return (uint16_t)(sign | 0x7c00u | payload);
    }
    const int e = (int)exp - 127 + 15;
    if (e >= 31) return (uint16_t)(sign | 0x7c00u);
    if (e <= 0) {
        const int shift = 14 - e;
        if (shift > 24) return sign;
        const uint32_t m = mant | 0x00800000u;
        const uint32_t q = m >> shift;
        const uint32_t rem = m & ((1u << shift) - 1u);
        const uint32_t half = 1u << (shift - 1);
        uint32_t r = q;
        if (rem > half || (rem == half && (q & 1u))) ++r;
        return (uint16_t)(sign | r);
    }
    uint32_t out = ((uint32_t)e << 10) | (mant >> 13);
    const uint32_t rem = mant & 0x1fffu;
    if (rem > 0x1000u || (rem == 0x1000u && (out & 1u))) ++out;
    return (uint16_t)(sign | out);
}

/* src/half.cpp:46-65: exact widening. */
VO_EXPORT float vo_f16_to_f32(uint16_t h) {
    const uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
    const uint32_t exp = (h >> 10) & 0x1fu;
    uint32_t mant = h & 0x3ffu;
    if (exp == 0x1fu) return u2f(sign | 0x7f800000u | (mant << 13));
    if (exp == 0) {
        if (mant == 0) return u2f(sign);
        int e = -14;
        while ((mant & 0x400u) == 0) { mant <<= 1; --e; }
        mant &= 0x3ffu;
        return u2f(sign | ((uint32_t)(e + 127) << 23) | (mant << 13));
    }
    return u2f(sign | ((exp - 15 + 127) << 23) | (mant << 13));
}

/* bfloat16: RNE narrowing (NaN quieted).  No reference counterpart;
 * it is the same rounding cvt.rn.bf16x2.f32 performs on the device. */
VO_EXPORT uint16_t vo_f32_to_bf16(float x) {
    uint32_t u = f2u(x);
    if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40u);
    u += 0x7fffu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}

VO_EXPORT float vo_bf16_to_f32(uint16_t h) { return u2f((uint32_t)h << 16); }

static inline float widen16(uint16_t h, int bf16) { return bf16 ? vo_bf16_to_f32(h) : vo_f16_to_f32(h); }

/* include/vattn/workload.hpp:10-17: normal_tensor_f16(seed, stream, dims).
 * bf16 != 0 rounds the same binary32 normals to bfloat16 instead. */
VO_EXPORT void vo_normal_tensor16(uint64_t seed, uint64_t stream, uint64_t count, int bf16,
                                  uint16_t* out) {
    const uint64_t base = vo_hash_combine(seed, stream);
    for (uint64_t i = 0; i < count; ++i) {
        const float x = vo_normal_at(base, i);
        out[i] = bf16 ? vo_f32_to_bf16(x) : vo_f32_to_f16(x);
    }
}

VO_EXPORT void vo_widen16(const uint16_t* in, uint64_t count, int bf16, double* out) {
    for (uint64_t i = 0; i < count; ++i) out[i] = (double)widen16(in[i], bf16);
}

/* ------------------------------------------------------ binary64 oracle -- */

/* src/reference.cpp:26-80 (dropout_p = 0): dense softmax attention in binary64.
 * scale <= 0 picks 1/sqrt(d) in binary32 first, like AttnConfig::scale()
 * (src/attention_forward.cpp:42-45). */
static double cfg_scale(float scale, int d) {
    return scale > 0.0f ? (double)scale : (double)(1.0f / sqrtf((float)d));
}

VO_EXPORT void vo_attention_ref_dropout(int B, int H, int N, int d, int causal, float scale_f,
                                        float p_drop, uint64_t seed, const double* q, const double* k,
                                        const double* v, double* out, double* lse);

VO_EXPORT void vo_attention_ref(int B, int H, int N, int d, int causal, float scale_f,
                                const double* q, const double* k, const double* v,
                                double* out, double* lse) {
    vo_attention_ref_dropout(B, H, N, d, causal, scale_f, 0.0f, 0, q, k, v, out, lse);
}

/* src/reference.cpp:26-80 including the dropout branch (:66-69). */
VO_EXPORT void vo_attention_ref_dropout(int B, int H, int N, int d, int causal, float scale_f,
                                        float p_drop, uint64_t seed, const double* q, const double* k,
                                        const double* v, double* out, double* lse) {
    const double scale = cfg_scale(scale_f, d);
    const double inv_keep = 1.0 / (1.0 - (double)p_drop);
    double* s = (double*)malloc(sizeof(double) * (size_t)N);
    double* p = (double*)malloc(sizeof(double) * (size_t)N);
    for (int bh = 0; bh < B * H; ++bh) {
        const double* Q = q + (size_t)bh * N * d;
        const double* K = k + (size_t)bh * N * d;
        const double* V = v + (size_t)bh * N * d;
        for (int i = 0; i < N; ++i) {
            double m = -INFINITY;
            for (int j = 0; j < N; ++j) {
                if (causal && j > i) {
                    s[j] = -INFINITY;
                } else {
                    double dot = 0.0;
                    for (int e = 0; e < d; ++e) dot += Q[(size_t)i * d + e] * K[(size_t)j * d + e];
                    s[j] = scale * dot;
                }
                m = fmax(m, s[j]);
            }
            double l = 0.0;
            for (int j = 0; j < N; ++j) l += s[j] == -INFINITY ? 0.0 : exp(s[j] - m);
            lse[(size_t)bh * N + i] = m + log(l);
            for (int j = 0; j < N; ++j) {
                p[j] = s[j] == -INFINITY ? 0.0 : exp(s[j] - m) / l;
                if (p_drop > 0.0f)
                    p[j] = vo_dropout_keep(seed, (uint64_t)(bh / H), (uint64_t)(bh % H), (uint64_t)i, (uint64_t)j, p_drop)
                               ? p[j] * inv_keep : 0.0;
            }
            for (int e = 0; e < d; ++e) {
                double acc = 0.0;
                for (int j = 0; j < N; ++j) acc += p[j] * V[(size_t)j * d + e];
                out[((size_t)bh * N + i) * d + e] = acc;
            }
        }
    }
    free(s);
    free(p);
}

/* src/reference.cpp:82-167 (dropout_p = 0): analytic gradients in binary64.
 *   dV = P^T dO, dP = dO V^T, dS = P o (dP - rowsum(dP o P)) * scale,
 *   dQ = dS K, dK = dS^T Q. */
VO_EXPORT void vo_attention_grad_ref_dropout(int B, int H, int N, int d, int causal, float scale_f,
                                             float p_drop, uint64_t seed, const double* q, const double* k,
                                             const double* v, const double* dout, double* dq, double* dk,
                                             double* dv);

VO_EXPORT void vo_attention_grad_ref(int B, int H, int N, int d, int causal, float scale_f,
                                     const double* q, const double* k, const double* v,
                                     const double* dout, double* dq, double* dk, double* dv) {
    vo_attention_grad_ref_dropout(B, H, N, d, causal, scale_f, 0.0f, 0, q, k, v, dout, dq, dk, dv);
}

/* src/reference.cpp:82-167 including the dropout factor matrix D (:118-121). */
VO_EXPORT void vo_attention_grad_ref_dropout(int B, int H, int N, int d, int causal, float scale_f,
                                             float p_drop, uint64_t seed, const double* q, const double* k,
                                             const double* v, const double* dout, double* dq, double* dk,
                                             double* dv) {
    const double scale = cfg_scale(scale_f, d);
    const double inv_keep = 1.0 / (1.0 - (double)p_drop);
    double* drop = (double*)malloc(sizeof(double) * (size_t)N * N);
    const size_t nn = (size_t)N * N;
    double* p = (double*)malloc(sizeof(double) * nn);
    double* dp = (double*)malloc(sizeof(double) * nn);
    double* ds = (double*)malloc(sizeof(double) * nn);
    double* s = (double*)malloc(sizeof(double) * (size_t)N);
    for (int bh = 0; bh < B * H; ++bh) {
        const size_t off = (size_t)bh * N * d;
        const double *Q = q + off, *K = k + off, *V = v + off, *DO = dout + off;
        for (int i = 0; i < N; ++i) {
            double m = -INFINITY;
            for (int j = 0; j < N; ++j) {
                if (causal && j > i) {
                    s[j] = -INFINITY;
                } else {
                    double dot = 0.0;
                    for (int e = 0; e < d; ++e) dot += Q[(size_t)i * d + e] * K[(size_t)j * d + e];
                    s[j] = scale * dot;
                }
                m = fmax(m, s[j]);
            }
            double l = 0.0;
            for (int j = 0; j < N; ++j) l += s[j] == -INFINITY ? 0.0 : exp(s[j] - m);
            for (int j = 0; j < N; ++j) {
                p[(size_t)i * N + j] = s[j] == -INFINITY ? 0.0 : exp(s[j] - m) / l;
                drop[(size_t)i * N + j] =
                    p_drop > 0.0f ? (vo_dropout_keep(seed, (uint64_t)(bh / H), (uint64_t)(bh % H), (uint64_t)i,
                                                     (uint64_t)j, p_drop) ? inv_keep : 0.0)
                                  : 1.0;
            }
        }
        for (int j = 0; j < N; ++j)
            for (int e = 0; e < d; ++e) {
                double acc = 0.0;
                for (int i = 0; i < N; ++i) acc += drop[(size_t)i * N + j] * p[(size_t)i * N + j] * DO[(size_t)i * d + e];
                dv[off + (size_t)j * d + e] = acc;
            }
        for (int i = 0; i < N; ++i) {
            for (int j = 0; j < N; ++j) {
                double acc = 0.0;
                for (int e = 0; e < d; ++e) acc += DO[(size_t)i * d + e] * V[(size_t)j * d + e];
                dp[(size_t)i * N + j] = drop[(size_t)i * N + j] * acc;
            }
            double dpsum = 0.0;
            for (int j = 0; j < N; ++j) dpsum += dp[(size_t)i * N + j] * p[(size_t)i * N + j];
            for (int j = 0; j < N; ++j)
                ds[(size_t)i * N + j] = p[(size_t)i * N + j] * (dp[(size_t)i * N + j] - dpsum) * scale;
        }
        for (int i = 0; i < N; ++i)
            for (int e = 0; e < d; ++e) {
                double acc = 0.0;
                for (int j = 0; j < N; ++j) acc += ds[(size_t)i * N + j] * K[(size_t)j * d + e];
                dq[off + (size_t)i * d + e] = acc;
            }
        for (int j = 0; j < N; ++j)
            for (int e = 0; e < d; ++e) {
                double acc = 0.0;
                for (int i = 0; i < N; ++i) acc += ds[(size_t)i * N + j] * Q[(size_t)i * d + e];
                dk[off + (size_t)j * d + e] = acc;
            }
    }
    free(p);
    free(dp);
    free(ds);
    free(s);
    free(drop);
}

/* ------------------------------------------- fused FP32-ACC forward ---- */

/* The FP32-ACC arithmetic contract of one C element of a tile GEMM
 * (src/tile_pipeline.cpp:33-49 -> src/warp_mma.cpp:162-202 -> src/half.cpp:67-77):
 * for k4 ascending, acc = acc + (((0 + a0 b0) + a1 b1) + a2 b2) + a3 b3 with
 * every product exact in binary32 and each add rounded to binary32. */
static inline float dot_fp32acc(float acc, const float* a, const float* b, int bstride, int kdim) {
    for (int k4 = 0; k4 < kdim / 4; ++k4) {
        float s = 0.0f;
        for (int kk = 0; kk < 4; ++kk) s += a[k4 * 4 + kk] * b[(size_t)(k4 * 4 + kk) * bstride];
        acc = acc + s;
    }
    return acc;
}

/* src/attention_forward.cpp:191-227 + run_forward_unit :110-187, FP32-ACC,
 * dropout_p = 0, tiles br x bc (reference defaults 64 x 64).  q/k/v are
 * binary16 bit patterns; out receives binary16 bit patterns, lse binary32.
 * Returns 0, or -1 for a config AttnConfig::validate() rejects
 * (src/attention_forward.cpp:31-40), or -2 for a fully masked row
 * (src/online_softmax.cpp:81-82). */
VO_EXPORT int vo_forward_fused_fp32acc_dropout(int B, int H, int N, int d, int br, int bc, int causal,
                                               float scale_f, float p_drop, uint64_t seed, const uint16_t* q,
                                               const uint16_t* k, const uint16_t* v, uint16_t* out, float* lse);

VO_EXPORT int vo_forward_fused_fp32acc(int B, int H, int N, int d, int br, int bc, int causal,
                                       float scale_f, const uint16_t* q, const uint16_t* k,
                                       const uint16_t* v, uint16_t* out, float* lse) {
    return vo_forward_fused_fp32acc_dropout(B, H, N, d, br, bc, causal, scale_f, 0.0f, 0, q, k, v, out, lse);
}

/* ... with the dropout step of src/attention_forward.cpp:77-106 (applied to the
 * binary16 P fragments: kept weights f16(f16(P) * (1/(1-p))), dropped ones 0). */
VO_EXPORT int vo_forward_fused_fp32acc_dropout(int B, int H, int N, int d, int br, int bc, int causal,
                                               float scale_f, float p_drop, uint64_t seed, const uint16_t* q,
                                               const uint16_t* k, const uint16_t* v, uint16_t* out, float* lse) {
    if (!(p_drop >= 0.0f && p_drop < 1.0f)) return -1;
    const float inv_keep = 1.0f / (1.0f - p_drop);
    if (B < 1 || H < 1 || N <= 0 || d <= 0 || br <= 0 || br % 8 || bc <= 0 || bc % 8 || d % 4 ||
        N % br || N % bc)
        return -1;
    const float scale = scale_f > 0.0f ? scale_f : 1.0f / sqrtf((float)d);
    float* qt = (float*)malloc(sizeof(float) * (size_t)br * d);
    float* kT = (float*)malloc(sizeof(float) * (size_t)d * bc); /* K tile transposed: [d][bc] */
    float* vt = (float*)malloc(sizeof(float) * (size_t)bc * d); /* [bc][d] */
    float* s = (float*)malloc(sizeof(float) * (size_t)br * bc);
    float* p16 = (float*)malloc(sizeof(float) * (size_t)br * bc); /* P narrowed once, widened */
    float* o = (float*)malloc(sizeof(float) * (size_t)br * d);
    float* m = (float*)malloc(sizeof(float) * (size_t)br);
    float* l = (float*)malloc(sizeof(float) * (size_t)br);
    int rc = 0;
    for (int bh = 0; bh < B * H && rc == 0; ++bh) {
        const size_t off = (size_t)bh * N * d;
        for (int qb = 0; qb < N / br && rc == 0; ++qb) {
            const int row0 = qb * br;
            for (int i = 0; i < br; ++i)
                for (int e = 0; e < d; ++e) qt[(size_t)i * d + e] = vo_f16_to_f32(q[off + (size_t)(row0 + i) * d + e]);
            for (size_t x = 0; x < (size_t)br * d; ++x) o[x] = 0.0f;
            for (int i = 0; i < br; ++i) { m[i] = -INFINITY; l[i] = 0.0f; }
            for (int kb = 0; kb < N / bc; ++kb) {
                const int col0 = kb * bc;
                if (causal && col0 > row0 + br - 1) break; /* :128 */
                for (int j = 0; j < bc; ++j)
                    for (int e = 0; e < d; ++e) {
                        kT[(size_t)e * bc + j] = vo_f16_to_f32(k[off + (size_t)(col0 + j) * d + e]);
                        vt[(size_t)j * d + e] = vo_f16_to_f32(v[off + (size_t)(col0 + j) * d + e]);
                    }
                /* S = Q K^T (:132-133), x scale (:138-139), diagonal -inf (:140-144). */
                for (int i = 0; i < br; ++i)
                    for (int j = 0; j < bc; ++j) {
                        float acc = dot_fp32acc(0.0f, qt + (size_t)i * d, kT + j, bc, d);
                        acc *= scale;
                        if (causal && col0 + bc - 1 > row0 && col0 + j > row0 + i) acc = -INFINITY;
                        s[(size_t)i * bc + j] = acc;
                    }
                /* softmax_block_update (src/online_softmax.cpp:21-62) + rescale_acc (:53-72). */
                for (int i = 0; i < br; ++i) {
                    float bmax = -INFINITY;
                    for (int j = 0; j < bc; ++j) {
                        const float x = s[(size_t)i * bc + j];
                        if (isnan(x)) { rc = -2; break; }
                        if (bmax < x) bmax = x; /* std::max(block_max, s) */
                    }
                    const float m_old = m[i];
                    const float m_new = m_old > bmax ? m_old : bmax;
                    if (m_new == -INFINITY) {
                        for (int j = 0; j < bc; ++j) p16[(size_t)i * bc + j] = 0.0f;
                        continue; /* rescale stays 1 */
                    }
                    const float resc = m_old == -INFINITY ? 1.0f : expf(m_old - m_new);
                    float bsum = 0.0f;
                    for (int j = 0; j < bc; ++j) {
                        const float x = s[(size_t)i * bc + j];
                        const float w = x == -INFINITY ? 0.0f : expf(x - m_new);
                        bsum += w;
                        float pw = vo_f16_to_f32(vo_f32_to_f16(w)); /* :163-167 */
                        if (p_drop > 0.0f)
                            pw = vo_dropout_keep(seed, (uint64_t)(bh / H), (uint64_t)(bh % H), (uint64_t)(row0 + i),
                                                 (uint64_t)(col0 + j), p_drop)
                                     ? vo_f16_to_f32(vo_f32_to_f16(pw * inv_keep))
                                     : 0.0f;
                        p16[(size_t)i * bc + j] = pw;
                    }
                    l[i] = l[i] * resc + bsum;
                    m[i] = m_new;
                    for (int e = 0; e < d; ++e) o[(size_t)i * d + e] *= resc;
                }
                if (rc) break;
                /* O += P V (:171-172), same FP32-ACC contract with K-dim = bc. */
                for (int i = 0; i < br; ++i)
                    for (int e = 0; e < d; ++e)
                        o[(size_t)i * d + e] = dot_fp32acc(o[(size_t)i * d + e], p16 + (size_t)i * bc, vt + e, d, bc);
            }
            if (rc) break;
            /* softmax_finalize (src/online_softmax.cpp:75-87); O = f16(acc * inv) (:179). */
            for (int i = 0; i < br; ++i) {
                if (!(l[i] > 0.0f)) { rc = -2; break; }
                const float inv = 1.0f / l[i];
                lse[(size_t)bh * N + row0 + i] = m[i] + logf(l[i]);
                for (int e = 0; e < d; ++e)
                    out[off + (size_t)(row0 + i) * d + e] = vo_f32_to_f16(o[(size_t)i * d + e] * inv);
            }
        }
    }
    free(qt); free(kT); free(vt); free(s); free(p16); free(o); free(m); free(l);
    return rc;
}

/* src/attention_backward.cpp:44-57: D_i = sum_j f32(dO_ij) * f32(O_ij), sequential binary32. */
VO_EXPORT void vo_compute_dpsum(int B, int H, int N, int d, int bf16, const uint16_t* dout,
                                const uint16_t* o, float* dpsum) {
    for (size_t r = 0; r < (size_t)B * H * N; ++r) {
        float s = 0.0f;
        for (int e = 0; e < d; ++e) s += widen16(dout[r * d + e], bf16) * widen16(o[r * d + e], bf16);
        dpsum[r] = s;
    }
}

/* ------------------------------------------------------------ metrics --- */

/* src/reference.cpp:186-210: rel = |t - r| / max(|r|, 1e-6). out = {mean_rel, max_rel, mean_abs, max_abs}. */
VO_EXPORT void vo_error_metrics(const double* test, const double* ref, uint64_t n, double* out4) {
    double mr = 0, xr = 0, ma = 0, xa = 0;
    for (uint64_t i = 0; i < n; ++i) {
        const double a = fabs(test[i] - ref[i]);
        const double r = a / fmax(fabs(ref[i]), 1e-6);
        ma += a; mr += r;
        if (a > xa) xa = a;
        if (r > xr) xr = r;
    }
    out4[0] = mr / (double)n; out4[1] = xr; out4[2] = ma / (double)n; out4[3] = xa;
}

/* src/reference.cpp:212-222 */
VO_EXPORT double vo_frobenius_rel(const double* test, const double* ref, uint64_t n) {
    double num = 0, den = 0;
    for (uint64_t i = 0; i < n; ++i) {
        const double dv = test[i] - ref[i];
        num += dv * dv;
        den += ref[i] * ref[i];
    }
    return den == 0.0 ? sqrt(num) : sqrt(num / den);
}
