/*
 * vattn_b200_traditional.h -- the unfused "traditional" attention forward on B200,
 * the comparator the paper measures the fused kernel against.
 *
 *   mha_forward_traditional  replaces vattn::forward_traditional
 *                            (proj/include/vattn/attention.hpp:56-60,
 *                             proj/src/attention_forward.cpp:229-310)
 *
 * Three passes through HBM, exactly the reference's structure (5 matrix-pass reads,
 * 3 writes): S = Q K^T materialised in binary32 (cuBLAS strided-batched GEMM, fp32
 * accumulate), a full-row softmax kernel (scale, top-left causal mask, natural exp,
 * lse = m + ln l, P = f16(w / l) -- normalised before P V, dropout with the
 * reference's keep bits and 1/(1-p)), and O = P V (cuBLAS, fp32 accumulate, one
 * rounding).  Every key tile is computed and masked (no causal tile skipping), as in
 * the reference.  It lives in its own library (libvattn_b200_traditional.so) so the
 * fused path never links cuBLAS.
 */
#ifndef VATTN_B200_TRADITIONAL_H
#define VATTN_B200_TRADITIONAL_H

#include "vattn_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Device workspace for S (binary32, B*H*N*N) and P (16-bit, B*H*N*N); 0 on bad cfg. */
size_t mha_forward_traditional_workspace_bytes(const vattn_config* cfg);

/* O, lse of the three-pass forward (any head_dim with head_dim % 4 == 0, as the reference).  Device pointers, stream ordered.  (The
 * reference's fully-masked-row domain_error, attention_forward.cpp:279-280, cannot
 * occur: a top-left causal row always sees key 0.) */
int mha_forward_traditional(const vattn_config* cfg, const void* q, const void* k, const void* v,
                            void* o, float* lse, void* workspace, size_t workspace_bytes,
                            void* stream);

const char* vattn_traditional_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* VATTN_B200_TRADITIONAL_H */
