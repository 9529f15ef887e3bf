/*
 * vattn_b200.h -- C ABI of the B200 (sm_100a) fused multi-head-attention
 * training path.  This is the drop-in boundary for the reference's operator
 * API (arxiv 2502.12784 "SparkAttention", reference tree /root/reference/proj):
 *
 *   mha_forward   replaces vattn::forward_fused
 *                 (proj/include/vattn/attention.hpp:51-52, proj/src/attention_forward.cpp:191-227)
 *   mha_backward  replaces vattn::backward_fused
 *                 (proj/include/vattn/backward.hpp:56-59, proj/src/attention_backward.cpp:59-219)
 *                 including compute_dpsum (backward.hpp:43, attention_backward.cpp:44-57)
 *                 and the DqAccumulator master buffer (backward.hpp:16-40)
 *   vattn_config  mirrors vattn::AttnConfig (proj/include/vattn/attention.hpp:11-26)
 *
 * Conventions
 *   - Tensors are device pointers, caller owned, dense row-major [B, H, N, d]
 *     (proj/include/vattn/tensor.hpp:45-50); lse is [B, H, N] binary32 in
 *     natural-log units (attention.hpp:30, online_softmax.cpp:84).
 *   - 16-bit element type is fp16 (VATTN_F16, the reference's Half) or bf16.
 *   - Calls are stream ordered and asynchronous; `stream` is a cudaStream_t
 *     (NULL = legacy default stream).  Safe to call concurrently from several
 *     host threads on different streams.
 *   - Every call returns a vattn_status; on failure vattn_last_error() returns a
 *     thread-local message.  VATTN_EINVAL corresponds to the reference's
 *     std::invalid_argument, VATTN_EDOMAIN to std::domain_error (a query row with
 *     a NaN / +inf score or an empty softmax sum, online_softmax.cpp:33-34, 81-82):
 *     the synchronous host entry points return it; the asynchronous device entry
 *     points report it through the optional status word of mha_forward_ex.
 *   - head_dim must be 64 or 128 at this boundary (the C++ layer
 *     include/vattn_b200/mha.hpp zero-pads other head dims); any seq_len >= 1.
 *   - No CPU fallback: when the sm_100a kernels cannot run, calls fail with
 *     VATTN_ECUDA / VATTN_EUNSUPPORTED.
 *   - Dropout (dropout_p > 0) follows the reference exactly: the same stateless
 *     SplitMix64 position hash decides every keep bit (proj/src/rng.cpp:35-49),
 *     the forward scales the 16-bit P by 1/(1-p) after its first rounding
 *     (attention_forward.cpp:77-106) and the backward replays the mask
 *     (attention_backward.cpp:145-182).  The reference's mask_digest is a
 *     tiling-dependent test hook and is not produced.
 *
 * Divergence from the reference (documented): the backward takes O as an
 * input (D = rowsum(dO o O) is computed from it) instead of re-running the
 * forward internally (attention_backward.cpp:91-104); the C++ layer provides
 * the reference's six-argument overload by calling mha_forward first.
 */
#ifndef VATTN_B200_H
#define VATTN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VATTN_B200_ABI_VERSION 4

typedef enum vattn_status {
    VATTN_OK = 0,
    VATTN_EINVAL = 1,       /* bad config / shape / pointer  (std::invalid_argument) */
    VATTN_EDOMAIN = 2,      /* numerical domain error        (std::domain_error)     */
    VATTN_EUNSUPPORTED = 3, /* valid for the reference, not implemented here         */
    VATTN_ECUDA = 4         /* CUDA runtime / launch failure, or no sm_100 device     */
} vattn_status;

typedef enum vattn_dtype { VATTN_F16 = 0, VATTN_BF16 = 1 } vattn_dtype;

typedef struct vattn_config {
    int32_t batch;          /* B >= 1                                              */
    int32_t heads;          /* H >= 1                                              */
    int32_t seq_len;        /* N >= 1                                              */
    int32_t head_dim;       /* d in {64, 128}                                      */
    int32_t causal;         /* top-left causal mask: key j visible iff j <= i      */
    float softmax_scale;    /* <= 0 selects 1/sqrt(head_dim) (AttnConfig::scale)   */
    int32_t dtype;          /* vattn_dtype                                         */
    float dropout_p;        /* in [0, 1); 0 = no dropout (AttnConfig::dropout_p)   */
    uint64_t seed;          /* dropout seed: keep masks are bit-identical to the
                               reference's dropout_keep(seed, b, h, row, col, p)   */
    int32_t bh_offset;      /* (batch, head) slab of the problem this call runs:   */
    int32_t bh_count;       /* units [bh_offset, bh_offset + bh_count) of the      */
                            /* flattened b*H + h axis; the tensor pointers point at
                               unit bh_offset.  bh_count = 0 selects the whole
                               problem (bh_offset must then be 0).  Units are
                               independent, so a slab's outputs are bit-identical
                               to the same units of a whole-problem call (dropout
                               masks use the global (b, h)).  This is how ranks
                               shard the path and how the host API
                               pipelines PCIe copies against compute.             */
} vattn_config;

/* O = softmax(Q K^T * scale [+ causal mask]) V ;  lse = logsumexp per query row. */
int mha_forward(const vattn_config* cfg, const void* q, const void* k, const void* v, void* o,
                float* lse, void* stream);

/* mha_forward with the two optional extras (replaces the reference's forward_fused
 * checks, attention_forward.cpp:191-227 -> online_softmax.cpp:33-34, 81-82):
 *   drop_mask  as mha_forward_dropout_mask (NULL = do not keep the keep bits);
 *   status     device word (4-byte aligned, zeroed by the caller) into which the
 *              kernel ORs VATTN_DOMAIN_ROW when any query row had a NaN or +inf
 *              score or an empty softmax sum (l == 0) -- the rows for which the
 *              reference throws std::domain_error.  NULL = unchecked.  Reading it
 *              after the stream synchronises is the caller's domain check. */
#define VATTN_DOMAIN_ROW 1u
int mha_forward_ex(const vattn_config* cfg, const void* q, const void* k, const void* v, void* o, float* lse,
                   void* drop_mask, unsigned int* status, void* stream);

/* Bytes of device workspace mha_backward needs for `cfg` (0 on invalid cfg). */
size_t mha_backward_workspace_bytes(const vattn_config* cfg);

/* Bytes of workspace mha_backward_dropout_mask needs: the caller's keep-bit mask
 * replaces the workspace's own mask region (equal to mha_backward_workspace_bytes
 * without dropout). */
size_t mha_backward_workspace_bytes_mask(const vattn_config* cfg);

/* dQ, dK, dV of the forward above given dO, O and lse.  `workspace` must hold
 * mha_backward_workspace_bytes(cfg) bytes (256-byte aligned); its contents on
 * entry are irrelevant.  All three gradients are bit-reproducible run to run
 * (no atomics; dQ is accumulated over key tiles in a fixed order). */
int mha_backward(const vattn_config* cfg, const void* q, const void* k, const void* v,
                 const void* o, const void* dout, const float* lse, void* dq, void* dk, void* dv,
                 void* workspace, size_t workspace_bytes, void* stream);

/* Dropout keep bits kept from the forward for the backward (optional fast path).
 * mha_dropout_mask_bytes(cfg): size of the keep-bit mask, 2*B*H*Npad*Npad/8 bytes with
 * Npad = N rounded up to 128: a query-major copy [unit][query][Npad/32] (bit = key)
 * followed by a key-major copy [unit][key][Npad/32] (bit = query).  0 when
 * dropout_p == 0, cfg is invalid, or masks are disabled with VATTN_DROP_MASK=0 (then
 * every kernel hashes the bits in place).
 * mha_forward_dropout_mask: mha_forward that first hashes the keep bits of every
 * visited position into `drop_mask` (one integer-bound kernel, off the softmax's
 * critical path) and then reads them.
 * mha_backward_dropout_mask: mha_backward that reads those bits instead of hashing
 * the positions again (same results, bit for bit; `drop_mask` must come from
 * mha_forward_dropout_mask with the same cfg).  Both require dropout_p > 0 and a
 * 256-byte aligned mask.  Without them the backward hashes the keep bits itself. */
size_t mha_dropout_mask_bytes(const vattn_config* cfg);
int mha_forward_dropout_mask(const vattn_config* cfg, const void* q, const void* k, const void* v, void* o,
                             float* lse, void* drop_mask, void* stream);
int mha_backward_dropout_mask(const vattn_config* cfg, const void* q, const void* k, const void* v,
                              const void* o, const void* dout, const float* lse, const void* drop_mask,
                              void* dq, void* dk, void* dv, void* workspace, size_t workspace_bytes,
                              void* stream);

/* D = rowsum(dO o O) per query row ([B, H, N] binary32, products widened before the
 * sum) -- vattn::compute_dpsum (proj/include/vattn/backward.hpp:43,
 * attention_backward.cpp:44-57), the backward's preprocessing pass on its own. */
int mha_dpsum(const vattn_config* cfg, const void* o, const void* dout, float* d_rows, void* stream);

/* The reference's dropout mask digest (ForwardOutput/GradOutputs::mask_digest,
 * attention.hpp:32): the order-independent 64-bit sum of dropout_digest_term over
 * the mask positions a pass with (tile_rows x tile_cols) tiles consumes -- the fused
 * passes' visited tile pairs (tile_rows = tile_cols = N, causal = 0 gives the
 * traditional pass's N x N).  Written to the device word `digest`; 0 when
 * dropout_p == 0.  Bit-identical to the reference's value. */
int vattn_dropout_digest(const vattn_config* cfg, int tile_rows, int tile_cols, unsigned long long* digest,
                         void* stream);

/* ---- host-buffer entry points (the reference's synchronous host API) ------
 * Same math as the device entry points, but every tensor is a HOST pointer
 * (pinned memory gives full copy/compute overlap; pageable memory works but
 * the copies serialise).  The call splits the (b, h) units into slabs and
 * pipelines them over three streams -- H2D of slab c+1, the kernels of slab c
 * (on `stream`), D2H of slab c-1 -- so PCIe traffic in both directions overlaps
 * the sm_100a kernels.  Device staging comes from a library-owned stream-ordered
 * pool.  Synchronous: outputs are valid when the call returns (like
 * vattn::forward_fused / backward_fused).  Results are bit-identical to the
 * device entry points. */

/* vattn::forward_fused on host buffers: O, lse.  Returns VATTN_EDOMAIN where the
 * reference throws std::domain_error (see mha_forward_ex). */
int mha_forward_host(const vattn_config* cfg, const void* q, const void* k, const void* v, void* o,
                     float* lse, void* stream);

/* vattn::backward_fused on host buffers (O given, see the divergence note). */
int mha_backward_host(const vattn_config* cfg, const void* q, const void* k, const void* v,
                      const void* o, const void* dout, const float* lse, void* dq, void* dk,
                      void* dv, void* stream);

/* One attention training step on host buffers: forward then backward with Q, K,
 * V and dO crossing PCIe once, O, lse, dQ, dK, dV returned.  VATTN_EDOMAIN as
 * mha_forward_host. */
int mha_step_host(const vattn_config* cfg, const void* q, const void* k, const void* v,
                  const void* dout, void* o, float* lse, void* dq, void* dk, void* dv,
                  void* stream);

/* Thread-local description of the last failure on this thread ("" if none). */
const char* vattn_last_error(void);

/* VATTN_B200_ABI_VERSION of the loaded library. */
int vattn_abi_version(void);

/* Number of kernels the last successful call on this thread launched. */
int vattn_last_launch_count(void);

/* TMA descriptor cache counters (tensor maps are cached per pointer, shape and
 * dtype): lookups served from the cache and maps encoded. */
void vattn_map_cache_stats(long long* hits, long long* misses);

/* Measurement hooks (bench / roofline only; off by default).  When enabled,
 * every call records CUDA events on its stream around the hot kernels;
 * vattn_profile_read(kind) synchronizes those events and returns the summed
 * kernel milliseconds and launch count of one kernel kind since the last
 * vattn_profile_enable(1).  Kinds: */
#define VATTN_KERNEL_FWD 0     /* fused forward                      */
#define VATTN_KERNEL_BWD_DKDV 1 /* backward, key-major dK / dV kernel */
#define VATTN_KERNEL_BWD_DQ 2   /* backward, query-major dQ kernel    */
#define VATTN_KERNEL_BWD_PRE 3  /* backward preprocess (D, lse2)      */
#define VATTN_KERNEL_DROPMASK 4 /* dropout keep-bit mask (both copies) */
void vattn_profile_enable(int on);
int vattn_profile_read(int kind, double* ms_total, int* launches);

#ifdef __cplusplus
}
#endif

#endif /* VATTN_B200_H */
