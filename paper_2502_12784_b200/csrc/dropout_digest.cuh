// dropout_digest.cuh -- the reference's dropout mask digest on the device.
//
// vattn::ForwardOutput::mask_digest / GradOutputs::mask_digest (reference
// proj/include/vattn/attention.hpp:32, rng.hpp:26-29) is an order-independent sum of
// dropout_digest_term(seed, b, h, row, col, keep) = mix64(position_hash ^ (keep ?
// "keep" : 0)) over every mask position the pass consumed: all positions of the
// visited (query tile, key tile) pairs for the fused passes (causal: key tile kt is
// visited by query tile qt iff kt*Bc <= qt*Br + Br - 1, attention_forward.cpp:128 /
// attention_backward.cpp:125), all N x N positions for the traditional pass.  The sum
// is taken modulo 2^64 with 64-bit atomics: integer addition is associative and
// commutative, so the result is bit-identical to the reference's whatever the order.
#pragma once

#include "sm100_ptx.cuh"

namespace vattn_sm100 {

__global__ void __launch_bounds__(256) dropout_digest_kernel(unsigned long long* out, uint64_t seed, int H, int bh_off,
                                                             int N, int br, int bc, int causal, uint64_t thresh) {
    __shared__ unsigned long long red[8];
    const int bh = blockIdx.y;
    const int qt = blockIdx.x;
    const int row0 = qt * br;
    const int cols = causal ? min(N, ((row0 + br - 1) / bc + 1) * bc) : N;
    const uint64_t base = drop_bh_base(seed, (bh + bh_off) / H, (bh + bh_off) % H);
    unsigned long long acc = 0;
    for (int i = 0; i < br && row0 + i < N; ++i) {
        const DropRow r = drop_row(base, row0 + i);
        for (int j = threadIdx.x; j < cols; j += blockDim.x) {
            const uint64_t ph = mix64(r.s ^ (static_cast<uint64_t>(j) + r.k));
            const bool keep = (ph >> 11) >= thresh;
            acc += mix64(ph ^ (keep ? 0x6b656570ull : 0ull));
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        atomicAdd(out, t);
    }
}

}  // namespace vattn_sm100
