// capi_host.cu -- host-buffer entry points of the C ABI (include/vattn_b200.h):
// mha_forward_host, mha_backward_host, mha_step_host.
//
// The reference's operator API is synchronous and host-resident
// (vattn::forward_fused / backward_fused, proj/include/vattn/attention.hpp:51-52,
// proj/include/vattn/backward.hpp:56-59).  On B200 the kernels are ~50x faster
// than PCIe can feed them (C3: 4.4 ms of kernels vs ~1 GB of copies), so the
// host path is a copy-bound pipeline: the (b, h) units are cut into slabs and
//   in-stream      H2D of slab c+1
//   `stream`       the sm_100a kernels of slab c (vattn_config.bh_offset/count)
//   out-stream     D2H of slab c-1
// run concurrently; each direction of the link stays busy and the kernels hide
// underneath.  Slabs rotate through R device slots; a slot is refilled only
// after the D2H of its previous slab completed (one event wait covers every
// hazard: the slab's kernels precede its D2H on the out-stream).  Device
// staging comes from a library-owned stream-ordered memory pool (cached across
// calls, never the caller's allocator).  Units are independent and the kernels
// deterministic, so results are bit-identical to one whole-problem call.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/vattn_b200.h"

namespace {

thread_local std::string g_host_err;

struct Fail {
    int code;
};

void cu(cudaError_t e, const char* where) {
    if (e != cudaSuccess) {
        g_host_err = std::string(where) + ": " + cudaGetErrorString(e);
        throw Fail{VATTN_ECUDA};
    }
}

void chk(int rc, const char* where) {
    if (rc != VATTN_OK) {
        g_host_err = std::string(where) + ": " + vattn_last_error();
        throw Fail{rc};
    }
}

// Library-owned pool per device (release threshold = unlimited: staging
// buffers stay cached between calls instead of being returned at every sync).
cudaMemPool_t staging_pool(int dev) {
    static std::mutex mu;
    static cudaMemPool_t pools[64] = {};
    std::lock_guard<std::mutex> l(mu);
    if (!pools[dev]) {
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.handleTypes = cudaMemHandleTypeNone;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        cu(cudaMemPoolCreate(&pools[dev], &props), "cudaMemPoolCreate");
        uint64_t thr = UINT64_MAX;
        cu(cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &thr), "pool threshold");
    }
    return pools[dev];
}

// Copy streams per (thread, device): non-blocking, so they never serialise
// against the legacy default stream.
struct CopyStreams {
    cudaStream_t in = nullptr, out = nullptr;
};
CopyStreams copy_streams(int dev) {
    thread_local CopyStreams cs[64];
    if (!cs[dev].in) {
        cu(cudaStreamCreateWithFlags(&cs[dev].in, cudaStreamNonBlocking), "stream create");
        cu(cudaStreamCreateWithFlags(&cs[dev].out, cudaStreamNonBlocking), "stream create");
    }
    return cs[dev];
}

constexpr int kMaxT = 8;

// One host tensor of the pipeline: `unit` bytes per (b, h) unit.
struct HostT {
    const uint8_t* in = nullptr;  // host source (inputs)
    uint8_t* out = nullptr;       // host destination (outputs)
    size_t unit = 0;
};

struct Job {
    HostT in[kMaxT];
    int n_in = 0;
    HostT out[kMaxT];
    int n_out = 0;
    size_t ws_unit = 0;  // device scratch bytes per unit (backward workspace)
    // run the kernels of one slab: d_in[i] / d_out[i] point at the slot's buffers;
    // `status` is the call's device domain-error word (the forward ORs into it)
    int (*run)(const vattn_config* slab, void* const* d_in, void* const* d_out, void* ws, size_t ws_bytes,
               unsigned int* status, cudaStream_t s) = nullptr;
    bool check_domain = false;  // map a non-zero status word to VATTN_EDOMAIN
};

int units_of(const vattn_config* c) { return c->bh_count ? c->bh_count : c->batch * c->heads; }

// Slab size: every launch should still fill the GPU (one CTA per SM over the 128-row
// tiles of a head) while keeping >= 16 slabs for the copies to overlap.  Measured at
// C3 (64 units): 4 units per slab 12.05 ms per step, 5 units 13.6 ms, 2 units 12.4 ms,
// 1 unit 16.4 ms; a fourth staging slot changes nothing.
int slab_units(const vattn_config* c, int U) {
    static const int env = [] {  // tuning override: slabs per call
        const char* e = getenv("VATTN_HOST_SLABS");
        return e ? atoi(e) : 0;
    }();
    const int tiles = (c->seq_len + 127) / 128;
    const int fill = (148 + tiles - 1) / tiles;
    const int for_overlap = (U + 15) / 16;  // aim for >= 16 slabs
    if (env > 0) return std::max(1, (U + env - 1) / env);
    return std::max(1, std::min(U, std::max(fill, for_overlap)));
}

int run_pipeline(const vattn_config* cfg, const Job& job, cudaStream_t stream) {
    int dev = 0;
    cu(cudaGetDevice(&dev), "cudaGetDevice");
    const int U = units_of(cfg);
    const int cu_units = slab_units(cfg, U);
    const int n_slabs = (U + cu_units - 1) / cu_units;
    const int R = std::min(3, n_slabs);
    const CopyStreams cs = copy_streams(dev);
    cudaMemPool_t pool = staging_pool(dev);

    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    size_t slot_bytes = 0;
    for (int i = 0; i < job.n_in; ++i) slot_bytes += al(job.in[i].unit * cu_units);
    for (int i = 0; i < job.n_out; ++i) slot_bytes += al(job.out[i].unit * cu_units);
    // workspace: the largest over the full and the (smaller) last slab -- the backward's
    // dQ design is chosen from a slab's own unit count, so a short last slab may need
    // more than a full one (e.g. it falls under the dS materialisation cap)
    size_t ws_bytes = 0;
    if (job.ws_unit) {
        vattn_config sl = *cfg;
        sl.bh_count = cu_units;
        ws_bytes = mha_backward_workspace_bytes(&sl);
        const int last = U - (n_slabs - 1) * cu_units;
        if (last != cu_units) {
            sl.bh_count = last;
            ws_bytes = std::max(ws_bytes, mha_backward_workspace_bytes(&sl));
        }
    }
    slot_bytes += al(ws_bytes);

    uint8_t* base = nullptr;
    cu(cudaMallocFromPoolAsync(reinterpret_cast<void**>(&base), slot_bytes * R + 256, pool, stream), "staging alloc");
    unsigned int* status = reinterpret_cast<unsigned int*>(base + slot_bytes * R);
    unsigned int h_status = 0;
    cudaEvent_t ready, in_done[3], comp_done[3], out_done[3];
    cu(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming), "event");
    for (int r = 0; r < 3; ++r) {
        cu(cudaEventCreateWithFlags(&in_done[r], cudaEventDisableTiming), "event");
        cu(cudaEventCreateWithFlags(&comp_done[r], cudaEventDisableTiming), "event");
        cu(cudaEventCreateWithFlags(&out_done[r], cudaEventDisableTiming), "event");
    }
    int rc = VATTN_OK;
    try {
        // the staging buffers (and everything the caller queued) precede the copies
        cu(cudaMemsetAsync(status, 0, sizeof(unsigned int), stream), "status memset");
        cu(cudaEventRecord(ready, stream), "event record");
        cu(cudaStreamWaitEvent(cs.in, ready, 0), "wait");
        cu(cudaStreamWaitEvent(cs.out, ready, 0), "wait");
        for (int c = 0; c < n_slabs; ++c) {
            const int r = c % R;
            const int u0 = c * cu_units;
            const int nu = std::min(cu_units, U - u0);
            uint8_t* p = base + r * slot_bytes;
            void* d_in[kMaxT];
            void* d_out[kMaxT];
            for (int i = 0; i < job.n_in; ++i) {
                d_in[i] = p;
                p += al(job.in[i].unit * cu_units);
            }
            for (int i = 0; i < job.n_out; ++i) {
                d_out[i] = p;
                p += al(job.out[i].unit * cu_units);
            }
            void* ws = ws_bytes ? p : nullptr;
            // H2D: the slot's previous slab must have left the device
            if (c >= R) cu(cudaStreamWaitEvent(cs.in, out_done[r], 0), "wait");
            for (int i = 0; i < job.n_in; ++i)
                cu(cudaMemcpyAsync(d_in[i], job.in[i].in + job.in[i].unit * u0, job.in[i].unit * nu,
                                   cudaMemcpyHostToDevice, cs.in),
                   "H2D");
            cu(cudaEventRecord(in_done[r], cs.in), "event record");
            // kernels of this slab on the caller's stream
            cu(cudaStreamWaitEvent(stream, in_done[r], 0), "wait");
            vattn_config slab = *cfg;
            slab.bh_offset = cfg->bh_offset + u0;
            slab.bh_count = nu;
            chk(job.run(&slab, d_in, d_out, ws, ws_bytes, status, stream), "slab kernels");
            cu(cudaEventRecord(comp_done[r], stream), "event record");
            // D2H
            cu(cudaStreamWaitEvent(cs.out, comp_done[r], 0), "wait");
            for (int i = 0; i < job.n_out; ++i)
                cu(cudaMemcpyAsync(job.out[i].out + job.out[i].unit * u0, d_out[i], job.out[i].unit * nu,
                                   cudaMemcpyDeviceToHost, cs.out),
                   "D2H");
            cu(cudaEventRecord(out_done[r], cs.out), "event record");
        }
        // join: the caller's stream owns the staging memory again, then release it
        cu(cudaStreamWaitEvent(stream, out_done[(n_slabs - 1) % R], 0), "wait");
        if (job.check_domain)
            cu(cudaMemcpyAsync(&h_status, status, sizeof(unsigned int), cudaMemcpyDeviceToHost, stream), "status D2H");
    } catch (const Fail& f) {
        rc = f.code;
        cudaStreamSynchronize(cs.in);
        cudaStreamSynchronize(cs.out);
    }
    cudaFreeAsync(base, stream);
    const cudaError_t se = cudaStreamSynchronize(stream);
    cudaEventDestroy(ready);
    for (int r = 0; r < 3; ++r) {
        cudaEventDestroy(in_done[r]);
        cudaEventDestroy(comp_done[r]);
        cudaEventDestroy(out_done[r]);
    }
    if (rc == VATTN_OK && se != cudaSuccess) {
        g_host_err = std::string("host pipeline: ") + cudaGetErrorString(se);
        rc = VATTN_ECUDA;
    }
    if (rc == VATTN_OK && h_status != 0) {
        // the reference throws std::domain_error here (online_softmax.cpp:33-34, 81-82)
        g_host_err = "softmax: NaN score or fully masked row (l == 0) in a query row (domain error)";
        rc = VATTN_EDOMAIN;
    }
    return rc;
}

size_t t16_unit(const vattn_config* c) { return static_cast<size_t>(c->seq_len) * c->head_dim * 2; }
size_t lse_unit(const vattn_config* c) { return static_cast<size_t>(c->seq_len) * 4; }

}  // namespace
extern "C" int vattn_validate_(const vattn_config* cfg);  // capi.cu
extern "C" int vattn_step_device_(const vattn_config* cfg, const void* q, const void* k, const void* v,
                                  const void* dout, void* o, float* lse, void* dq, void* dk, void* dv,
                                  void* workspace, size_t workspace_bytes, unsigned int* status,
                                  void* stream);  // capi.cu
extern "C" int vattn_forward_status_(const vattn_config* cfg, const void* q, const void* k, const void* v, void* o,
                                     float* lse, unsigned int* status, void* stream);  // capi.cu
namespace {

// The device entry points' own validation (same codes and messages).
int precheck(const vattn_config* c) {
    const int rc = vattn_validate_(c);
    if (rc) g_host_err = vattn_last_error();
    return rc;
}

int run_fwd(const vattn_config* s, void* const* in, void* const* out, void*, size_t, unsigned int* status,
            cudaStream_t st) {
    return vattn_forward_status_(s, in[0], in[1], in[2], out[0], static_cast<float*>(out[1]), status, st);
}

int run_bwd(const vattn_config* s, void* const* in, void* const* out, void* ws, size_t wsb, unsigned int*,
            cudaStream_t st) {
    return mha_backward(s, in[0], in[1], in[2], in[3], in[4], static_cast<const float*>(in[5]), out[0], out[1],
                        out[2], ws, wsb, st);
}

int run_step(const vattn_config* s, void* const* in, void* const* out, void* ws, size_t wsb, unsigned int* status,
             cudaStream_t st) {
    return vattn_step_device_(s, in[0], in[1], in[2], in[3], out[0], static_cast<float*>(out[1]), out[2], out[3],
                              out[4], ws, wsb, status, st);
}

template <typename F>
int guarded(F&& f) {
    try {
        return f();
    } catch (const Fail& e) {
        return e.code;
    }
}

}  // namespace

// vattn_last_error() reports the device-path message; host-path failures are
// appended to it through this hook (capi.cu owns the thread-local string).
extern "C" void vattn_set_error_(const char* msg);

extern "C" {

int mha_forward_host(const vattn_config* cfg, const void* q, const void* k, const void* v, void* o, float* lse,
                     void* stream) {
    int rc = precheck(cfg);
    if (!rc && (!q || !k || !v || !o || !lse)) {
        g_host_err = "mha_forward_host: null tensor pointer";
        rc = VATTN_EINVAL;
    }
    if (!rc) {
        Job j;
        const size_t t = t16_unit(cfg);
        j.in[0] = {static_cast<const uint8_t*>(q), nullptr, t};
        j.in[1] = {static_cast<const uint8_t*>(k), nullptr, t};
        j.in[2] = {static_cast<const uint8_t*>(v), nullptr, t};
        j.n_in = 3;
        j.out[0] = {nullptr, static_cast<uint8_t*>(o), t};
        j.out[1] = {nullptr, reinterpret_cast<uint8_t*>(lse), lse_unit(cfg)};
        j.n_out = 2;
        j.run = run_fwd;
        j.check_domain = true;
        rc = guarded([&] { return run_pipeline(cfg, j, static_cast<cudaStream_t>(stream)); });
    }
    if (rc) vattn_set_error_(g_host_err.c_str());
    return rc;
}

int mha_backward_host(const vattn_config* cfg, const void* q, const void* k, const void* v, const void* o,
                      const void* dout, const float* lse, void* dq, void* dk, void* dv, void* stream) {
    int rc = precheck(cfg);
    if (!rc && (!q || !k || !v || !o || !dout || !lse || !dq || !dk || !dv)) {
        g_host_err = "mha_backward_host: null tensor pointer";
        rc = VATTN_EINVAL;
    }
    if (!rc) {
        Job j;
        const size_t t = t16_unit(cfg);
        j.in[0] = {static_cast<const uint8_t*>(q), nullptr, t};
        j.in[1] = {static_cast<const uint8_t*>(k), nullptr, t};
        j.in[2] = {static_cast<const uint8_t*>(v), nullptr, t};
        j.in[3] = {static_cast<const uint8_t*>(o), nullptr, t};
        j.in[4] = {static_cast<const uint8_t*>(dout), nullptr, t};
        j.in[5] = {reinterpret_cast<const uint8_t*>(lse), nullptr, lse_unit(cfg)};
        j.n_in = 6;
        j.out[0] = {nullptr, static_cast<uint8_t*>(dq), t};
        j.out[1] = {nullptr, static_cast<uint8_t*>(dk), t};
        j.out[2] = {nullptr, static_cast<uint8_t*>(dv), t};
        j.n_out = 3;
        j.ws_unit = 1;
        j.run = run_bwd;
        rc = guarded([&] { return run_pipeline(cfg, j, static_cast<cudaStream_t>(stream)); });
    }
    if (rc) vattn_set_error_(g_host_err.c_str());
    return rc;
}

int mha_step_host(const vattn_config* cfg, const void* q, const void* k, const void* v, const void* dout, void* o,
                  float* lse, void* dq, void* dk, void* dv, void* stream) {
    int rc = precheck(cfg);
    if (!rc && (!q || !k || !v || !dout || !o || !lse || !dq || !dk || !dv)) {
        g_host_err = "mha_step_host: null tensor pointer";
        rc = VATTN_EINVAL;
    }
    if (!rc) {
        Job j;
        const size_t t = t16_unit(cfg);
        j.in[0] = {static_cast<const uint8_t*>(q), nullptr, t};
        j.in[1] = {static_cast<const uint8_t*>(k), nullptr, t};
        j.in[2] = {static_cast<const uint8_t*>(v), nullptr, t};
        j.in[3] = {static_cast<const uint8_t*>(dout), nullptr, t};
        j.n_in = 4;
        j.out[0] = {nullptr, static_cast<uint8_t*>(o), t};
        j.out[1] = {nullptr, reinterpret_cast<uint8_t*>(lse), lse_unit(cfg)};
        j.out[2] = {nullptr, static_cast<uint8_t*>(dq), t};
        j.out[3] = {nullptr, static_cast<uint8_t*>(dk), t};
        j.out[4] = {nullptr, static_cast<uint8_t*>(dv), t};
        j.n_out = 5;
        j.ws_unit = 1;
        j.run = run_step;
        j.check_domain = true;
        rc = guarded([&] { return run_pipeline(cfg, j, static_cast<cudaStream_t>(stream)); });
    }
    if (rc) vattn_set_error_(g_host_err.c_str());
    return rc;
}

}  // extern "C"
