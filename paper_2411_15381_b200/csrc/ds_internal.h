// Internal host-side plumbing shared by the .cu translation units: the
// context object behind ds_ctx*, error capture, grow-only device scratch.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <string>

#include "ds_gpu.h"

struct ds_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    std::atomic<int64_t> launches{0};
    // grow-only device scratch for the host-buffer (copying) entry points
    void* scratch = nullptr;
    size_t scratch_bytes = 0;
    // pinned host staging for small results
    void* pinned = nullptr;
    size_t pinned_bytes = 0;
    // second stream + events for copy/compute overlap in host-buffer calls
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    // first invalid confidence a device variant met (LLONG_MAX if none): the
    // _device calls cannot return the reference's domain_error at launch time
    // (ds_ctx_take_error reads and clears it)
    long long* d_err = nullptr;
    // decoupled look-back flags of K2 / K9 (lookback.cuh): words + a done
    // counter, zero at allocation and left zero by every launch
    void* route_flags = nullptr;
    size_t route_flags_bytes = 0;
    unsigned route_attr_set = 0;   // kernels whose shared-memory attribute is set
    // K8's jump-ahead tables on the device: the set-bit exponents of
    // x^(s L) mod phi for s >= 1 (offsets, then uint16 exponents)
    void* jump_polys = nullptr;
    int jump_polys_n = 0;
    size_t jump_idx_offset = 0;
};

namespace dsi {

// Thread-local last error text (ds_last_error).
void set_error(const std::string& msg);
ds_status fail(ds_status s, const std::string& msg);
ds_status cuda_fail(cudaError_t e, const char* what);

// Device scratch of at least `bytes` (stream-ordered reuse; callers on one
// ctx are serialized by the stream).
ds_status ensure_scratch(ds_ctx* ctx, size_t bytes, void** out);
ds_status ensure_pinned(ds_ctx* ctx, size_t bytes, void** out);
ds_status ensure_copy_stream(ds_ctx* ctx);

// At least `words` zeroed look-back flag words and the done counter
// (lookback.cuh; grow-only, shared by the launches of one context).
ds_status lookback_flags(ds_ctx* ctx, size_t words, unsigned long long** flags, unsigned** done);

// Stream-ordered reset of ctx->d_err to LLONG_MAX.
ds_status reset_device_error(ds_ctx* ctx, cudaStream_t st);

// ds_curve_observe_device + the device word with the first invalid index
// (curve.cu).
ds_status curve_observe_device_bad(ds_ctx* ctx, ds_curve* curve, const void* conf, int32_t dtype,
                                   int64_t n, double decay, cudaStream_t st, const int** bad);

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

} // namespace dsi

#define DS_CUDA_TRY(expr)                                                        \
    do {                                                                         \
        cudaError_t e_ = (expr);                                                 \
        if (e_ != cudaSuccess) return dsi::cuda_fail(e_, #expr);                 \
    } while (0)

#define DS_LAUNCH_CHECK(ctx, what)                                               \
    do {                                                                         \
        (ctx)->launches.fetch_add(1, std::memory_order_relaxed);                 \
        cudaError_t e_ = cudaGetLastError();                                     \
        if (e_ != cudaSuccess) return dsi::cuda_fail(e_, what);                  \
    } while (0)
