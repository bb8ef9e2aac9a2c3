// Context lifecycle and error plumbing of the C ABI (include/ds_gpu.h).
#include <cstdio>
#include <cstring>
#include <string>

#include "ds_internal.h"

namespace {
thread_local std::string g_last_error;
}

namespace dsi {

void set_error(const std::string& msg) { g_last_error = msg; }

ds_status fail(ds_status s, const std::string& msg) {
    g_last_error = msg;
    return s;
}

ds_status cuda_fail(cudaError_t e, const char* what) {
    g_last_error = std::string(what) + ": " + cudaGetErrorName(e) + " (" +
                   cudaGetErrorString(e) + ")";
    return DS_ERR_CUDA;
}

ds_status ensure_scratch(ds_ctx* ctx, size_t bytes, void** out) {
    if (bytes > ctx->scratch_bytes) {
        if (ctx->scratch) {
            // the _device entry points use this scratch on the CALLER's stream:
            // drain the whole device, not only ctx->stream, before freeing it
            DS_CUDA_TRY(cudaDeviceSynchronize());
            DS_CUDA_TRY(cudaFree(ctx->scratch));
            ctx->scratch = nullptr;
            ctx->scratch_bytes = 0;
        }
        size_t want = align_up(bytes < (1u << 20) ? (1u << 20) : bytes, 1u << 20);
        DS_CUDA_TRY(cudaMalloc(&ctx->scratch, want));
        ctx->scratch_bytes = want;
    }
    *out = ctx->scratch;
    return DS_OK;
}

ds_status ensure_pinned(ds_ctx* ctx, size_t bytes, void** out) {
    if (bytes > ctx->pinned_bytes) {
        if (ctx->pinned) {
            DS_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
            DS_CUDA_TRY(cudaFreeHost(ctx->pinned));
            ctx->pinned = nullptr;
            ctx->pinned_bytes = 0;
        }
        size_t want = align_up(bytes < (1u << 16) ? (1u << 16) : bytes, 1u << 16);
        DS_CUDA_TRY(cudaMallocHost(&ctx->pinned, want));
        ctx->pinned_bytes = want;
    }
    *out = ctx->pinned;
    return DS_OK;
}

ds_status lookback_flags(ds_ctx* ctx, size_t words, unsigned long long** flags, unsigned** done) {
    const size_t need = sizeof(unsigned long long) * words + 256;
    if (need > ctx->route_flags_bytes) {
        if (ctx->route_flags) {
            DS_CUDA_TRY(cudaDeviceSynchronize());
            DS_CUDA_TRY(cudaFree(ctx->route_flags));
            ctx->route_flags = nullptr;
            ctx->route_flags_bytes = 0;
        }
        const size_t want = align_up(need < (1u << 16) ? (1u << 16) : need, 1u << 16);
        DS_CUDA_TRY(cudaMalloc(&ctx->route_flags, want));
        DS_CUDA_TRY(cudaMemset(ctx->route_flags, 0, want));
        ctx->route_flags_bytes = want;
    }
    *flags = static_cast<unsigned long long*>(ctx->route_flags);
    *done = reinterpret_cast<unsigned*>(static_cast<char*>(ctx->route_flags) +
                                        ctx->route_flags_bytes - 256);
    return DS_OK;
}

ds_status reset_device_error(ds_ctx* ctx, cudaStream_t st) {
    static const long long kNone = 0x7fffffffffffffffLL;
    // pageable source: staged before the call returns
    DS_CUDA_TRY(cudaMemcpyAsync(ctx->d_err, &kNone, sizeof(kNone), cudaMemcpyHostToDevice, st));
    return DS_OK;
}

ds_status ensure_copy_stream(ds_ctx* ctx) {
    if (ctx->copy_stream) return DS_OK;
    DS_CUDA_TRY(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
    for (auto& e : ctx->ev) DS_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    return DS_OK;
}

} // namespace dsi

extern "C" {

const char* ds_version(void) { return "ds_b200 abi 1 (sm_100a)"; }

const char* ds_last_error(void) { return g_last_error.c_str(); }

ds_status ds_ctx_create(int device, ds_ctx** out) {
    if (!out) return dsi::fail(DS_ERR_INVALID_ARGUMENT, "ds_ctx_create: out is null");
    *out = nullptr;
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
        return dsi::fail(DS_ERR_NO_DEVICE, "ds_ctx_create: no CUDA device visible");
    if (device < 0 || device >= n)
        return dsi::fail(DS_ERR_INVALID_ARGUMENT, "ds_ctx_create: device index out of range");
    cudaDeviceProp prop;
    DS_CUDA_TRY(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10 || prop.minor != 0)
        return dsi::fail(DS_ERR_NO_DEVICE, "ds_ctx_create: kernels are built for sm_100a only, "
                                           "device is sm_" + std::to_string(prop.major) +
                                               std::to_string(prop.minor));
    DS_CUDA_TRY(cudaSetDevice(device));
    // The per-launch stream-ordered temporaries (cudaMallocAsync) come from the
    // device's default pool; keep freed blocks cached in it instead of returning
    // them to the driver at every synchronization (a re-map costs tens of us).
    {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            uint64_t keep = 1ull << 30;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
    }
    ds_ctx* ctx = new ds_ctx();
    ctx->device = device;
    e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        delete ctx;
        return dsi::cuda_fail(e, "cudaStreamCreate");
    }
    e = cudaMalloc(&ctx->d_err, sizeof(long long));
    if (e != cudaSuccess) {
        cudaStreamDestroy(ctx->stream);
        delete ctx;
        return dsi::cuda_fail(e, "cudaMalloc");
    }
    if (dsi::reset_device_error(ctx, ctx->stream) != DS_OK) {
        cudaFree(ctx->d_err);
        cudaStreamDestroy(ctx->stream);
        delete ctx;
        return DS_ERR_CUDA;
    }
    *out = ctx;
    return DS_OK;
}

ds_status ds_ctx_destroy(ds_ctx* ctx) {
    if (!ctx) return DS_OK;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    if (ctx->scratch) cudaFree(ctx->scratch);
    if (ctx->d_err) cudaFree(ctx->d_err);
    if (ctx->route_flags) cudaFree(ctx->route_flags);
    if (ctx->jump_polys) cudaFree(ctx->jump_polys);
    if (ctx->pinned) cudaFreeHost(ctx->pinned);
    if (ctx->copy_stream) {
        cudaStreamSynchronize(ctx->copy_stream);
        cudaStreamDestroy(ctx->copy_stream);
    }
    for (auto& e : ctx->ev)
        if (e) cudaEventDestroy(e);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
    return DS_OK;
}

ds_status ds_ctx_synchronize(ds_ctx* ctx) {
    if (!ctx) return dsi::fail(DS_ERR_INVALID_ARGUMENT, "null ctx");
    DS_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    return DS_OK;
}

int64_t ds_ctx_launch_count(const ds_ctx* ctx) {
    return ctx ? ctx->launches.load(std::memory_order_relaxed) : 0;
}

ds_status ds_ctx_take_error(ds_ctx* ctx, void* stream, int64_t* first_bad) {
    if (!ctx) return dsi::fail(DS_ERR_INVALID_ARGUMENT, "null ctx");
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
    DS_CUDA_TRY(cudaSetDevice(ctx->device));
    long long v = 0;
    DS_CUDA_TRY(cudaMemcpyAsync(&v, ctx->d_err, sizeof(v), cudaMemcpyDeviceToHost, st));
    DS_CUDA_TRY(cudaStreamSynchronize(st));
    if (first_bad) *first_bad = v == 0x7fffffffffffffffLL ? -1 : v;
    if (v == 0x7fffffffffffffffLL) return DS_OK;
    ds_status s = dsi::reset_device_error(ctx, st);
    if (s != DS_OK) return s;
    return dsi::fail(DS_ERR_DOMAIN, "confidence must lie in [0, 1] (observation " +
                                        std::to_string(v) + " of a device call)");
}

void* ds_ctx_stream(ds_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

} // extern "C"
