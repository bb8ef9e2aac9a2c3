// K3 curve_observe: the online deferral-curve update on the GPU.
//
// Replaces repeated diffserve::observe_confidence (reference
// proj/src/profiles.cpp:108-120) over an ordered confidence sequence (the
// light-batch completion order of cluster.cpp:290-296). Per observation the
// reference scales every bin and the total by `decay`, then adds 1 to the
// observation's bin and to the total. Rounding makes the result
// order-dependent, so each of the 101 bins (plus the total) is replayed
// sequentially by its own thread: bit-identical to the reference (SURVEY probe
// A.4). The observations' bins are computed once per chunk in parallel and
// staged through shared memory.
#include <cuda_runtime.h>

#include "ds_internal.h"

namespace {

constexpr int kThreads = 128;   // 101 bins + total, padded to 4 warps
constexpr int kChunk = 4096;

// m + 1 on a hit, else m. A real (divergent) branch rather than an
// add-and-select: a bin's thread hits on ~1% of observations, and only the
// warp holding the hit bin waits for the add.
__device__ __forceinline__ double add_one_if(double m, bool hit) {
    if (hit) {
        asm volatile("" ::: "memory");   // keep the branch (no if-conversion)
        m = __dadd_rn(m, 1.0);
    }
    return m;
}

template <typename T, bool kScale>
__global__ void __launch_bounds__(kThreads)
curve_observe_kernel(ds_curve* __restrict__ curve, const T* __restrict__ conf, int64_t n,
                     double decay, int* __restrict__ bad) {
    __shared__ __align__(16) unsigned char bins[kChunk];
    __shared__ int chunk_bad;
    const int tid = threadIdx.x;
    double m = 0.0;
    if (tid < DS_CURVE_BINS) m = curve->bin_mass[tid];
    else if (tid == DS_CURVE_BINS) m = curve->total_mass;
    bool settled = false;
    // the total-mass thread matches every observation; bin threads their own bin
    const unsigned mine = tid < DS_CURVE_BINS ? static_cast<unsigned>(tid) : 0xFFu;
    const bool is_total = tid == DS_CURVE_BINS;
    for (int64_t base = 0; base < n; base += kChunk) {
        const int cnt = static_cast<int>(n - base < kChunk ? n - base : kChunk);
        if (tid == 0) chunk_bad = 0;
        __syncthreads();
        for (int k = tid; k < cnt; k += kThreads) {
            const double c = static_cast<double>(conf[base + k]);
            if (!(c >= 0.0) || !(c <= 1.0)) {
                atomicMin(bad, static_cast<int>(base + k < 0x7fffffff ? base + k : 0x7fffffff));
                chunk_bad = 1;
                bins[k] = 255;
                continue;
            }
            // bin_of (profiles.cpp:60-65): floor(c*100 + 1e-9) clamped to [0, 100]
            int b = static_cast<int>(floor(__dadd_rn(__dmul_rn(c, 100.0), 1e-9)));
            b = b < 0 ? 0 : (b > DS_CURVE_BINS - 1 ? DS_CURVE_BINS - 1 : b);
            bins[k] = static_cast<unsigned char>(b);
        }
        __syncthreads();
        if (tid <= DS_CURVE_BINS) {
            if (!chunk_bad) {
                if (is_total) {
                    // every observation hits the total: t <- fl(fl(t*d) + 1). The map is
                    // deterministic, so once a step leaves t unchanged (t reaches the
                    // rounded fixed point, ~1/(1-d) after ~40K steps at d = 0.999) every
                    // later step does too and the replay of the total can stop.
                    // The fixed-point test runs once per 32 steps (one extra step,
                    // discarded unless it proves the fixed point), off the chain.
                    if (!settled) {
                        int k = 0;
                        for (; k + 32 <= cnt; k += 32) {
                            if (kScale && __dadd_rn(__dmul_rn(m, decay), 1.0) == m) {
                                settled = true;
                                break;
                            }
#pragma unroll
                            for (int u = 0; u < 32; ++u)
                                m = __dadd_rn(kScale ? __dmul_rn(m, decay) : m, 1.0);
                        }
                        if (!settled)
                            for (; k < cnt; ++k) m = __dadd_rn(kScale ? __dmul_rn(m, decay) : m, 1.0);
                    }
                } else {
                    // 8 observations per 64-bit shared load; the add on a hit is a
                    // predicated instruction so a miss costs only the multiply
                    const int full8 = cnt & ~7;
                    for (int k = 0; k < full8; k += 8) {
                        const uint2 w = *reinterpret_cast<const uint2*>(&bins[k]);
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            const unsigned b = ((u < 4 ? w.x : w.y) >> (8 * (u & 3))) & 0xFFu;
                            if (kScale) m = __dmul_rn(m, decay);
                            m = add_one_if(m, b == mine);
                        }
                    }
                    for (int k = full8; k < cnt; ++k) {
                        if (kScale) m = __dmul_rn(m, decay);
                        m = add_one_if(m, bins[k] == mine);
                    }
                }
            } else {
                for (int k = 0; k < cnt; ++k) {
                    const unsigned char b = bins[k];
                    if (b == 255) break;   // the reference throws here; state stops
                    if (kScale) m = __dmul_rn(m, decay);
                    if (is_total || b == mine) m = __dadd_rn(m, 1.0);
                }
            }
        }
        __syncthreads();
        if (chunk_bad) break;
    }
    if (tid < DS_CURVE_BINS) curve->bin_mass[tid] = m;
    else if (tid == DS_CURVE_BINS) curve->total_mass = m;
}

__global__ void init_bad(int* bad) { *bad = 0x7fffffff; }

ds_status launch(ds_ctx* ctx, ds_curve* dcurve, const void* conf, int32_t dtype, int64_t n,
                 double decay, int* dbad, cudaStream_t st) {
    init_bad<<<1, 1, 0, st>>>(dbad);
    DS_LAUNCH_CHECK(ctx, "init_bad");
    const bool scale = decay != 1.0;
    if (dtype == DS_CONF_F64) {
        const double* c = static_cast<const double*>(conf);
        if (scale) curve_observe_kernel<double, true><<<1, kThreads, 0, st>>>(dcurve, c, n, decay, dbad);
        else curve_observe_kernel<double, false><<<1, kThreads, 0, st>>>(dcurve, c, n, decay, dbad);
    } else {
        const float* c = static_cast<const float*>(conf);
        if (scale) curve_observe_kernel<float, true><<<1, kThreads, 0, st>>>(dcurve, c, n, decay, dbad);
        else curve_observe_kernel<float, false><<<1, kThreads, 0, st>>>(dcurve, c, n, decay, dbad);
    }
    DS_LAUNCH_CHECK(ctx, "curve_observe_kernel");
    return DS_OK;
}

} // namespace

// Device variant: `curve` is a device ds_curve updated in place. A confidence
// outside [0, 1] stops the replay where the reference would throw; the
// host-buffer variant reports it as DS_ERR_DOMAIN.
extern "C" ds_status ds_curve_observe_device(ds_ctx* ctx, ds_curve* curve, const void* conf,
                                             int32_t dtype, int64_t n, double decay,
                                             void* stream) {
    if (!ctx || !curve) return dsi::fail(DS_ERR_INVALID_ARGUMENT, "null argument");
    if (dtype != DS_CONF_F64 && dtype != DS_CONF_F32)
        return dsi::fail(DS_ERR_INVALID_ARGUMENT, "unknown confidence dtype");
    if (!(decay > 0.0) || !(decay <= 1.0))
        return dsi::fail(DS_ERR_DOMAIN, "curve decay must lie in (0, 1]");
    if (n <= 0) return DS_OK;
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
    void* scratch = nullptr;
    ds_status s = dsi::ensure_scratch(ctx, 256, &scratch);
    if (s != DS_OK) return s;
    return launch(ctx, curve, conf, dtype, n, decay, static_cast<int*>(scratch), st);
}

extern "C" ds_status ds_curve_observe(ds_ctx* ctx, ds_curve* curve, const void* conf,
                                      int32_t dtype, int64_t n, double decay) {
    if (!ctx || !curve || (n > 0 && !conf))
        return dsi::fail(DS_ERR_INVALID_ARGUMENT, "null argument");
    if (dtype != DS_CONF_F64 && dtype != DS_CONF_F32)
        return dsi::fail(DS_ERR_INVALID_ARGUMENT, "unknown confidence dtype");
    if (n <= 0) return DS_OK;
    // observe_confidence checks confidence first, then decay (profiles.cpp:109-112)
    const size_t esz = dtype == DS_CONF_F64 ? 8 : 4;
    const size_t bc = dsi::align_up(esz * n, 256);
    const size_t bv = dsi::align_up(sizeof(ds_curve), 256);
    char* d = nullptr;
    ds_status s = dsi::ensure_scratch(ctx, bc + bv + 256, reinterpret_cast<void**>(&d));
    if (s != DS_OK) return s;
    DS_CUDA_TRY(cudaMemcpyAsync(d, conf, esz * n, cudaMemcpyHostToDevice, ctx->stream));
    DS_CUDA_TRY(cudaMemcpyAsync(d + bc, curve, sizeof(ds_curve), cudaMemcpyHostToDevice,
                                ctx->stream));
    int* dbad = reinterpret_cast<int*>(d + bc + bv);
    if (!(decay > 0.0) || !(decay <= 1.0)) {
        // the first observation's confidence check precedes the decay check
        const double c0 = dtype == DS_CONF_F64 ? static_cast<const double*>(conf)[0]
                                               : static_cast<const float*>(conf)[0];
        if (!(c0 >= 0.0) || !(c0 <= 1.0))
            return dsi::fail(DS_ERR_DOMAIN, "confidence must lie in [0, 1]");
        return dsi::fail(DS_ERR_DOMAIN, "curve decay must lie in (0, 1]");
    }
    s = launch(ctx, reinterpret_cast<ds_curve*>(d + bc), d, dtype, n, decay, dbad, ctx->stream);
    if (s != DS_OK) return s;
    int bad = 0;
    DS_CUDA_TRY(cudaMemcpyAsync(curve, d + bc, sizeof(ds_curve), cudaMemcpyDeviceToHost,
                                ctx->stream));
    DS_CUDA_TRY(cudaMemcpyAsync(&bad, dbad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    DS_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    if (bad != 0x7fffffff)
        return dsi::fail(DS_ERR_DOMAIN, "confidence must lie in [0, 1] (observation " +
                                            std::to_string(bad) + ")");
    return DS_OK;
}
