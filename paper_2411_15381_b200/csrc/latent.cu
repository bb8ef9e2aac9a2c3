// K4 latent_score: the reference's discriminator stand-in on the GPU.
//
// Replaces the per-query loop over diffserve::sample_query
// (reference proj/src/experiment.cpp:76-79 -> proj/src/workload.cpp:108-129).
// Each query seeds a fresh std::mt19937_64 from
//     RandomStream(splitmix64(seed) ^ splitmix64(id), "query")      (rng.hpp:20-21)
// and consumes exactly 5 outputs: 1 Bernoulli + 2 Box-Muller normals
// (workload.cpp:116-119, rng.cpp:30-36). Those 5 outputs only depend on state
// words x_0..x_5 and x_156..x_160 of the seeding recurrence, so the engine is
// streamed in registers (161 recurrence steps) instead of materialising
// 2.5 KB of state and a full 312-word twist (SURVEY.md hard part 3).
//
// fp64 arithmetic is written with explicit _rn intrinsics in the reference's
// evaluation order (no FMA contraction). sqrt is correctly rounded on both
// sides; log and cos are glibc's FMA builds restated operation by operation
// (glibc_libm.h), so every confidence and quality value is bit-identical to
// the reference's (tests/test_gpu_score_route.py requires all of them).
#include <cuda_runtime.h>

#include "ds_internal.h"
#include "glibc_libm.h"

namespace {

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {   // rng.cpp:8-13
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

uint64_t fnv1a(const char* s) {                                          // rng.cpp:15-22
    uint64_t h = 0xcbf29ce484222325ULL;
    for (; *s; ++s) {
        h ^= static_cast<unsigned char>(*s);
        h *= 0x100000001b3ULL;
    }
    return h;
}

__device__ __forceinline__ uint64_t temper(uint64_t z) {
    z ^= (z >> 29) & 0x5555555555555555ULL;
    z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
    z ^= (z << 37) & 0xFFF7EEE000000000ULL;
    z ^= z >> 43;
    return z;
}

__device__ __forceinline__ uint64_t twist(uint64_t xk, uint64_t xk1, uint64_t xkm) {
    const uint64_t y = (xk & 0xFFFFFFFF80000000ULL) | (xk1 & 0x7FFFFFFFULL);
    uint64_t v = xkm ^ (y >> 1);
    if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
    return v;
}

// First 5 outputs of std::mt19937_64(seed).
__device__ __forceinline__ void mt64_first5(uint64_t seed, uint64_t out[5]) {
    uint64_t lo[6], hi[5];
    uint64_t x = seed;
    lo[0] = x;
#pragma unroll
    for (int i = 1; i <= 5; ++i) {
        x = 6364136223846793005ULL * (x ^ (x >> 62)) + static_cast<uint64_t>(i);
        lo[i] = x;
    }
#pragma unroll 10
    for (int i = 6; i <= 155; ++i)
        x = 6364136223846793005ULL * (x ^ (x >> 62)) + static_cast<uint64_t>(i);
#pragma unroll
    for (int i = 156; i <= 160; ++i) {
        x = 6364136223846793005ULL * (x ^ (x >> 62)) + static_cast<uint64_t>(i);
        hi[i - 156] = x;
    }
#pragma unroll
    for (int k = 0; k < 5; ++k) out[k] = temper(twist(lo[k], lo[k + 1], hi[k]));
}

__device__ __forceinline__ double uniform53(uint64_t r) {              // rng.hpp:26
    return __dmul_rn(static_cast<double>(r >> 11), 0x1.0p-53);
}

__device__ __forceinline__ double box_muller(uint64_t r1, uint64_t r2) { // rng.cpp:30-36
    double u1 = uniform53(r1);
    const double u2 = uniform53(r2);
    if (u1 <= 0.0) u1 = 0x1.0p-53;
    // 2.0 * M_PI * u2 == (2.0 * M_PI) * u2; 2*pi is exact in double
    // log and cos exactly as glibc's FMA builds compute them (glibc_libm.h):
    // the draw is bit-identical to the reference's
    return __dmul_rn(__dsqrt_rn(__dmul_rn(-2.0, glibc_log(u1))),
                     glibc_cos(__dmul_rn(6.283185307179586, u2)));
}

// kRecords: write full Query records (workload.cpp:121-128) instead of the
// conf / quality_light columns.
template <bool kRecords>
__global__ void __launch_bounds__(256)
latent_kernel(double easy_fraction, double gap_scale, double fidelity, double sigma,
              uint64_t seed_mix, uint64_t id0, int64_t n, double* __restrict__ conf,
              double* __restrict__ quality_light, const double* __restrict__ arrivals,
              double slo_seconds, ds_query* __restrict__ records) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += stride) {
        const uint64_t id = id0 + static_cast<uint64_t>(i);
        // splitmix64( (splitmix64(seed) ^ splitmix64(id)) ^ splitmix64(fnv1a("query")) )
        const uint64_t eng_seed = splitmix64(seed_mix ^ splitmix64(id));
        uint64_t r[5];
        mt64_first5(eng_seed, r);
        const bool easy = uniform53(r[0]) < easy_fraction;               // workload.cpp:116
        const double gap = __dmul_rn(gap_scale, fabs(box_muller(r[1], r[2])));
        const double dq = easy ? gap : -gap;
        const double noise = __dadd_rn(0.0, __dmul_rn(sigma, box_muller(r[3], r[4])));
        double c = __dadd_rn(__dadd_rn(0.5, __dmul_rn(fidelity, dq)), noise);
        c = c < 0.0 ? 0.0 : (1.0 < c ? 1.0 : c);                        // std::clamp
        if constexpr (kRecords) {
            const double arrival = arrivals[i];
            ds_query q;
            q.id = id;
            q.arrival = arrival;
            q.deadline = __dadd_rn(arrival, slo_seconds);
            q.quality_light = __dadd_rn(1.0, dq);
            q.quality_heavy = 1.0;
            q.confidence = c;
            records[i] = q;
        } else {
            conf[i] = c;
            if (quality_light) quality_light[i] = __dadd_rn(1.0, dq);
        }
    }
}

int latent_blocks(int64_t n) {
    int64_t blocks = (n + 255) / 256;
    const int64_t cap = 148 * 16;   // grid-stride beyond 16 waves of 256
    return static_cast<int>(blocks > cap ? cap : blocks);
}

ds_status check_model(const ds_query_model* m) {   // workload.cpp:110-111
    if (!(m->easy_fraction >= 0.0) || !(m->easy_fraction <= 1.0))
        return dsi::fail(DS_ERR_DOMAIN, "easy_fraction must lie in [0, 1]");
    return DS_OK;
}

} // namespace

extern "C" ds_status ds_score_latent_device(ds_ctx* ctx, const ds_query_model* m, uint64_t id0,
                                            int64_t n, double* conf, double* quality_light,
                                            void* stream) {
    if (!ctx || !m) return dsi::fail(DS_ERR_INVALID_ARGUMENT, "null argument");
    if (ds_status s = check_model(m); s != DS_OK) return s;
    if (n <= 0) return DS_OK;
    const uint64_t seed_mix = splitmix64(m->seed) ^ splitmix64(fnv1a("query"));
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
    latent_kernel<false><<<latent_blocks(n), 256, 0, st>>>(
        m->easy_fraction, m->quality_gap_scale, m->confidence_fidelity, m->noise_sigma,
        seed_mix, id0, n, conf, quality_light, nullptr, 0.0, nullptr);
    DS_LAUNCH_CHECK(ctx, "latent_kernel");
    return DS_OK;
}

extern "C" ds_status ds_score_latent(ds_ctx* ctx, const ds_query_model* m, uint64_t id0,
                                     int64_t n, double* conf, double* quality_light) {
    if (!ctx || !m || (n > 0 && !conf)) return dsi::fail(DS_ERR_INVALID_ARGUMENT, "null argument");
    // sample_query's checks (workload.cpp:110-112); slo is not an input here.
    if (ds_status s = check_model(m); s != DS_OK) return s;
    if (n <= 0) return DS_OK;
    const size_t bytes = dsi::align_up(sizeof(double) * n, 256);
    char* d = nullptr;
    ds_status st = dsi::ensure_scratch(ctx, bytes * 2, reinterpret_cast<void**>(&d));
    if (st != DS_OK) return st;
    double* dconf = reinterpret_cast<double*>(d);
    double* dql = quality_light ? reinterpret_cast<double*>(d + bytes) : nullptr;
    st = ds_score_latent_device(ctx, m, id0, n, dconf, dql, ctx->stream);
    if (st != DS_OK) return st;
    DS_CUDA_TRY(cudaMemcpyAsync(conf, dconf, sizeof(double) * n, cudaMemcpyDeviceToHost,
                                ctx->stream));
    if (quality_light)
        DS_CUDA_TRY(cudaMemcpyAsync(quality_light, dql, sizeof(double) * n,
                                    cudaMemcpyDeviceToHost, ctx->stream));
    DS_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    return DS_OK;
}

extern "C" ds_status ds_sample_queries_device(ds_ctx* ctx, const ds_query_model* m, uint64_t id0,
                                             const double* arrivals, int64_t n,
                                             double slo_seconds, ds_query* out, void* stream) {
    if (!ctx || !m || (n > 0 && (!arrivals || !out)))
        return dsi::fail(DS_ERR_INVALID_ARGUMENT, "null argument");
    if (ds_status s = check_model(m); s != DS_OK) return s;
    if (!(slo_seconds > 0.0)) return dsi::fail(DS_ERR_DOMAIN, "slo_seconds must be positive");
    if (n <= 0) return DS_OK;
    const uint64_t seed_mix = splitmix64(m->seed) ^ splitmix64(fnv1a("query"));
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
    latent_kernel<true><<<latent_blocks(n), 256, 0, st>>>(
        m->easy_fraction, m->quality_gap_scale, m->confidence_fidelity, m->noise_sigma,
        seed_mix, id0, n, nullptr, nullptr, arrivals, slo_seconds, out);
    DS_LAUNCH_CHECK(ctx, "latent_kernel<records>");
    return DS_OK;
}

extern "C" ds_status ds_sample_queries(ds_ctx* ctx, const ds_query_model* m, uint64_t id0,
                                      const double* arrivals, int64_t n, double slo_seconds,
                                      ds_query* out) {
    if (!ctx || !m || (n > 0 && (!arrivals || !out)))
        return dsi::fail(DS_ERR_INVALID_ARGUMENT, "null argument");
    if (ds_status s = check_model(m); s != DS_OK) return s;
    if (!(slo_seconds > 0.0)) return dsi::fail(DS_ERR_DOMAIN, "slo_seconds must be positive");
    if (n <= 0) return DS_OK;
    const size_t ba = dsi::align_up(sizeof(double) * n, 256);
    char* d = nullptr;
    ds_status st = dsi::ensure_scratch(ctx, ba + sizeof(ds_query) * n, reinterpret_cast<void**>(&d));
    if (st != DS_OK) return st;
    double* darr = reinterpret_cast<double*>(d);
    ds_query* dq = reinterpret_cast<ds_query*>(d + ba);
    DS_CUDA_TRY(cudaMemcpyAsync(darr, arrivals, sizeof(double) * n, cudaMemcpyHostToDevice,
                                ctx->stream));
    st = ds_sample_queries_device(ctx, m, id0, darr, n, slo_seconds, dq, ctx->stream);
    if (st != DS_OK) return st;
    DS_CUDA_TRY(cudaMemcpyAsync(out, dq, sizeof(ds_query) * n, cudaMemcpyDeviceToHost,
                                ctx->stream));
    DS_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    return DS_OK;
}
