// Synthetic image pool (DESIGN.md "Synthetic
// data"). Pixel bytes are a pure function of (seed, image id, pixel index):
//   noise(id, p) = byte (p & 7) of splitmix64(splitmix64(seed) ^ (id << 24 | p >> 3))
//   level(id)    = top byte of splitmix64(splitmix64(seed) ^ ~id)
//   pixel        = (noise + level) >> 1
// so images differ in brightness (the discriminator's confidences spread over
// (0, 1)) and the same bytes can be regenerated on the host for the oracle.
#include <cuda_runtime.h>

#include "ds_internal.h"

namespace {

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

// One thread writes 16 bytes (two splitmix64 words) with one 128-bit store.
__global__ void __launch_bounds__(256)
synth_kernel(uint64_t seed_mix, uint64_t id0, int64_t n, int64_t img_bytes,
             uint8_t* __restrict__ out) {
    const int64_t vecs_per_img = img_bytes / 16;
    const int64_t total = n * vecs_per_img;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t v = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; v < total;
         v += stride) {
        const int64_t img = v / vecs_per_img;
        const int64_t p = (v - img * vecs_per_img) * 16;   // first pixel byte index
        const uint64_t id = id0 + static_cast<uint64_t>(img);
        const unsigned level = static_cast<unsigned>(splitmix64(seed_mix ^ ~id) >> 56);
        uint32_t w[4];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint64_t r =
                splitmix64(seed_mix ^ ((id << 24) | static_cast<uint64_t>((p >> 3) + h)));
            uint32_t lo = 0, hi = 0;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                lo |= ((static_cast<unsigned>((r >> (8 * b)) & 0xFF) + level) >> 1) << (8 * b);
                hi |= ((static_cast<unsigned>((r >> (8 * (b + 4))) & 0xFF) + level) >> 1)
                      << (8 * b);
            }
            w[2 * h] = lo;
            w[2 * h + 1] = hi;
        }
        reinterpret_cast<uint4*>(out)[v] = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

} // namespace

extern "C" ds_status ds_synth_images_device(ds_ctx* ctx, uint64_t seed, uint64_t id0,
                                            int64_t n, int32_t h, int32_t w, uint8_t* out,
                                            void* stream) {
    if (!ctx || (n > 0 && !out)) return dsi::fail(DS_ERR_INVALID_ARGUMENT, "null argument");
    if (h <= 0 || w <= 0 || (static_cast<int64_t>(h) * w * 3) % 16 != 0)
        return dsi::fail(DS_ERR_INVALID_ARGUMENT, "image bytes must be a multiple of 16");
    if (n <= 0) return DS_OK;
    if (id0 + static_cast<uint64_t>(n) >= (1ull << 40))
        return dsi::fail(DS_ERR_CAPACITY, "image ids must stay below 2^40");
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
    const int64_t img_bytes = static_cast<int64_t>(h) * w * 3;
    synth_kernel<<<148 * 8, 256, 0, st>>>(splitmix64(seed), id0, n, img_bytes, out);
    DS_LAUNCH_CHECK(ctx, "synth_kernel");
    return DS_OK;
}
