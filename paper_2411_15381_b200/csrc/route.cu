// K2 route_compact: threshold routing with order-preserving stream compaction.
//
// Replaces the per-query Policy::defers loop of the light-batch completion
// handler (reference proj/src/cluster.cpp:290-306, proj/src/policies.cpp:37-39):
// a query defers iff confidence < t (strict; c == t stays light,
// test_policies.cpp:46-48), and deferred ids enter the heavy queue in id
// order. For every threshold t_k the output is that ordered id list.
//
// Two passes over tiles of kTile confidences (HBM-bound: 4-8 B read + 8 B
// written per deferred query; the second pass re-reads the tile from L2):
//   count  : per (tile, threshold) number of deferrals (warp ballot + popc)
//   scatter: block-exclusive prefix of earlier tiles' counts, then a warp
//            ballot/popc prefix inside the tile gives each deferred query its
//            slot; indices are written coalesced-in-order.
#include <cuda_runtime.h>

#include "ds_internal.h"

namespace {

constexpr int kThreads = 256;
constexpr int kPerThread = 8;
constexpr int kTile = kThreads * kPerThread;   // 2048 queries per tile

template <typename T>
__device__ __forceinline__ double load_conf(const T* c, int64_t i) {
    return static_cast<double>(__ldg(c + i));
}

// Grid (tiles, thresholds). counts[k * tiles + tile]
template <typename T>
__global__ void __launch_bounds__(kThreads)
route_count_kernel(const T* __restrict__ conf, int64_t n, const double* __restrict__ thr,
                   int32_t* __restrict__ counts) {
    const int tile = blockIdx.x, k = blockIdx.y, tiles = gridDim.x;
    const double t = thr[k];
    const int64_t base = static_cast<int64_t>(tile) * kTile;
    int mine = 0;
#pragma unroll
    for (int r = 0; r < kPerThread; ++r) {
        const int64_t i = base + r * kThreads + threadIdx.x;
        if (i < n && load_conf(conf, i) < t) ++mine;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
    __shared__ int warp_sum[kThreads / 32];
    if ((threadIdx.x & 31) == 0) warp_sum[threadIdx.x >> 5] = mine;
    __syncthreads();
    if (threadIdx.x == 0) {
        int s = 0;
#pragma unroll
        for (int w = 0; w < kThreads / 32; ++w) s += warp_sum[w];
        counts[static_cast<int64_t>(k) * tiles + tile] = s;
    }
}

// kSingle: n fits one tile (n <= kTile, the light batches): no count pass, the
// prefix of earlier tiles is 0 and the tile's own count is the total.
template <typename T, bool kSingle = false>
__global__ void __launch_bounds__(kThreads)
route_scatter_kernel(const T* __restrict__ conf, int64_t n, const double* __restrict__ thr,
                     const int32_t* __restrict__ counts, int64_t index_base,
                     int64_t* __restrict__ heavy_idx, int64_t* __restrict__ total_out) {
    const int tile = blockIdx.x, k = blockIdx.y, tiles = gridDim.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const double t = thr[k];
    const int32_t* ck = counts + static_cast<int64_t>(k) * tiles;
    __shared__ long long s_prefix;
    __shared__ int warp_cnt[kPerThread][kThreads / 32];
    // exclusive prefix of earlier tiles (warp 0), and the grand total (last tile)
    if (kSingle) {
        if (threadIdx.x == 0) s_prefix = 0;
    } else if (warp == 0) {
        long long acc = 0;
        for (int b = lane; b < tile; b += 32) acc += ck[b];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) {
            s_prefix = acc;
            if (tile == tiles - 1) total_out[k] = acc + ck[tile];
        }
    }
    // Element order inside the tile: row r (kThreads wide), then thread.
    const int64_t base = static_cast<int64_t>(tile) * kTile;
    unsigned ballots[kPerThread];
#pragma unroll
    for (int r = 0; r < kPerThread; ++r) {
        const int64_t i = base + r * kThreads + threadIdx.x;
        const bool p = i < n && load_conf(conf, i) < t;
        ballots[r] = __ballot_sync(0xffffffffu, p);
        if (lane == 0) warp_cnt[r][warp] = __popc(ballots[r]);
    }
    __syncthreads();
    // Offsets: all rows before r (all warps), then warps before `warp` in row r.
    long long off = s_prefix;
    int64_t* out = heavy_idx + static_cast<int64_t>(k) * n;
#pragma unroll
    for (int r = 0; r < kPerThread; ++r) {
        int before = 0, row = 0;
#pragma unroll
        for (int w = 0; w < kThreads / 32; ++w) {
            const int c = warp_cnt[r][w];
            before += w < warp ? c : 0;
            row += c;
        }
        const unsigned b = ballots[r];
        if ((b >> lane) & 1u) {
            const int within = __popc(b & ((1u << lane) - 1u));
            out[off + before + within] = index_base + base + r * kThreads + threadIdx.x;
        }
        off += row;
    }
    if (kSingle && threadIdx.x == 0) total_out[k] = off;
}

} // namespace

extern "C" size_t ds_route_scratch_bytes(int64_t n, int32_t n_thresholds) {
    const int64_t tiles = (n + kTile - 1) / kTile;
    return dsi::align_up(sizeof(int32_t) * tiles * (n_thresholds > 0 ? n_thresholds : 1), 256);
}

namespace {

ds_status route_launch(ds_ctx* ctx, const void* conf, int32_t dtype, int64_t n,
                       const double* thresholds, int32_t nt, int64_t index_base,
                       int64_t* heavy_idx, int64_t* counts, int32_t* scratch, cudaStream_t st) {
    const int64_t tiles = (n + kTile - 1) / kTile;
    if (tiles > 0x7fffffff || nt > 65535)
        return dsi::fail(DS_ERR_CAPACITY, "ds_route: too many tiles or thresholds");
    dim3 grid(static_cast<unsigned>(tiles), static_cast<unsigned>(nt));
    if (tiles == 1) {   // one launch for a light batch
        if (dtype == DS_CONF_F64)
            route_scatter_kernel<double, true><<<grid, kThreads, 0, st>>>(
                static_cast<const double*>(conf), n, thresholds, nullptr, index_base, heavy_idx,
                counts);
        else
            route_scatter_kernel<float, true><<<grid, kThreads, 0, st>>>(
                static_cast<const float*>(conf), n, thresholds, nullptr, index_base, heavy_idx,
                counts);
        DS_LAUNCH_CHECK(ctx, "route_scatter_kernel");
        return DS_OK;
    }
    if (dtype == DS_CONF_F64) {
        route_count_kernel<double><<<grid, kThreads, 0, st>>>(
            static_cast<const double*>(conf), n, thresholds, scratch);
        DS_LAUNCH_CHECK(ctx, "route_count_kernel");
        route_scatter_kernel<double><<<grid, kThreads, 0, st>>>(
            static_cast<const double*>(conf), n, thresholds, scratch, index_base, heavy_idx,
            counts);
    } else {
        route_count_kernel<float><<<grid, kThreads, 0, st>>>(
            static_cast<const float*>(conf), n, thresholds, scratch);
        DS_LAUNCH_CHECK(ctx, "route_count_kernel");
        route_scatter_kernel<float><<<grid, kThreads, 0, st>>>(
            static_cast<const float*>(conf), n, thresholds, scratch, index_base, heavy_idx,
            counts);
    }
    DS_LAUNCH_CHECK(ctx, "route_scatter_kernel");
    return DS_OK;
}

} // namespace

// Device variant: `counts` must be device memory; scratch comes from the ctx
// (stream-ordered, so callers on other streams must not overlap two calls).
extern "C" ds_status ds_route_device(ds_ctx* ctx, const void* conf, int32_t dtype, int64_t n,
                                     const double* thresholds, int32_t nt, int64_t index_base,
                                     int64_t* heavy_idx, int64_t* counts, void* stream) {
    if (!ctx) return dsi::fail(DS_ERR_INVALID_ARGUMENT, "null ctx");
    if (dtype != DS_CONF_F64 && dtype != DS_CONF_F32)
        return dsi::fail(DS_ERR_INVALID_ARGUMENT, "ds_route: unknown confidence dtype");
    if (nt <= 0) return DS_OK;
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
    if (n <= 0) {
        DS_CUDA_TRY(cudaMemsetAsync(counts, 0, sizeof(int64_t) * nt, st));
        return DS_OK;
    }
    void* scratch = nullptr;
    ds_status s = dsi::ensure_scratch(ctx, ds_route_scratch_bytes(n, nt), &scratch);
    if (s != DS_OK) return s;
    return route_launch(ctx, conf, dtype, n, thresholds, nt, index_base, heavy_idx, counts,
                        static_cast<int32_t*>(scratch), st);
}

extern "C" ds_status ds_route(ds_ctx* ctx, const void* conf, int32_t dtype, int64_t n,
                              const double* thresholds, int32_t nt, int64_t index_base,
                              int64_t* heavy_idx, int64_t* counts) {
    if (!ctx || (n > 0 && !conf) || (nt > 0 && (!thresholds || !counts)))
        return dsi::fail(DS_ERR_INVALID_ARGUMENT, "ds_route: null argument");
    if (dtype != DS_CONF_F64 && dtype != DS_CONF_F32)
        return dsi::fail(DS_ERR_INVALID_ARGUMENT, "ds_route: unknown confidence dtype");
    if (nt <= 0) return DS_OK;
    if (n <= 0) {
        for (int k = 0; k < nt; ++k) counts[k] = 0;
        return DS_OK;
    }
    const size_t esz = dtype == DS_CONF_F64 ? 8 : 4;
    const size_t bc = dsi::align_up(esz * n, 256);
    const size_t bt = dsi::align_up(sizeof(double) * nt, 256);
    const size_t bk = dsi::align_up(sizeof(int64_t) * nt, 256);
    const size_t bs = ds_route_scratch_bytes(n, nt);
    const size_t bi = dsi::align_up(sizeof(int64_t) * n * nt, 256);
    char* d = nullptr;
    ds_status s = dsi::ensure_scratch(ctx, bc + bt + bk + bs + bi, reinterpret_cast<void**>(&d));
    if (s != DS_OK) return s;
    DS_CUDA_TRY(cudaMemcpyAsync(d, conf, esz * n, cudaMemcpyHostToDevice, ctx->stream));
    DS_CUDA_TRY(cudaMemcpyAsync(d + bc, thresholds, sizeof(double) * nt, cudaMemcpyHostToDevice,
                                ctx->stream));
    int64_t* dcounts = reinterpret_cast<int64_t*>(d + bc + bt);
    int32_t* dscr = reinterpret_cast<int32_t*>(d + bc + bt + bk);
    int64_t* didx = reinterpret_cast<int64_t*>(d + bc + bt + bk + bs);
    s = route_launch(ctx, d, dtype, n, reinterpret_cast<double*>(d + bc), nt, index_base, didx,
                     dcounts, dscr, ctx->stream);
    if (s != DS_OK) return s;
    DS_CUDA_TRY(cudaMemcpyAsync(counts, dcounts, sizeof(int64_t) * nt, cudaMemcpyDeviceToHost,
                                ctx->stream));
    DS_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    if (heavy_idx) {
        // copy only the filled prefix of every per-threshold list
        for (int k = 0; k < nt; ++k)
            if (counts[k] > 0)
                DS_CUDA_TRY(cudaMemcpyAsync(heavy_idx + static_cast<int64_t>(k) * n,
                                            didx + static_cast<int64_t>(k) * n,
                                            sizeof(int64_t) * counts[k], cudaMemcpyDeviceToHost,
                                            ctx->stream));
        DS_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    }
    return DS_OK;
}
