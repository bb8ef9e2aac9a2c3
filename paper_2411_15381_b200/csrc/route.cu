// K2 route_compact: threshold routing with order-preserving stream compaction.
//
// Replaces the per-query Policy::defers loop of the light-batch completion
// handler (reference proj/src/cluster.cpp:290-306, proj/src/policies.cpp:37-39):
// a query defers iff confidence < t (strict; c == t stays light,
// test_policies.cpp:46-48), and deferred ids enter the heavy queue in id
// order. For every threshold t_k the output is that ordered id list.
//
// ONE pass, one launch (HBM-bound: the confidences are read once, 8 B are
// written per deferred query). Grid (tiles, thresholds); a CTA owns a tile of
// kTile confidences for one threshold:
//   * ingest: 128-bit loads (double2 / float4), striped so a warp reads 512
//     contiguous bytes per instruction; element e of row r, thread t, slot j
//     is tile_base + r*kThreads*V + t*V + j;
//   * count: warp ballots per (row, slot), popc -> per-warp row counts in
//     shared memory -> the tile's deferral count;
//   * decoupled look-back (single-pass scan): the tile publishes its count
//     (status A), warp 0 walks the predecessors' flags 32 at a time back to
//     the nearest inclusive prefix (status P), then publishes its own P. A
//     flag word is [epoch:20 | status:2 | value:42]; the epoch is bumped per
//     launch, so stale words from earlier launches read as "not ready" and no
//     memset is needed between launches. Tiles of a threshold are blockIdx.x
//     in dispatch order, so every predecessor is running or done;
//   * scatter: exclusive prefix + rows before + warps before + the lane's rank
//     among the warp's deferrals of that row: ordered, coalesced id writes.
#include <cuda_runtime.h>

#include "ds_internal.h"

namespace {

constexpr int kThreads = 256;
constexpr int kPerThread = 16;                 // confidences per thread
constexpr int kTile = kThreads * kPerThread;   // 4096 per tile
constexpr int kWarps = kThreads / 32;
constexpr unsigned long long kValBits = 42, kValMask = (1ull << kValBits) - 1;
constexpr unsigned kEpochBits = 20;
constexpr unsigned long long kStatusA = 1, kStatusP = 2;

template <typename T> struct Vec;
template <> struct Vec<double> {
    using type = double2;
    static constexpr int V = 2;
    __device__ static void get(const type& v, double (&o)[2]) { o[0] = v.x; o[1] = v.y; }
};
template <> struct Vec<float> {
    using type = float4;
    static constexpr int V = 4;
    __device__ static void get(const type& v, double (&o)[4]) {
        o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
    }
};

__device__ __forceinline__ unsigned long long flag_word(unsigned epoch, unsigned long long st,
                                                        long long v) {
    return (static_cast<unsigned long long>(epoch) << (kValBits + 2)) | (st << kValBits) |
           (static_cast<unsigned long long>(v) & kValMask);
}
__device__ __forceinline__ void flag_store(unsigned long long* p, unsigned long long w) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(w) : "memory");
}
__device__ __forceinline__ unsigned long long flag_load(const unsigned long long* p) {
    unsigned long long w;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(w) : "l"(p) : "memory");
    return w;
}

// Exclusive prefix of this tile's count over tiles [0, tile) of one threshold
// (warp 0 only; every lane returns it).
__device__ long long look_back(const unsigned long long* flags, int tile, unsigned epoch) {
    const int lane = threadIdx.x & 31;
    long long excl = 0;
    for (int base = tile - 1;; base -= 32) {
        const int idx = base - lane;   // lane 0: the nearest predecessor
        unsigned long long st = kStatusP, val = 0;
        if (idx >= 0) {
            unsigned long long w;
            do {
                w = flag_load(flags + idx);
            } while ((w >> (kValBits + 2)) != epoch || ((w >> kValBits) & 3ull) == 0);
            st = (w >> kValBits) & 3ull;
            val = w & kValMask;
        }
        const unsigned pmask = __ballot_sync(0xffffffffu, st == kStatusP);
        const int stop = pmask ? __ffs(pmask) - 1 : 32;
        long long v = lane <= stop ? static_cast<long long>(val) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        excl += v;
        if (pmask) return excl;
    }
}

template <typename T>
__global__ void __launch_bounds__(kThreads)
route_kernel(const T* __restrict__ conf, long long n, const double* __restrict__ thr,
             unsigned long long* __restrict__ flags, unsigned epoch, long long index_base,
             long long* __restrict__ heavy_idx, long long* __restrict__ total_out) {
    using VT = Vec<T>;
    constexpr int V = VT::V, R = kPerThread / V;
    const int tile = blockIdx.x, k = blockIdx.y, tiles = gridDim.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const double t = thr[k];
    const long long base = static_cast<long long>(tile) * kTile;
    __shared__ int warp_cnt[R][kWarps];
    __shared__ long long s_excl;
    // ingest (128-bit, striped) and the predicate
    unsigned pred = 0;   // bit r*V + j
    const bool full = base + kTile <= n && (reinterpret_cast<uintptr_t>(conf) % 16) == 0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const long long e0 = base + static_cast<long long>(r) * kThreads * V + threadIdx.x * V;
        double c[V];
        if (full) {
            VT::get(__ldg(reinterpret_cast<const typename VT::type*>(conf + e0)), c);
        } else {
#pragma unroll
            for (int j = 0; j < V; ++j)
                c[j] = e0 + j < n ? static_cast<double>(__ldg(conf + e0 + j)) : 2.0;
        }
#pragma unroll
        for (int j = 0; j < V; ++j) pred |= (c[j] < t ? 1u : 0u) << (r * V + j);
    }
    // ballots -> per-warp row counts; the lane's rank inside its warp row
    unsigned char rank_in_row[R][V];
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        int before = 0, all = 0;
        unsigned b[V];
#pragma unroll
        for (int j = 0; j < V; ++j) {
            b[j] = __ballot_sync(0xffffffffu, (pred >> (r * V + j)) & 1u);
            before += __popc(b[j] & lt);
            all += __popc(b[j]);
        }
#pragma unroll
        for (int j = 0; j < V; ++j) {
            rank_in_row[r][j] = static_cast<unsigned char>(before);
            before += (pred >> (r * V + j)) & 1u;
        }
        if (lane == 0) warp_cnt[r][warp] = all;
    }
    __syncthreads();
    unsigned long long* fk = flags + static_cast<long long>(k) * tiles;
    if (warp == 0) {
        long long cnt = 0;
        for (int i = lane; i < R * kWarps; i += 32) cnt += (&warp_cnt[0][0])[i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        long long excl = 0;
        if (tile == 0) {
            if (lane == 0 && tiles > 1) flag_store(fk, flag_word(epoch, kStatusP, cnt));
        } else {
            if (lane == 0) flag_store(fk + tile, flag_word(epoch, kStatusA, cnt));
            excl = look_back(fk, tile, epoch);
            if (lane == 0 && tile < tiles - 1)
                flag_store(fk + tile, flag_word(epoch, kStatusP, excl + cnt));
        }
        if (lane == 0) {
            s_excl = excl;
            if (tile == tiles - 1) total_out[k] = excl + cnt;
        }
    }
    __syncthreads();
    // scatter in id order
    long long off = s_excl;
    long long* out = heavy_idx + static_cast<long long>(k) * n;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        int wb = 0, row = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            const int c = warp_cnt[r][w];
            wb += w < warp ? c : 0;
            row += c;
        }
        const long long e0 = base + static_cast<long long>(r) * kThreads * V + threadIdx.x * V;
#pragma unroll
        for (int j = 0; j < V; ++j)
            if ((pred >> (r * V + j)) & 1u) out[off + wb + rank_in_row[r][j]] = index_base + e0 + j;
        off += row;
    }
}

} // namespace

extern "C" size_t ds_route_scratch_bytes(int64_t n, int32_t n_thresholds) {
    (void)n;
    (void)n_thresholds;
    return 0;   // the look-back flags live in the context (epoch-tagged, reused)
}

namespace {

ds_status route_launch(ds_ctx* ctx, const void* conf, int32_t dtype, int64_t n,
                       const double* thresholds, int32_t nt, int64_t index_base,
                       int64_t* heavy_idx, int64_t* counts, cudaStream_t st) {
    const int64_t tiles = (n + kTile - 1) / kTile;
    if (tiles > 0x7fffffff || nt > 65535 || n >= (1ll << kValBits))
        return dsi::fail(DS_ERR_CAPACITY, "ds_route: too many queries, tiles or thresholds");
    // look-back flags: [nt][tiles] words in a context buffer, reused across
    // launches through the epoch tag; zeroed on growth and on epoch wrap
    const size_t need = sizeof(unsigned long long) * static_cast<size_t>(tiles) * nt;
    if (need > ctx->route_flags_bytes || ctx->route_epoch + 1 >= (1u << kEpochBits)) {
        if (need > ctx->route_flags_bytes) {
            if (ctx->route_flags) {
                DS_CUDA_TRY(cudaDeviceSynchronize());
                DS_CUDA_TRY(cudaFree(ctx->route_flags));
                ctx->route_flags = nullptr;
                ctx->route_flags_bytes = 0;
            }
            const size_t want = dsi::align_up(need < (1u << 16) ? (1u << 16) : need, 1u << 16);
            DS_CUDA_TRY(cudaMalloc(&ctx->route_flags, want));
            ctx->route_flags_bytes = want;
        }
        DS_CUDA_TRY(cudaMemsetAsync(ctx->route_flags, 0, ctx->route_flags_bytes, st));
        ctx->route_epoch = 0;
    }
    const unsigned epoch = ++ctx->route_epoch;
    dim3 grid(static_cast<unsigned>(tiles), static_cast<unsigned>(nt));
    auto* flags = static_cast<unsigned long long*>(ctx->route_flags);
    if (dtype == DS_CONF_F64)
        route_kernel<double><<<grid, kThreads, 0, st>>>(
            static_cast<const double*>(conf), n, thresholds, flags, epoch, index_base,
            reinterpret_cast<long long*>(heavy_idx), reinterpret_cast<long long*>(counts));
    else
        route_kernel<float><<<grid, kThreads, 0, st>>>(
            static_cast<const float*>(conf), n, thresholds, flags, epoch, index_base,
            reinterpret_cast<long long*>(heavy_idx), reinterpret_cast<long long*>(counts));
    DS_LAUNCH_CHECK(ctx, "route_kernel");
    return DS_OK;
}

} // namespace

// Device variant: `counts` must be device memory. The look-back flags come
// from the ctx (stream-ordered: calls on one ctx from several streams must not
// overlap).
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
    return route_launch(ctx, conf, dtype, n, thresholds, nt, index_base, heavy_idx, counts, st);
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
    const size_t bi = dsi::align_up(sizeof(int64_t) * n * nt, 256);
    char* d = nullptr;
    ds_status s = dsi::ensure_scratch(ctx, bc + bt + bk + bi, reinterpret_cast<void**>(&d));
    if (s != DS_OK) return s;
    DS_CUDA_TRY(cudaMemcpyAsync(d, conf, esz * n, cudaMemcpyHostToDevice, ctx->stream));
    DS_CUDA_TRY(cudaMemcpyAsync(d + bc, thresholds, sizeof(double) * nt, cudaMemcpyHostToDevice,
                                ctx->stream));
    int64_t* dcounts = reinterpret_cast<int64_t*>(d + bc + bt);
    int64_t* didx = reinterpret_cast<int64_t*>(d + bc + bt + bk);
    s = route_launch(ctx, d, dtype, n, reinterpret_cast<double*>(d + bc), nt, index_base, didx,
                     dcounts, ctx->stream);
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
