// K2 route_compact: threshold routing with order-preserving stream compaction.
//
// Replaces the per-query Policy::defers loop of the light-batch completion
// handler (reference proj/src/cluster.cpp:290-306, proj/src/policies.cpp:37-39):
// a query defers iff confidence < t (strict; c == t stays light,
// test_policies.cpp:46-48), and deferred ids enter the heavy queue in id
// order. For every threshold t_k the output is that ordered id list.
//
// ONE pass, one launch (HBM-bound: the confidences are read once, 8 B are
// written per deferred query). Grid (tiles, thresholds); a CTA of 8 element
// warps + 1 control warp owns a tile of 8,192 confidences for one threshold:
//   * ingest: 128-bit loads (double2 / float4), all in flight before the
//     first use, striped so a warp reads 512 contiguous bytes per
//     instruction; element e of row r, thread t, slot j is
//     tile_base + r*kThreads*V + t*V + j;
//   * count: warp ballots per (row, slot), popc -> per-warp row counts in
//     shared memory -> the tile's deferral count;
//   * decoupled look-back (single-pass scan), by the control warp: publish
//     the tile's count (status A; tile 0 publishes its prefix, status P),
//     read the 128 nearest predecessors' flags at once back to the nearest P,
//     publish its own P. A flag word is [status:2 | value:62]. Tiles of a
//     threshold are blockIdx.x in dispatch order, so every predecessor is
//     running or done. The last CTA to retire (a done counter) zeroes the
//     flags, so every launch -- eager or replayed from a CUDA graph -- starts
//     from clean flags without a memset;
//   * meanwhile the element warps stage the tile's deferred ids in shared
//     memory at their tile-local rank (row offsets by a shuffle scan,
//     branch-free stores), then the whole CTA copies them out at the
//     exclusive prefix with 16-byte stores: ordered, coalesced id writes.
// Measured (tools/route_speed.py, CUDA-graph GPU time; DS_ROUTE_TRACE=1 prints
// per-phase times): 1M f64 at t = 0.5 in 6.0 us (was 17.4 us as a count pass
// + scatter pass with scalar loads).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "ds_internal.h"
#include "lookback.cuh"

namespace {

using namespace dslb;

constexpr int kThreads = 256;                  // element threads (8 warps)
constexpr int kBlock = kThreads + 32;          // + one control warp: count, look-back
constexpr int kPerThreadMax = 32;              // confidences per thread (<= 32: one bit each)
constexpr int kWarps = kThreads / 32;
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

template <typename T, int kPerThread>
__global__ void __launch_bounds__(kBlock)
route_kernel(const T* __restrict__ conf, long long n, const double* __restrict__ thr,
             unsigned long long* __restrict__ flags, unsigned* __restrict__ done,
             long long index_base,
             long long* __restrict__ heavy_idx, long long* __restrict__ total_out, int exp,
             unsigned long long* __restrict__ trace) {
    using VT = Vec<T>;
    constexpr int V = VT::V, R = kPerThread / V, kTile = kThreads * kPerThread;
    auto stamp = [&](int slot) {   // debug (DS_ROUTE_TRACE): phase times per tile
        if (trace && blockIdx.y == 0) {   // callers: one thread
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            trace[blockIdx.x * 6 + slot] = t;
        }
    };
    if (threadIdx.x == 0) stamp(0);
    const int tile = blockIdx.x, k = blockIdx.y, tiles = gridDim.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const double t = thr[k];
    const long long base = static_cast<long long>(tile) * kTile;
    __shared__ int warp_cnt[R][kWarps];
    __shared__ long long s_excl;
    __shared__ int s_cnt;
    extern __shared__ __align__(16) unsigned char dyn_smem[];   // kTile staged ids + 32
    unsigned pred = 0;   // bit r*V + j (kPerThread <= 32 bits)
    const unsigned lt = (1u << lane) - 1u;
    if (warp < kWarps) {
        // ingest (128-bit, striped; every load in flight before the first use)
        // and the predicate
        const bool full = base + kTile <= n && (reinterpret_cast<uintptr_t>(conf) % 16) == 0;
        if (full) {
            typename VT::type v[R];
#pragma unroll
            for (int r = 0; r < R; ++r)
                v[r] = __ldg(reinterpret_cast<const typename VT::type*>(
                    conf + base + static_cast<long long>(r) * kThreads * V + threadIdx.x * V));
#pragma unroll
            for (int r = 0; r < R; ++r) {
                double c[V];
                VT::get(v[r], c);
#pragma unroll
                for (int j = 0; j < V; ++j) pred |= (c[j] < t ? 1u : 0u) << (r * V + j);
            }
        } else {
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const long long e0 = base + static_cast<long long>(r) * kThreads * V + threadIdx.x * V;
#pragma unroll
                for (int j = 0; j < V; ++j) {
                    const double c = e0 + j < n ? static_cast<double>(__ldg(conf + e0 + j)) : 2.0;
                    pred |= (c < t ? 1u : 0u) << (r * V + j);
                }
            }
        }
        // ballots -> per-warp row counts
#pragma unroll
        for (int r = 0; r < R; ++r) {
            int all = 0;
#pragma unroll
            for (int j = 0; j < V; ++j)
                all += __popc(__ballot_sync(0xffffffffu, (pred >> (r * V + j)) & 1u));
            if (lane == 0) warp_cnt[r][warp] = all;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) stamp(1);
    unsigned long long* fk = flags + static_cast<long long>(k) * tiles;
    long long* sid = reinterpret_cast<long long*>(dyn_smem);
    if (warp == kWarps) {
        // control warp: publish the tile's count (successors wait on it),
        // then its exclusive prefix over the predecessors (decoupled
        // look-back), while the element warps stage their ids
        long long cnt = 0;
        for (int i = lane; i < R * kWarps; i += 32) cnt += (&warp_cnt[0][0])[i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        if (lane == 0 && !(exp & 1) && tiles > 1)
            flag_store(fk + tile, flag_word(tile == 0 ? kStatusP : kStatusA, cnt));
        if (lane == 0) stamp(2);
        long long excl = 0;
        if (!(exp & 1) && tile > 0) {
            excl = look_back(fk, tile);
            if (lane == 0 && tile < tiles - 1)
                flag_store(fk + tile, flag_word(kStatusP, excl + cnt));
        }
        if (lane == 0) {
            stamp(3);
            s_excl = excl;
            s_cnt = static_cast<int>(cnt);
            if (tile == tiles - 1) total_out[k] = excl + cnt;
        }
    } else {
        // the tile's deferred ids in id order, staged in shared memory at their
        // tile-local rank (rows before + warps before in the row + the lane's rank
        // among its warp's deferrals of the row) -- while the control warp looks back
        {
            // lane r < R: row r's total and this warp's start inside it, then an
            // exclusive scan of the row totals over the lanes (shuffles) -- every
            // row's base offset for this warp in a handful of dependent steps
            int my_off = 0;
            {
                int before = 0, tot = 0;
                if (lane < R) {
#pragma unroll
                    for (int w = 0; w < kWarps; ++w) {
                        const int c = warp_cnt[lane][w];
                        before += w < warp ? c : 0;
                        tot += c;
                    }
                }
                int incl = tot;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += y;
                }
                my_off = incl - tot + before;
            }
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int row_off = __shfl_sync(0xffffffffu, my_off, r);
                unsigned b[V];
                int before = 0;
#pragma unroll
                for (int j = 0; j < V; ++j) {
                    b[j] = __ballot_sync(0xffffffffu, (pred >> (r * V + j)) & 1u);
                    before += __popc(b[j] & lt);
                }
                const long long e0 = base + static_cast<long long>(r) * kThreads * V + threadIdx.x * V;
                // branch-free: a query that stays light writes its lane's
                // dummy slot past the tile (a divergent store per element
                // measured ~1.3 us per 1M queries)
#pragma unroll
                for (int j = 0; j < V; ++j) {
                    const unsigned f = (pred >> (r * V + j)) & 1u;
                    sid[f ? row_off + before : kTile + lane] = index_base + e0 + j;
                    before += f;
                }
            }
        }
    }
    __syncthreads();   // s_excl and the staged ids
    if (threadIdx.x == 0) stamp(4);
    // coalesced copy-out of [s_excl, s_excl + cnt) of row k: 16-byte stores
    // once the destination is 16-byte aligned
    const int tcnt = s_cnt;
    long long* out = heavy_idx + static_cast<long long>(k) * n + s_excl;
    const int head = (reinterpret_cast<uintptr_t>(out) & 15u) ? 1 : 0;
    if (head && threadIdx.x == 0 && tcnt > 0) out[0] = sid[0];
    const int pairs = (tcnt - head) / 2;
    // 4 independent pairs per thread per iteration: the shared loads of all
    // four are in flight before the first store
    for (int i0 = threadIdx.x; i0 < pairs; i0 += 4 * kBlock) {
        longlong2 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int i = i0 + u * kBlock;
            if (i < pairs) v[u] = make_longlong2(sid[head + 2 * i], sid[head + 2 * i + 1]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int i = i0 + u * kBlock;
            if (i < pairs) *reinterpret_cast<longlong2*>(out + head + 2 * i) = v[u];
        }
    }
    if (threadIdx.x == 0 && tcnt > head && ((tcnt - head) & 1)) out[tcnt - 1] = sid[tcnt - 1];
    if (threadIdx.x == 0) stamp(5);
    retire(flags, done, tiles);
}

} // namespace

extern "C" size_t ds_route_scratch_bytes(int64_t n, int32_t n_thresholds) {
    (void)n;
    (void)n_thresholds;
    return 0;   // the look-back flags live in the context (zeroed by each launch)
}

namespace {

template <int PT>
ds_status route_launch_pt(ds_ctx* ctx, const void* conf, int32_t dtype, int64_t n,
                          const double* thresholds, int32_t nt, int64_t index_base,
                          int64_t* heavy_idx, int64_t* counts, cudaStream_t st) {
    constexpr int kTile = kThreads * PT;
    const int64_t tiles = (n + kTile - 1) / kTile;
    if (tiles > 0x7fffffff || nt > 65535)
        return dsi::fail(DS_ERR_CAPACITY, "ds_route: too many tiles or thresholds");
    unsigned long long* flags = nullptr;
    unsigned* done = nullptr;
    ds_status s = dsi::lookback_flags(ctx, static_cast<size_t>(tiles) * nt, &flags, &done);
    if (s != DS_OK) return s;
    static const int exp = getenv("DS_ROUTE_EXP") ? atoi(getenv("DS_ROUTE_EXP")) : 0;
    dim3 grid(static_cast<unsigned>(tiles), static_cast<unsigned>(nt));
    constexpr int kSmem = (kTile + 32) * sizeof(long long);   // + one dummy slot per lane
    if (kSmem > 48 * 1024 && !(ctx->route_attr_set & (1u << (PT / 8)))) {   // once per device
        DS_CUDA_TRY(cudaFuncSetAttribute(route_kernel<double, PT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
        DS_CUDA_TRY(cudaFuncSetAttribute(route_kernel<float, PT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
        ctx->route_attr_set |= 1u << (PT / 8);
    }
    static unsigned long long* trace = nullptr;   // debug: DS_ROUTE_TRACE=1
    static const bool want_trace = getenv("DS_ROUTE_TRACE") != nullptr;
    if (want_trace && !trace) DS_CUDA_TRY(cudaMalloc(&trace, 6 * 8 * 65536));
    unsigned long long* tr = want_trace && tiles <= 65536 ? trace : nullptr;
    if (tr) DS_CUDA_TRY(cudaMemsetAsync(tr, 0, 6 * 8 * tiles, st));
    if (dtype == DS_CONF_F64)
        route_kernel<double, PT><<<grid, kBlock, kSmem, st>>>(
            static_cast<const double*>(conf), n, thresholds, flags, done, index_base,
            reinterpret_cast<long long*>(heavy_idx), reinterpret_cast<long long*>(counts), exp, tr);
    else
        route_kernel<float, PT><<<grid, kBlock, kSmem, st>>>(
            static_cast<const float*>(conf), n, thresholds, flags, done, index_base,
            reinterpret_cast<long long*>(heavy_idx), reinterpret_cast<long long*>(counts), exp, tr);
    DS_LAUNCH_CHECK(ctx, "route_kernel");
    if (tr) {
        std::vector<unsigned long long> h(6 * tiles);
        DS_CUDA_TRY(cudaMemcpyAsync(h.data(), tr, 8 * h.size(), cudaMemcpyDeviceToHost, st));
        DS_CUDA_TRY(cudaStreamSynchronize(st));
        unsigned long long t0 = ~0ull;
        for (int64_t i = 0; i < tiles; ++i) t0 = h[6 * i] < t0 ? h[6 * i] : t0;
        const char* names[6] = {"start", "counted", "A published", "looked back", "staged", "written"};
        fprintf(stderr, "route n=%lld nt=%d tiles=%lld (ns from the first CTA start):", (long long)n,
                nt, (long long)tiles);
        for (int sl = 0; sl < 6; ++sl) {
            std::vector<long long> v;
            for (int64_t i = 0; i < tiles; ++i)
                if (h[6 * i + sl]) v.push_back(static_cast<long long>(h[6 * i + sl] - t0));
            if (v.empty()) continue;
            std::sort(v.begin(), v.end());
            fprintf(stderr, " | %s min %lld med %lld max %lld", names[sl], v.front(), v[v.size() / 2],
                    v.back());
        }
        fprintf(stderr, "\n");
    }
    return DS_OK;
}

// Tiles of 8,192 (32 per thread): 1M queries = 123 tiles, one look-back
// round. Measured slower (tools/route_speed.py, CUDA-graph GPU time, 1M f64):
// 4,096 per tile 14.0 us, 2,048 per tile 13.9 us (longer look-back chains).
ds_status route_launch(ds_ctx* ctx, const void* conf, int32_t dtype, int64_t n,
                       const double* thresholds, int32_t nt, int64_t index_base,
                       int64_t* heavy_idx, int64_t* counts, cudaStream_t st) {
    return route_launch_pt<kPerThreadMax>(ctx, conf, dtype, n, thresholds, nt, index_base,
                                          heavy_idx, counts, st);
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
