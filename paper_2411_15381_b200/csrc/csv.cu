// K9 csv_format: the rows of diffserve::write_csv (reference
// proj/src/metrics.cpp:91-127) formatted on the device, byte-identical.
//
// Every real number goes through fmt6 = snprintf("%.6g") (metrics.cpp:67-71),
// restated exactly in fmt6.h; integers print as operator<< does; optionals
// print empty when disengaged (opt6, metrics.cpp:75). Rows are independent, so
// the file is built in three passes:
//   format  one thread per row renders into a 256-byte slot (local buffer,
//           16-byte stores) and a per-block byte count;
//   carry   one block: exclusive scan of the block counts (file offsets);
//   scatter per block: in-block exclusive scan of the row lengths, then each
//           warp copies its rows to their offsets, lanes on consecutive bytes.
// The header line is copied in by the host. Formatting (~11 exact decimal
// conversions per query row) dominates; the passes move ~3x the output bytes.
#include <cuda_runtime.h>

#include <cstring>

#include "ds_internal.h"
#include "fmt6.h"

static_assert(sizeof(ds_query_record) == 104, "ds_query_record layout");
static_assert(sizeof(ds_interval_snapshot) == 120, "ds_interval_snapshot layout");
static_assert(sizeof(ds_plan_log_entry) == 56, "ds_plan_log_entry layout");

namespace {

constexpr int kSlot = 256;
constexpr int kThreads = 256;

__device__ __forceinline__ int put(char* o, const char* s) {
    int n = 0;
    while (s[n]) {
        o[n] = s[n];
        ++n;
    }
    return n;
}

__device__ __forceinline__ int opt6(char* o, bool present, double v) {
    return present ? ds_fmt_g6(v, o) : 0;
}

struct QueryRow {
    using Row = ds_query_record;
    static constexpr const char* kHeader =
        "id,arrival,confidence,quality_light,quality_heavy,deadline,light_start,"
        "light_end,heavy_start,heavy_end,completion,outcome,delivered_quality\n";
    // metrics.cpp:108-114
    __device__ static int format(const Row& r, char* o) {
        int n = ds_fmt_u64(r.id, o);
        o[n++] = ',';
        n += ds_fmt_g6(r.arrival, o + n);
        o[n++] = ',';
        n += ds_fmt_g6(r.confidence, o + n);
        o[n++] = ',';
        n += ds_fmt_g6(r.quality_light, o + n);
        o[n++] = ',';
        n += ds_fmt_g6(r.quality_heavy, o + n);
        o[n++] = ',';
        n += ds_fmt_g6(r.deadline, o + n);
        o[n++] = ',';
        n += opt6(o + n, r.present & DS_REC_LIGHT_START, r.light_start);
        o[n++] = ',';
        n += opt6(o + n, r.present & DS_REC_LIGHT_END, r.light_end);
        o[n++] = ',';
        n += opt6(o + n, r.present & DS_REC_HEAVY_START, r.heavy_start);
        o[n++] = ',';
        n += opt6(o + n, r.present & DS_REC_HEAVY_END, r.heavy_end);
        o[n++] = ',';
        n += opt6(o + n, r.present & DS_REC_COMPLETION, r.completion);
        o[n++] = ',';
        if (r.present & DS_REC_OUTCOME) {   // to_string(Outcome), metrics.cpp:11-19
            switch (r.outcome) {
            case DS_OUTCOME_SERVED_LIGHT: n += put(o + n, "served_light"); break;
            case DS_OUTCOME_SERVED_HEAVY: n += put(o + n, "served_heavy"); break;
            case DS_OUTCOME_DROPPED: n += put(o + n, "dropped"); break;
            case DS_OUTCOME_LATE: n += put(o + n, "late"); break;
            default: n += put(o + n, "?"); break;
            }
        }
        o[n++] = ',';
        n += opt6(o + n, r.present & DS_REC_DELIVERED_QUALITY, r.delivered_quality);
        o[n++] = '\n';
        return n;
    }
};

struct IntervalRow {
    using Row = ds_interval_snapshot;
    static constexpr const char* kHeader =
        "interval_start,demand_observed,demand_estimated,threshold,x1,x2,b1,b2,"
        "feasible,arrived,served_light,served_heavy,dropped,late,"
        "mean_delivered_quality\n";
    // metrics.cpp:95-102
    __device__ static int format(const Row& s, char* o) {
        int n = ds_fmt_g6(s.interval_start, o);
        o[n++] = ',';
        n += ds_fmt_g6(s.demand_observed, o + n);
        o[n++] = ',';
        n += ds_fmt_g6(s.demand_estimated, o + n);
        o[n++] = ',';
        n += ds_fmt_g6(s.threshold, o + n);
        o[n++] = ',';
        n += ds_fmt_i64(s.plan.x1, o + n);
        o[n++] = ',';
        n += ds_fmt_i64(s.plan.x2, o + n);
        o[n++] = ',';
        n += ds_fmt_i64(s.plan.b1, o + n);
        o[n++] = ',';
        n += ds_fmt_i64(s.plan.b2, o + n);
        o[n++] = ',';
        o[n++] = s.plan.feasible ? '1' : '0';
        o[n++] = ',';
        n += ds_fmt_u64(s.arrived, o + n);
        o[n++] = ',';
        n += ds_fmt_u64(s.served_light, o + n);
        o[n++] = ',';
        n += ds_fmt_u64(s.served_heavy, o + n);
        o[n++] = ',';
        n += ds_fmt_u64(s.dropped, o + n);
        o[n++] = ',';
        n += ds_fmt_u64(s.late, o + n);
        o[n++] = ',';
        n += opt6(o + n, s.has_mean_delivered_quality, s.mean_delivered_quality);
        o[n++] = '\n';
        return n;
    }
};

struct PlanRow {
    using Row = ds_plan_log_entry;
    static constexpr const char* kHeader =
        "tick,time,demand_estimated,threshold,x1,x2,b1,b2,feasible\n";
    // metrics.cpp:120-123
    __device__ static int format(const Row& e, char* o) {
        int n = ds_fmt_i64(e.tick, o);
        o[n++] = ',';
        n += ds_fmt_g6(e.time, o + n);
        o[n++] = ',';
        n += ds_fmt_g6(e.demand_estimated, o + n);
        o[n++] = ',';
        n += ds_fmt_g6(e.plan.threshold, o + n);
        o[n++] = ',';
        n += ds_fmt_i64(e.plan.x1, o + n);
        o[n++] = ',';
        n += ds_fmt_i64(e.plan.x2, o + n);
        o[n++] = ',';
        n += ds_fmt_i64(e.plan.b1, o + n);
        o[n++] = ',';
        n += ds_fmt_i64(e.plan.b2, o + n);
        o[n++] = ',';
        o[n++] = e.plan.feasible ? '1' : '0';
        o[n++] = '\n';
        return n;
    }
};

// min 4 blocks/SM caps registers at 64: the rare 1280-bit path (ds_ratio_big)
// lives in local memory instead of setting the whole kernel's register count.
template <typename F>
__global__ void __launch_bounds__(kThreads, 4)
format_kernel(const typename F::Row* __restrict__ rows, int64_t n, char* __restrict__ slots,
              int32_t* __restrict__ lens, long long* __restrict__ block_bytes) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x;
    int len = 0;
    if (i < n) {
        alignas(16) char buf[kSlot];
        len = F::format(rows[i], buf);
        uint4* dst = reinterpret_cast<uint4*>(slots + i * kSlot);
        const uint4* src = reinterpret_cast<const uint4*>(buf);
        for (int k = 0; k < (len + 15) / 16; ++k) dst[k] = src[k];
        lens[i] = len;
    }
    __shared__ int warp_sum[kThreads / 32];
    int s = len;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) warp_sum[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long b = 0;
        for (int w = 0; w < kThreads / 32; ++w) b += warp_sum[w];
        block_bytes[blockIdx.x] = b;
    }
}

// In place: block_bytes[b] <- bytes of blocks < b; total -> *total.
__global__ void __launch_bounds__(1024) carry_kernel(long long* __restrict__ block_bytes, int nb,
                                                     long long* __restrict__ total) {
    __shared__ long long warp_tot[32];
    long long run = 0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int base = 0; base < nb; base += 1024) {
        const int b = base + threadIdx.x;
        const long long v = b < nb ? block_bytes[b] : 0;
        long long inc = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += t;
        }
        if (lane == 31) warp_tot[warp] = inc;
        __syncthreads();
        if (warp == 0) {
            const long long w = warp_tot[lane];
            long long wi = w;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const long long t = __shfl_up_sync(0xffffffffu, wi, o);
                if (lane >= o) wi += t;
            }
            warp_tot[lane] = wi - w;
        }
        __syncthreads();
        const long long excl = run + warp_tot[warp] + inc - v;
        if (b < nb) block_bytes[b] = excl;
        __syncthreads();
        // the chunk total is the last thread's inclusive value
        __shared__ long long s_run;
        if (threadIdx.x == 1023) s_run = excl + v;
        __syncthreads();
        run = s_run;
        __syncthreads();
    }
    if (threadIdx.x == 0) *total = run;
}

__global__ void __launch_bounds__(kThreads)
scatter_kernel(const char* __restrict__ slots, const int32_t* __restrict__ lens, int64_t n,
               const long long* __restrict__ block_off, long long header,
               char* __restrict__ out) {
    __shared__ long long off[kThreads];
    __shared__ int warp_tot[kThreads / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t i = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x;
    const int len = i < n ? lens[i] : 0;
    int inc = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) warp_tot[warp] = inc;
    __syncthreads();
    int wbase = 0;
    for (int w = 0; w < warp; ++w) wbase += warp_tot[w];
    off[threadIdx.x] = header + block_off[blockIdx.x] + wbase + inc - len;
    __syncthreads();
    // warp w copies rows w*32 .. w*32+31 of this block
    for (int r = 0; r < 32; ++r) {
        const int row = warp * 32 + r;
        const int64_t gi = static_cast<int64_t>(blockIdx.x) * kThreads + row;
        if (gi >= n) break;
        const int rl = lens[gi];
        const char* src = slots + gi * kSlot;
        char* dst = out + off[row];
        for (int k = lane; k < rl; k += 32) dst[k] = src[k];
    }
}

__global__ void __launch_bounds__(256, 4) g6_kernel(const double* __restrict__ v, int64_t n, char* __restrict__ out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    alignas(16) char buf[16] = {};
    ds_fmt_g6(v[i], buf);
    *reinterpret_cast<uint4*>(out + i * 16) = *reinterpret_cast<const uint4*>(buf);
}

// rows_dev -> out_dev (header + rows). Synchronizes once to read the size.
template <typename F>
ds_status format_device(ds_ctx* ctx, const typename F::Row* rows, int64_t n, char* out,
                        int64_t capacity, int64_t* bytes, cudaStream_t st, void* work) {
    const int64_t header = static_cast<int64_t>(std::strlen(F::kHeader));
    const int64_t nb = (n + kThreads - 1) / kThreads;
    char* p = static_cast<char*>(work);
    char* slots = p;
    p += dsi::align_up(static_cast<size_t>(n) * kSlot, 256);
    int32_t* lens = reinterpret_cast<int32_t*>(p);
    p += dsi::align_up(sizeof(int32_t) * n, 256);
    long long* boff = reinterpret_cast<long long*>(p);
    p += dsi::align_up(sizeof(long long) * nb, 256);
    long long* total = reinterpret_cast<long long*>(p);
    long long* htotal = nullptr;
    ds_status s = dsi::ensure_pinned(ctx, sizeof(long long), reinterpret_cast<void**>(&htotal));
    if (s != DS_OK) return s;
    *htotal = 0;
    if (n > 0) {
        format_kernel<F><<<static_cast<unsigned>(nb), kThreads, 0, st>>>(rows, n, slots, lens,
                                                                          boff);
        DS_LAUNCH_CHECK(ctx, "format_kernel");
        carry_kernel<<<1, 1024, 0, st>>>(boff, static_cast<int>(nb), total);
        DS_LAUNCH_CHECK(ctx, "csv carry_kernel");
        DS_CUDA_TRY(cudaMemcpyAsync(htotal, total, sizeof(long long), cudaMemcpyDeviceToHost, st));
        DS_CUDA_TRY(cudaStreamSynchronize(st));
    }
    *bytes = header + *htotal;
    if (!out) return DS_OK;
    if (capacity < *bytes) return dsi::fail(DS_ERR_CAPACITY, "csv buffer too small");
    DS_CUDA_TRY(cudaMemcpyAsync(out, F::kHeader, header, cudaMemcpyHostToDevice, st));
    if (n > 0) {
        scatter_kernel<<<static_cast<unsigned>(nb), kThreads, 0, st>>>(slots, lens, n, boff,
                                                                       header, out);
        DS_LAUNCH_CHECK(ctx, "scatter_kernel");
    }
    return DS_OK;
}

template <typename F>
size_t work_bytes(int64_t n) {
    const int64_t nb = (n + kThreads - 1) / kThreads;
    return dsi::align_up(static_cast<size_t>(n) * kSlot, 256) +
           dsi::align_up(sizeof(int32_t) * n, 256) + dsi::align_up(sizeof(long long) * nb, 256) +
           256;
}

template <typename F>
ds_status format_host(ds_ctx* ctx, const typename F::Row* rows, int64_t n, char* out,
                      int64_t capacity, int64_t* bytes) {
    if (!ctx || !bytes || n < 0 || (n > 0 && !rows))
        return dsi::fail(DS_ERR_INVALID_ARGUMENT, "null argument");
    using Row = typename F::Row;
    const size_t brows = dsi::align_up(sizeof(Row) * n, 256);
    const size_t bwork = work_bytes<F>(n);
    const size_t bout = dsi::align_up(static_cast<size_t>(n) * kSlot + 4096, 256);
    char* d = nullptr;
    ds_status s = dsi::ensure_scratch(ctx, brows + bwork + bout, reinterpret_cast<void**>(&d));
    if (s != DS_OK) return s;
    Row* drows = reinterpret_cast<Row*>(d);
    char* dout = d + brows + bwork;
    if (n > 0)
        DS_CUDA_TRY(cudaMemcpyAsync(drows, rows, sizeof(Row) * n, cudaMemcpyHostToDevice,
                                    ctx->stream));
    s = format_device<F>(ctx, drows, n, out ? dout : nullptr, out ? capacity : 0, bytes,
                         ctx->stream, d + brows);
    if (s != DS_OK) return s;
    if (out) {
        DS_CUDA_TRY(cudaMemcpyAsync(out, dout, *bytes, cudaMemcpyDeviceToHost, ctx->stream));
        DS_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    }
    return DS_OK;
}

} // namespace

extern "C" ds_status ds_format_queries_csv(ds_ctx* ctx, const ds_query_record* records,
                                           int64_t n, char* out, int64_t capacity,
                                           int64_t* bytes) {
    return format_host<QueryRow>(ctx, records, n, out, capacity, bytes);
}

extern "C" ds_status ds_format_intervals_csv(ds_ctx* ctx, const ds_interval_snapshot* rows,
                                             int64_t n, char* out, int64_t capacity,
                                             int64_t* bytes) {
    return format_host<IntervalRow>(ctx, rows, n, out, capacity, bytes);
}

extern "C" ds_status ds_format_plans_csv(ds_ctx* ctx, const ds_plan_log_entry* rows, int64_t n,
                                         char* out, int64_t capacity, int64_t* bytes) {
    return format_host<PlanRow>(ctx, rows, n, out, capacity, bytes);
}

extern "C" ds_status ds_format_queries_csv_device(ds_ctx* ctx, const ds_query_record* records,
                                                  int64_t n, char* out, int64_t capacity,
                                                  int64_t* bytes, void* stream) {
    if (!ctx || !bytes || n < 0 || (n > 0 && !records))
        return dsi::fail(DS_ERR_INVALID_ARGUMENT, "null argument");
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
    void* work = nullptr;
    ds_status s = dsi::ensure_scratch(ctx, work_bytes<QueryRow>(n), &work);
    if (s != DS_OK) return s;
    return format_device<QueryRow>(ctx, records, n, out, capacity, bytes, st, work);
}

extern "C" ds_status ds_format_g6(ds_ctx* ctx, const double* values, int64_t n, char* out16) {
    if (!ctx || n < 0 || (n > 0 && (!values || !out16)))
        return dsi::fail(DS_ERR_INVALID_ARGUMENT, "null argument");
    if (n == 0) return DS_OK;
    const size_t bv = dsi::align_up(sizeof(double) * n, 256);
    char* d = nullptr;
    ds_status s = dsi::ensure_scratch(ctx, bv + 16 * n, reinterpret_cast<void**>(&d));
    if (s != DS_OK) return s;
    DS_CUDA_TRY(cudaMemcpyAsync(d, values, sizeof(double) * n, cudaMemcpyHostToDevice,
                                ctx->stream));
    g6_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, ctx->stream>>>(
        reinterpret_cast<const double*>(d), n, d + bv);
    DS_LAUNCH_CHECK(ctx, "g6_kernel");
    DS_CUDA_TRY(cudaMemcpyAsync(out16, d + bv, 16 * n, cudaMemcpyDeviceToHost, ctx->stream));
    DS_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    return DS_OK;
}
