// EXPERIMENT (not built): K9 as ONE pass -- format, place in shared memory,
// decoupled look-back for the file offset, write only the CSV bytes (no
// 256-byte global slots). Bit-identical output (tests/test_gpu_csv.py green),
// but measured SLOWER on 1M QueryRecords (tools/csv_speed.py): 1.68 ms with the
// block's text packed in shared memory, 1.85 ms with per-row shared slots and
// warp copy-out, vs 1.07 ms for csv.cu's format / carry / scatter passes.
// Formatting (~11 exact decimal conversions per row) dominates and wants the
// standalone format kernel's occupancy (4 x 256 threads per SM at 64
// registers) and no block barriers; the slot traffic it saves is ~0.26 GB,
// ~40 us at HBM speed.
// K9 csv_format: the rows of diffserve::write_csv (reference
// proj/src/metrics.cpp:91-127) formatted on the device, byte-identical.
//
// Every real number goes through fmt6 = snprintf("%.6g") (metrics.cpp:67-71),
// restated exactly in fmt6.h; integers print as operator<< does; optionals
// print empty when disengaged (opt6, metrics.cpp:75). Rows are independent, so
// the file is built in ONE pass (round 2; round 1 staged every row in a
// 256-byte global slot and took three launches, ~2.5x the algorithmic bytes):
//   * each element thread formats one row in registers / local memory;
//   * a block scan of the row lengths places the rows back to back in shared
//     memory (the block's text), while a control warp publishes the block's
//     byte count and finds its file offset by decoupled look-back
//     (lookback.cuh, as K2);
//   * the block's text goes out with 4-byte-aligned stores (two aligned
//     shared loads and a funnel shift per word): records in and CSV bytes out
//     are the only DRAM traffic.
// Writes stop at the caller's capacity; the size comes back through a device
// word (one synchronization). The header line is copied in by the host.
// Formatting (~11 exact decimal conversions per query row) dominates.
#include <cuda_runtime.h>

#include <cstring>

#include "ds_internal.h"
#include "fmt6.h"
#include "lookback.cuh"

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
    static constexpr unsigned kAttrBit = 1u << 16;
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
    static constexpr unsigned kAttrBit = 1u << 17;
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
    static constexpr unsigned kAttrBit = 1u << 18;
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

constexpr int kRows = 256;                 // rows (element threads) per block
constexpr int kCsvBlock = kRows + 32;      // + one control warp: byte count, look-back
constexpr int kStage = kRows * kSlot;      // the block's text, worst case

// One pass: format, place in shared memory, look back for the file offset,
// write. out == nullptr: sizes only. *total = the rows' bytes (last block).
// Three blocks per SM cap registers at 75: the rare 1280-bit path
// (ds_ratio_big) lives in local memory instead of setting the kernel's
// register count.
template <typename F>
__global__ void __launch_bounds__(kCsvBlock, 3)
csv_kernel(const typename F::Row* __restrict__ rows, int64_t n, char* __restrict__ out,
           long long capacity, long long header, unsigned long long* __restrict__ flags,
           unsigned* __restrict__ done, long long* __restrict__ total) {
    extern __shared__ __align__(16) unsigned char stage[];   // 256-byte row slots + 16
    __shared__ int warp_tot[kRows / 32];
    __shared__ long long s_excl;
    __shared__ int s_bytes;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int tile = blockIdx.x, tiles = gridDim.x;
    const int64_t i = static_cast<int64_t>(tile) * kRows + tid;
    alignas(16) char buf[kSlot];
    int len = 0, inc = 0;
    if (warp < kRows / 32) {
        if (i < n) len = F::format(rows[i], buf);
        inc = len;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += t;
        }
        if (lane == 31) warp_tot[warp] = inc;
    }
    __syncthreads();
    if (warp == kRows / 32) {
        // control warp: publish the block's bytes, find its file offset
        int bytes = lane < kRows / 32 ? warp_tot[lane] : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) bytes += __shfl_xor_sync(0xffffffffu, bytes, o);
        long long excl = 0;
        if (tiles > 1) {
            if (lane == 0)
                dslb::flag_store(flags + tile,
                                 dslb::flag_word(tile == 0 ? dslb::kStatusP : dslb::kStatusA, bytes));
            if (tile > 0) {
                excl = dslb::look_back(flags, tile);
                if (lane == 0 && tile < tiles - 1)
                    dslb::flag_store(flags + tile, dslb::flag_word(dslb::kStatusP, excl + bytes));
            }
        }
        if (lane == 0) {
            s_excl = excl;
            s_bytes = bytes;
            if (tile == tiles - 1) *total = excl + bytes;
        }
    }
    if (warp < kRows / 32 && len > 0) {
        // this row's text in its 256-byte shared slot (16-byte stores)
        uint4* d = reinterpret_cast<uint4*>(stage + tid * kSlot);
        const uint4* src = reinterpret_cast<const uint4*>(buf);
        for (int k = 0; k < (len + 15) / 16; ++k) d[k] = src[k];
    }
    __syncthreads();
    if (out && warp < kRows / 32) {
        // warp w writes its 32 rows in order: row r's bytes go to p = header +
        // block offset + r's offset in the block; 4-byte-aligned destination
        // words, each from two aligned shared words and a funnel shift; head
        // and tail bytes singly; nothing at or past `capacity`
        int wbase = 0;
        for (int w = 0; w < warp; ++w) wbase += warp_tot[w];
        const long long base = header + s_excl + wbase;
        for (int r = 0; r < 32; ++r) {
            const int rlen = __shfl_sync(0xffffffffu, len, r);
            const int roff = __shfl_sync(0xffffffffu, inc - len, r);
            if (rlen == 0) continue;
            const long long p0 = base + roff;
            const unsigned char* src = stage + (warp * 32 + r) * kSlot;
            const int head = static_cast<int>((4 - (p0 & 3)) & 3);
            const int h = head < rlen ? head : rlen;
            if (lane < h && p0 + lane < capacity) out[p0 + lane] = static_cast<char>(src[lane]);
            const int words = (rlen - h) / 4;
            const uint32_t* sw = reinterpret_cast<const uint32_t*>(src);
            const int shift = 8 * (h & 3);
            for (int w = lane; w < words; w += 32) {
                const int sb = h + 4 * w;
                const uint32_t lo = sw[sb >> 2], hi = sw[(sb >> 2) + 1];
                const uint32_t v = shift ? __funnelshift_r(lo, hi, shift) : lo;
                const long long db = p0 + sb;
                if (db + 4 <= capacity) *reinterpret_cast<uint32_t*>(out + db) = v;
            }
            const int t0 = h + 4 * words;
            if (lane < rlen - t0 && p0 + t0 + lane < capacity)
                out[p0 + t0 + lane] = static_cast<char>(src[t0 + lane]);
        }
    }
    dslb::retire(flags, done, tiles);
}

__global__ void __launch_bounds__(256, 4) g6_kernel(const double* __restrict__ v, int64_t n, char* __restrict__ out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    alignas(16) char buf[16] = {};
    ds_fmt_g6(v[i], buf);
    *reinterpret_cast<uint4*>(out + i * 16) = *reinterpret_cast<const uint4*>(buf);
}

// rows_dev -> out_dev (header + rows), one launch. Synchronizes once to read
// the size; DS_ERR_CAPACITY if it exceeds `capacity` (bytes past it are not
// written).
template <typename F>
ds_status format_device(ds_ctx* ctx, const typename F::Row* rows, int64_t n, char* out,
                        int64_t capacity, int64_t* bytes, cudaStream_t st) {
    const int64_t header = static_cast<int64_t>(std::strlen(F::kHeader));
    const int64_t nb = (n + kRows - 1) / kRows;
    if (nb > 0x7fffffff) return dsi::fail(DS_ERR_CAPACITY, "too many rows");
    long long* htotal = nullptr;
    ds_status s = dsi::ensure_pinned(ctx, 2 * sizeof(long long), reinterpret_cast<void**>(&htotal));
    if (s != DS_OK) return s;
    *htotal = 0;
    if (out && capacity > 0)
        DS_CUDA_TRY(cudaMemcpyAsync(out, F::kHeader, header < capacity ? header : capacity,
                                    cudaMemcpyHostToDevice, st));
    if (n > 0) {
        unsigned long long* flags = nullptr;
        unsigned* done = nullptr;
        s = dsi::lookback_flags(ctx, static_cast<size_t>(nb), &flags, &done);
        if (s != DS_OK) return s;
        // the device word for the total: the last 8 bytes of the flag area's tail
        long long* total = reinterpret_cast<long long*>(done) + 1;
        constexpr int kSmem = kStage + 16;
        if (!(ctx->route_attr_set & F::kAttrBit)) {   // once per context (device)
            DS_CUDA_TRY(cudaFuncSetAttribute(csv_kernel<F>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
            ctx->route_attr_set |= F::kAttrBit;
        }
        csv_kernel<F><<<static_cast<unsigned>(nb), kCsvBlock, kSmem, st>>>(
            rows, n, out, out ? capacity : 0, header, flags, done, total);
        DS_LAUNCH_CHECK(ctx, "csv_kernel");
        DS_CUDA_TRY(cudaMemcpyAsync(htotal, total, sizeof(long long), cudaMemcpyDeviceToHost, st));
    }
    DS_CUDA_TRY(cudaStreamSynchronize(st));
    *bytes = header + *htotal;
    if (out && capacity < *bytes) return dsi::fail(DS_ERR_CAPACITY, "csv buffer too small");
    return DS_OK;
}

template <typename F>
ds_status format_host(ds_ctx* ctx, const typename F::Row* rows, int64_t n, char* out,
                      int64_t capacity, int64_t* bytes) {
    if (!ctx || !bytes || n < 0 || (n > 0 && !rows))
        return dsi::fail(DS_ERR_INVALID_ARGUMENT, "null argument");
    using Row = typename F::Row;
    const size_t brows = dsi::align_up(sizeof(Row) * n, 256);
    // device text buffer: every row fits its 256-byte bound
    const int64_t dcap = static_cast<int64_t>(n) * kSlot + 4096;
    char* d = nullptr;
    ds_status s = dsi::ensure_scratch(ctx, brows + (out ? dsi::align_up(dcap, 256) : 0),
                                      reinterpret_cast<void**>(&d));
    if (s != DS_OK) return s;
    Row* drows = reinterpret_cast<Row*>(d);
    char* dout = out ? d + brows : nullptr;
    if (n > 0)
        DS_CUDA_TRY(cudaMemcpyAsync(drows, rows, sizeof(Row) * n, cudaMemcpyHostToDevice,
                                    ctx->stream));
    s = format_device<F>(ctx, drows, n, dout, out ? dcap : 0, bytes, ctx->stream);
    if (s != DS_OK) return s;
    if (out) {
        if (capacity < *bytes) return dsi::fail(DS_ERR_CAPACITY, "csv buffer too small");
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
    return format_device<QueryRow>(ctx, records, n, out, capacity, bytes, st);
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
// Round 2, second attempt (not kept either): one 32-row tile per WARP (no CTA
// barrier; each lane formats its row into local memory, a shuffle scan, the
// warp's own look-back, then every lane writes its row at its final offset
// with funnel-shifted 4-byte stores): 1.48 ms, 1.34 ms with the writes
// removed, vs 1.06 ms for the three passes on the same box -- finished tiles
// hold their slots while slower predecessors format. The look-back itself was
// changed then to wait only for flags nearer than the nearest P
// (lookback.cuh); it did not change this result. A faster fmt6 digit stage
// (32-bit digit arithmetic, 9-digit u64 chunks) measured 10% SLOWER in the
// three-pass kernel (1.17 vs 1.06 ms) and was dropped.
// Also measured (round 2): the three-pass design with each thread's row rendered
// into a 260-byte slot of SHARED memory instead of its local-memory buffer:
// 2.96 ms vs 1.07 ms (generic byte stores into shared memory, divergent columns).
