// Multi-GPU plumbing of the hot path (include/ds_gpu.h "multi-GPU"; SURVEY.md
// 8(b) "NCCL-aware multi-GPU variant", 8(e)).
//
// The reference is one process, one thread: the heavy queue is
// one vector filled in id order (cluster.cpp:290-306), the deferral curve one
// object updated observation by observation (profiles.cpp:108-120), the plan
// one search over the whole grid (allocator.cpp:91-121). Sharded over ranks,
// each of those needs exactly one exchange, and only that exchange goes over
// the wire:
//   route   : [T] int64 routed counts all-gathered; a one-warp kernel turns
//             them into this rank's offset in every global queue (exclusive
//             scan over ranks) and the global lengths;
//   queues  : each rank's ordered ids (packed row after row) gathered at the
//             root, whose place kernel writes every (rank, threshold) block
//             at its offset -- rank order is global id order;
//   curve   : the ordered confidences all-gathered (4-8 B per query), every
//             rank replays the global sequence with K3;
//   planner : packed u64 selection keys MIN-all-reduced (their unsigned order
//             is the reference's choice order, allocator.cpp:57-67).
// Transports: NCCL (dlopen'ed -- the process's libnccl.so.2 when torch or the
// host already loaded one), or caller-supplied host callbacks (ds_comm_ops)
// for hosts without NCCL and for several ranks sharing one GPU in tests.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "ds_internal.h"

namespace {

// ---- NCCL, resolved at run time ----------------------------------------------
struct NcclApi {
    bool ok = false;
    std::string err;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
    ncclResult_t (*CommUserRank)(const ncclComm_t, int*) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t,
                         cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            const char* e = dlerror();
            api.err = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
            return;
        }
        bool all = true;
        auto sym = [&](auto& fn, const char* name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
            if (!fn) {
                all = false;
                api.err += std::string(" missing ") + name;
            }
        };
        sym(api.GetUniqueId, "ncclGetUniqueId");
        sym(api.CommInitRank, "ncclCommInitRank");
        sym(api.CommInitAll, "ncclCommInitAll");
        sym(api.CommDestroy, "ncclCommDestroy");
        sym(api.CommCount, "ncclCommCount");
        sym(api.CommUserRank, "ncclCommUserRank");
        sym(api.AllGather, "ncclAllGather");
        sym(api.AllReduce, "ncclAllReduce");
        sym(api.Send, "ncclSend");
        sym(api.Recv, "ncclRecv");
        sym(api.GroupStart, "ncclGroupStart");
        sym(api.GroupEnd, "ncclGroupEnd");
        sym(api.GetErrorString, "ncclGetErrorString");
        api.ok = all;
    });
    return api;
}

ds_status nccl_fail(ncclResult_t r, const char* what) {
    const NcclApi& a = nccl();
    return dsi::fail(DS_ERR_COMM, std::string(what) + ": " +
                                      (a.GetErrorString ? a.GetErrorString(r) : "nccl error"));
}

#define DS_NCCL_TRY(expr, what)                                                  \
    do {                                                                         \
        ncclResult_t r_ = (expr);                                                \
        if (r_ != ncclSuccess) return nccl_fail(r_, what);                       \
    } while (0)

} // namespace

struct ds_comm {
    ds_ctx* ctx = nullptr;
    int nranks = 1, rank = 0;
    bool use_nccl = false;
    ncclComm_t nc = nullptr;
    bool owned = false;
    ds_comm_ops ops{};
    void* user = nullptr;
    // grow-only device scratch (separate from ctx->scratch, which the
    // single-GPU entry points called inside the sharded ones use)
    void* scratch = nullptr;
    size_t scratch_bytes = 0;
    void* host = nullptr;   // pinned staging for the host transport
    size_t host_bytes = 0;
    void* tabs = nullptr;   // pinned offset tables (never touched by the transport)
    size_t tabs_bytes = 0;
};

namespace {

ds_status comm_scratch(ds_comm* c, size_t bytes, char** out) {
    if (bytes > c->scratch_bytes) {
        if (c->scratch) {
            DS_CUDA_TRY(cudaDeviceSynchronize());
            DS_CUDA_TRY(cudaFree(c->scratch));
            c->scratch = nullptr;
            c->scratch_bytes = 0;
        }
        const size_t want = dsi::align_up(bytes < (1u << 20) ? (1u << 20) : bytes, 1u << 20);
        DS_CUDA_TRY(cudaMalloc(&c->scratch, want));
        c->scratch_bytes = want;
    }
    *out = static_cast<char*>(c->scratch);
    return DS_OK;
}

ds_status grow_pinned(void*& buf, size_t& have, size_t bytes, char** out) {
    if (bytes > have) {
        if (buf) {
            DS_CUDA_TRY(cudaDeviceSynchronize());
            DS_CUDA_TRY(cudaFreeHost(buf));
            buf = nullptr;
            have = 0;
        }
        const size_t want = dsi::align_up(bytes < (1u << 16) ? (1u << 16) : bytes, 1u << 16);
        DS_CUDA_TRY(cudaMallocHost(&buf, want));
        have = want;
    }
    *out = static_cast<char*>(buf);
    return DS_OK;
}

ds_status comm_host(ds_comm* c, size_t bytes, char** out) {
    return grow_pinned(c->host, c->host_bytes, bytes, out);
}

ds_status check_comm(ds_ctx* ctx, ds_comm* c) {
    if (!ctx || !c) return dsi::fail(DS_ERR_INVALID_ARGUMENT, "null ctx or comm");
    if (c->ctx != ctx) return dsi::fail(DS_ERR_INVALID_ARGUMENT, "comm belongs to another ctx");
    return DS_OK;
}

// ---- the three transport primitives ------------------------------------------

// recv[r * bytes .. ] = rank r's send (device buffers; send may alias nothing in recv)
// (NCCL is called even with one rank, so the one-GPU tests run the NCCL path.)
ds_status allgather(ds_comm* c, const void* send, void* recv, size_t bytes, cudaStream_t st) {
    if (bytes == 0) return DS_OK;
    if (c->use_nccl) {
        DS_NCCL_TRY(nccl().AllGather(send, recv, bytes, ncclUint8, c->nc, st), "ncclAllGather");
        return DS_OK;
    }
    char* h = nullptr;
    ds_status s = comm_host(c, bytes * (c->nranks + 1), &h);
    if (s != DS_OK) return s;
    if (c->nranks == 1) {
        if (send != recv)
            DS_CUDA_TRY(cudaMemcpyAsync(recv, send, bytes, cudaMemcpyDeviceToDevice, st));
        return DS_OK;
    }
    DS_CUDA_TRY(cudaMemcpyAsync(h, send, bytes, cudaMemcpyDeviceToHost, st));
    DS_CUDA_TRY(cudaStreamSynchronize(st));
    if (c->ops.allgather(h, h + bytes, bytes, c->user) != 0)
        return dsi::fail(DS_ERR_COMM, "host allgather callback failed");
    DS_CUDA_TRY(cudaMemcpyAsync(recv, h + bytes, bytes * c->nranks, cudaMemcpyHostToDevice, st));
    DS_CUDA_TRY(cudaStreamSynchronize(st));   // the staging is reused by the next call
    return DS_OK;
}

ds_status allreduce_min_u64(ds_comm* c, uint64_t* buf, size_t count, cudaStream_t st) {
    if (count == 0) return DS_OK;
    if (c->use_nccl) {
        DS_NCCL_TRY(nccl().AllReduce(buf, buf, count, ncclUint64, ncclMin, c->nc, st),
                    "ncclAllReduce");
        return DS_OK;
    }
    if (c->nranks == 1) return DS_OK;
    char* h = nullptr;
    ds_status s = comm_host(c, count * 8, &h);
    if (s != DS_OK) return s;
    DS_CUDA_TRY(cudaMemcpyAsync(h, buf, count * 8, cudaMemcpyDeviceToHost, st));
    DS_CUDA_TRY(cudaStreamSynchronize(st));
    if (c->ops.allreduce_min_u64(reinterpret_cast<uint64_t*>(h), count, c->user) != 0)
        return dsi::fail(DS_ERR_COMM, "host allreduce_min_u64 callback failed");
    DS_CUDA_TRY(cudaMemcpyAsync(buf, h, count * 8, cudaMemcpyHostToDevice, st));
    DS_CUDA_TRY(cudaStreamSynchronize(st));
    return DS_OK;
}

// Rank r contributes sizes[r] bytes (host array, known to every rank); root
// receives them back to back in rank order into recv (device).
ds_status gatherv(ds_comm* c, int root, const void* send, void* recv,
                  const std::vector<size_t>& sizes, cudaStream_t st) {
    size_t total = 0, mine_off = 0;
    for (int r = 0; r < c->nranks; ++r) {
        if (r == c->rank) mine_off = total;
        total += sizes[r];
    }
    const size_t mine = sizes[c->rank];
    if (c->use_nccl || c->nranks == 1) {
        if (c->rank == root && mine)
            DS_CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(recv) + mine_off, send, mine,
                                        cudaMemcpyDeviceToDevice, st));
        if (c->nranks == 1) return DS_OK;
        DS_NCCL_TRY(nccl().GroupStart(), "ncclGroupStart");
        if (c->rank == root) {
            size_t off = 0;
            for (int r = 0; r < c->nranks; ++r) {
                if (r != root && sizes[r])
                    DS_NCCL_TRY(nccl().Recv(static_cast<char*>(recv) + off, sizes[r], ncclUint8, r,
                                            c->nc, st),
                                "ncclRecv");
                off += sizes[r];
            }
        } else if (mine) {
            DS_NCCL_TRY(nccl().Send(send, mine, ncclUint8, root, c->nc, st), "ncclSend");
        }
        DS_NCCL_TRY(nccl().GroupEnd(), "ncclGroupEnd");
        return DS_OK;
    }
    char* h = nullptr;
    ds_status s = comm_host(c, mine + (c->rank == root ? total : 0) + 16, &h);
    if (s != DS_OK) return s;
    char* hr = h + dsi::align_up(mine, 16);
    if (mine) {
        DS_CUDA_TRY(cudaMemcpyAsync(h, send, mine, cudaMemcpyDeviceToHost, st));
        DS_CUDA_TRY(cudaStreamSynchronize(st));
    }
    if (c->ops.gatherv(h, c->rank == root ? hr : nullptr, sizes.data(), root, c->user) != 0)
        return dsi::fail(DS_ERR_COMM, "host gatherv callback failed");
    if (c->rank == root && total) {
        DS_CUDA_TRY(cudaMemcpyAsync(recv, hr, total, cudaMemcpyHostToDevice, st));
        DS_CUDA_TRY(cudaStreamSynchronize(st));
    }
    return DS_OK;
}

// ---- kernels --------------------------------------------------------------------

// g[r][k] gathered counts -> this rank's exclusive offset and the global total.
__global__ void rank_offsets_kernel(const long long* __restrict__ g, int nranks, int rank, int nt,
                                    long long* __restrict__ offsets, long long* __restrict__ totals) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nt; k += gridDim.x * blockDim.x) {
        long long before = 0, all = 0;
        for (int r = 0; r < nranks; ++r) {
            const long long v = g[static_cast<long long>(r) * nt + k];
            before += r < rank ? v : 0;
            all += v;
        }
        if (offsets) offsets[k] = before;
        if (totals) totals[k] = all;
    }
}

// Per (threshold k = blockIdx.y, rank r = blockIdx.z): copy `len` ids from
// src + src_off[r][k] to dst row k at dst_off[r][k]; 16-byte vector copies
// where both sides allow it (the common case: offsets are element counts of
// 8-byte ids, so pairs of ids).
__global__ void place_kernel(const long long* __restrict__ src, long long* __restrict__ dst,
                             long long dst_stride, const long long* __restrict__ tab, int nt) {
    const int k = blockIdx.y, r = blockIdx.z;
    const long long* t = tab + (static_cast<long long>(r) * nt + k) * 3;   // src_off, dst_off, len
    const long long so = t[0], dof = t[1], len = t[2];
    const long long* s = src + so;
    long long* d = dst + static_cast<long long>(k) * dst_stride + dof;
    const long long step = static_cast<long long>(gridDim.x) * blockDim.x;
    for (long long i = blockIdx.x * blockDim.x + threadIdx.x; i < len; i += step) d[i] = s[i];
}

// Rows k of a strided [nt][stride] id matrix, counts[k] each -> packed back
// to back (row order).
__global__ void pack_kernel(const long long* __restrict__ rows, long long stride,
                            const long long* __restrict__ tab, int nt,
                            long long* __restrict__ packed) {
    const int k = blockIdx.y;
    const long long off = tab[2 * k], len = tab[2 * k + 1];
    const long long* s = rows + static_cast<long long>(k) * stride;
    const long long step = static_cast<long long>(gridDim.x) * blockDim.x;
    for (long long i = blockIdx.x * blockDim.x + threadIdx.x; i < len; i += step)
        packed[off + i] = s[i];
}

} // namespace

// ---- lifecycle --------------------------------------------------------------------

extern "C" ds_status ds_comm_nccl_unique_id(uint8_t id[DS_NCCL_UNIQUE_ID_BYTES]) {
    if (!id) return dsi::fail(DS_ERR_INVALID_ARGUMENT, "null id");
    const NcclApi& a = nccl();
    if (!a.ok) return dsi::fail(DS_ERR_COMM, a.err);
    ncclUniqueId u;
    DS_NCCL_TRY(a.GetUniqueId(&u), "ncclGetUniqueId");
    static_assert(sizeof(u) == DS_NCCL_UNIQUE_ID_BYTES, "ncclUniqueId size");
    std::memcpy(id, &u, sizeof(u));
    return DS_OK;
}

extern "C" ds_status ds_comm_init_nccl(ds_ctx* ctx, int32_t nranks, int32_t rank,
                                       const uint8_t id[DS_NCCL_UNIQUE_ID_BYTES], ds_comm** out) {
    if (!ctx || !id || !out) return dsi::fail(DS_ERR_INVALID_ARGUMENT, "null argument");
    *out = nullptr;
    if (nranks < 1 || rank < 0 || rank >= nranks)
        return dsi::fail(DS_ERR_INVALID_ARGUMENT, "bad nranks/rank");
    const NcclApi& a = nccl();
    if (!a.ok) return dsi::fail(DS_ERR_COMM, a.err);
    DS_CUDA_TRY(cudaSetDevice(ctx->device));
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    ncclComm_t nc = nullptr;
    DS_NCCL_TRY(a.CommInitRank(&nc, nranks, u, rank), "ncclCommInitRank");
    ds_comm* c = new ds_comm();
    c->ctx = ctx;
    c->nranks = nranks;
    c->rank = rank;
    c->use_nccl = true;
    c->nc = nc;
    c->owned = true;
    *out = c;
    return DS_OK;
}

extern "C" ds_status ds_comm_wrap_nccl(ds_ctx* ctx, void* nccl_comm, ds_comm** out) {
    if (!ctx || !nccl_comm || !out) return dsi::fail(DS_ERR_INVALID_ARGUMENT, "null argument");
    *out = nullptr;
    const NcclApi& a = nccl();
    if (!a.ok) return dsi::fail(DS_ERR_COMM, a.err);
    ncclComm_t nc = static_cast<ncclComm_t>(nccl_comm);
    int n = 0, r = 0;
    DS_NCCL_TRY(a.CommCount(nc, &n), "ncclCommCount");
    DS_NCCL_TRY(a.CommUserRank(nc, &r), "ncclCommUserRank");
    ds_comm* c = new ds_comm();
    c->ctx = ctx;
    c->nranks = n;
    c->rank = r;
    c->use_nccl = true;
    c->nc = nc;
    c->owned = false;
    *out = c;
    return DS_OK;
}

extern "C" ds_status ds_comm_init_all(ds_ctx* const* ctxs, int32_t n, ds_comm** comms) {
    if (!ctxs || !comms || n < 1) return dsi::fail(DS_ERR_INVALID_ARGUMENT, "bad arguments");
    const NcclApi& a = nccl();
    if (!a.ok) return dsi::fail(DS_ERR_COMM, a.err);
    std::vector<int> devs(n);
    for (int i = 0; i < n; ++i) {
        if (!ctxs[i]) return dsi::fail(DS_ERR_INVALID_ARGUMENT, "null ctx");
        devs[i] = ctxs[i]->device;
        comms[i] = nullptr;
    }
    std::vector<ncclComm_t> nc(n, nullptr);
    DS_NCCL_TRY(a.CommInitAll(nc.data(), n, devs.data()), "ncclCommInitAll");
    for (int i = 0; i < n; ++i) {
        ds_comm* c = new ds_comm();
        c->ctx = ctxs[i];
        c->nranks = n;
        c->rank = i;
        c->use_nccl = true;
        c->nc = nc[i];
        c->owned = true;
        comms[i] = c;
    }
    return DS_OK;
}

extern "C" ds_status ds_comm_create_host(ds_ctx* ctx, int32_t nranks, int32_t rank,
                                         const ds_comm_ops* ops, void* user, ds_comm** out) {
    if (!ctx || !ops || !out) return dsi::fail(DS_ERR_INVALID_ARGUMENT, "null argument");
    *out = nullptr;
    if (nranks < 1 || rank < 0 || rank >= nranks)
        return dsi::fail(DS_ERR_INVALID_ARGUMENT, "bad nranks/rank");
    if (!ops->allgather || !ops->allreduce_min_u64 || !ops->gatherv)
        return dsi::fail(DS_ERR_INVALID_ARGUMENT, "ds_comm_ops: every callback is required");
    ds_comm* c = new ds_comm();
    c->ctx = ctx;
    c->nranks = nranks;
    c->rank = rank;
    c->ops = *ops;
    c->user = user;
    *out = c;
    return DS_OK;
}

extern "C" ds_status ds_comm_destroy(ds_comm* c) {
    if (!c) return DS_OK;
    cudaSetDevice(c->ctx->device);
    cudaDeviceSynchronize();
    if (c->scratch) cudaFree(c->scratch);
    if (c->host) cudaFreeHost(c->host);
    if (c->tabs) cudaFreeHost(c->tabs);
    if (c->use_nccl && c->owned && c->nc) nccl().CommDestroy(c->nc);
    delete c;
    return DS_OK;
}

extern "C" int32_t ds_comm_rank(const ds_comm* c) { return c ? c->rank : -1; }
extern "C" int32_t ds_comm_size(const ds_comm* c) { return c ? c->nranks : 0; }

extern "C" void ds_shard_range(int64_t n, int32_t nranks, int32_t rank, int64_t* lo, int64_t* hi) {
    if (nranks < 1 || rank < 0 || rank >= nranks || n < 0) {
        if (lo) *lo = 0;
        if (hi) *hi = 0;
        return;
    }
    // n * rank / nranks without overflow for n < 2^62 and nranks < 2^31
    const auto at = [&](int64_t r) {
        return static_cast<int64_t>((static_cast<__int128>(n) * r) / nranks);
    };
    if (lo) *lo = at(rank);
    if (hi) *hi = at(rank + 1);
}

// ---- sharded operations -----------------------------------------------------------

extern "C" ds_status ds_route_sharded_device(ds_ctx* ctx, ds_comm* comm, const void* conf,
                                             int32_t dtype, int64_t n_local,
                                             const double* thresholds, int32_t nt,
                                             int64_t index_base, int64_t* heavy_local,
                                             int64_t* counts_local, int64_t* rank_offsets,
                                             int64_t* global_counts, void* stream) {
    ds_status s = check_comm(ctx, comm);
    if (s != DS_OK) return s;
    if (nt <= 0) return DS_OK;
    if (!counts_local) return dsi::fail(DS_ERR_INVALID_ARGUMENT, "null counts_local");
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
    s = ds_route_device(ctx, conf, dtype, n_local, thresholds, nt, index_base, heavy_local,
                        counts_local, st);
    if (s != DS_OK) return s;
    if (!rank_offsets && !global_counts) return DS_OK;
    char* g = nullptr;
    const size_t row = sizeof(long long) * nt;
    s = comm_scratch(comm, row * comm->nranks, &g);
    if (s != DS_OK) return s;
    s = allgather(comm, counts_local, g, row, st);
    if (s != DS_OK) return s;
    rank_offsets_kernel<<<(nt + 127) / 128, 128, 0, st>>>(
        reinterpret_cast<const long long*>(g), comm->nranks, comm->rank, nt,
        reinterpret_cast<long long*>(rank_offsets), reinterpret_cast<long long*>(global_counts));
    DS_LAUNCH_CHECK(ctx, "rank_offsets_kernel");
    return DS_OK;
}

extern "C" ds_status ds_queue_gather_device(ds_ctx* ctx, ds_comm* comm, int32_t root,
                                            const int64_t* heavy_local, int64_t n_local,
                                            const int64_t* counts_local, int32_t nt,
                                            int64_t* global_heavy, int64_t global_stride,
                                            int64_t* global_counts, void* stream) {
    ds_status s = check_comm(ctx, comm);
    if (s != DS_OK) return s;
    if (root < 0 || root >= comm->nranks) return dsi::fail(DS_ERR_INVALID_ARGUMENT, "bad root");
    if (nt <= 0) return DS_OK;
    if (!counts_local || (n_local > 0 && !heavy_local))
        return dsi::fail(DS_ERR_INVALID_ARGUMENT, "null argument");
    const bool is_root = comm->rank == root;
    if (is_root && (!global_heavy || !global_counts))
        return dsi::fail(DS_ERR_INVALID_ARGUMENT, "root needs global_heavy and global_counts");
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
    const int R = comm->nranks;
    // 1. every rank's counts, on the host of every rank (the transfer sizes)
    const size_t row = sizeof(long long) * nt;
    char* dg = nullptr;
    s = comm_scratch(comm, dsi::align_up(row * R, 256), &dg);
    if (s != DS_OK) return s;
    s = allgather(comm, counts_local, dg, row, st);
    if (s != DS_OK) return s;
    std::vector<long long> g(static_cast<size_t>(R) * nt);
    DS_CUDA_TRY(cudaMemcpyAsync(g.data(), dg, row * R, cudaMemcpyDeviceToHost, st));
    DS_CUDA_TRY(cudaStreamSynchronize(st));
    std::vector<size_t> sizes(R);
    std::vector<long long> totals(nt, 0);
    size_t all = 0;
    for (int r = 0; r < R; ++r) {
        long long t = 0;
        for (int k = 0; k < nt; ++k) {
            const long long v = g[static_cast<size_t>(r) * nt + k];
            if (v < 0 || v > (r == comm->rank ? n_local : INT64_MAX / 16))
                return dsi::fail(DS_ERR_INVALID_ARGUMENT, "routed count out of range");
            t += v;
            totals[k] += v;
        }
        sizes[r] = sizeof(long long) * static_cast<size_t>(t);
        all += sizes[r];
    }
    if (is_root)
        for (int k = 0; k < nt; ++k)
            if (totals[k] > global_stride)
                return dsi::fail(DS_ERR_CAPACITY, "global_stride below a global queue's length");
    // 2. this rank's rows packed back to back (a single row is already packed)
    const size_t tab_pack = dsi::align_up(sizeof(long long) * 2 * nt, 256);
    const size_t tab_place = dsi::align_up(sizeof(long long) * 3 * nt * R, 256);
    const size_t packed_bytes = dsi::align_up(sizes[comm->rank], 256);
    const size_t staged_bytes = is_root ? dsi::align_up(all, 256) : 0;
    const size_t off_g = 0, off_tp = dsi::align_up(row * R, 256), off_tq = off_tp + tab_pack,
                 off_pk = off_tq + tab_place, off_sg = off_pk + packed_bytes;
    s = comm_scratch(comm, off_sg + staged_bytes + 256, &dg);
    if (s != DS_OK) return s;
    (void)off_g;
    char* hp = nullptr;
    s = grow_pinned(comm->tabs, comm->tabs_bytes, tab_pack + tab_place, &hp);
    if (s != DS_OK) return s;
    long long* ht_pack = reinterpret_cast<long long*>(hp);
    long long* ht_place = reinterpret_cast<long long*>(hp + tab_pack);
    const void* send = heavy_local;
    if (nt > 1) {
        long long off = 0;
        for (int k = 0; k < nt; ++k) {
            const long long v = g[static_cast<size_t>(comm->rank) * nt + k];
            ht_pack[2 * k] = off;
            ht_pack[2 * k + 1] = v;
            off += v;
        }
        DS_CUDA_TRY(cudaMemcpyAsync(dg + off_tp, ht_pack, sizeof(long long) * 2 * nt,
                                    cudaMemcpyHostToDevice, st));
        if (off > 0) {
            dim3 grid(static_cast<unsigned>((n_local + 1023) / 1024 < 8 ? (n_local + 1023) / 1024 : 8),
                      static_cast<unsigned>(nt));
            if (grid.x == 0) grid.x = 1;
            pack_kernel<<<grid, 256, 0, st>>>(reinterpret_cast<const long long*>(heavy_local),
                                              n_local, reinterpret_cast<const long long*>(dg + off_tp),
                                              nt, reinterpret_cast<long long*>(dg + off_pk));
            DS_LAUNCH_CHECK(ctx, "pack_kernel");
        }
        send = dg + off_pk;
    }
    // 3. gather at the root, rank order
    s = gatherv(comm, root, send, dg + off_sg, sizes, st);
    if (s != DS_OK) return s;
    if (!is_root) {
        // the pinned tables are reused by the next call on this comm
        DS_CUDA_TRY(cudaStreamSynchronize(st));
        return DS_OK;
    }
    // 4. root: every (rank, threshold) block to its offset in the global row
    long long base = 0;
    std::vector<long long> dst(nt, 0);
    for (int r = 0; r < R; ++r) {
        long long src = base;
        for (int k = 0; k < nt; ++k) {
            const long long v = g[static_cast<size_t>(r) * nt + k];
            long long* t = ht_place + (static_cast<size_t>(r) * nt + k) * 3;
            t[0] = src;
            t[1] = dst[k];
            t[2] = v;
            src += v;
            dst[k] += v;
        }
        base += static_cast<long long>(sizes[r] / sizeof(long long));
    }
    DS_CUDA_TRY(cudaMemcpyAsync(dg + off_tq, ht_place, sizeof(long long) * 3 * nt * R,
                                cudaMemcpyHostToDevice, st));
    DS_CUDA_TRY(cudaMemcpyAsync(global_counts, totals.data(), row, cudaMemcpyHostToDevice, st));
    if (all > 0) {
        long long mx = 0;
        for (long long v : g) mx = v > mx ? v : mx;
        dim3 grid(static_cast<unsigned>((mx + 1023) / 1024 < 16 ? (mx + 1023) / 1024 : 16),
                  static_cast<unsigned>(nt), static_cast<unsigned>(R));
        if (grid.x == 0) grid.x = 1;
        place_kernel<<<grid, 256, 0, st>>>(reinterpret_cast<const long long*>(dg + off_sg),
                                           reinterpret_cast<long long*>(global_heavy),
                                           global_stride,
                                           reinterpret_cast<const long long*>(dg + off_tq), nt);
        DS_LAUNCH_CHECK(ctx, "place_kernel");
    }
    // totals (a host vector) and the pinned tables must outlive the copies
    DS_CUDA_TRY(cudaStreamSynchronize(st));
    return DS_OK;
}

extern "C" ds_status ds_curve_observe_sharded_device(ds_ctx* ctx, ds_comm* comm, ds_curve* curve,
                                                     const void* conf_local, int32_t dtype,
                                                     const int64_t* shard_sizes, double decay,
                                                     void* stream) {
    ds_status s = check_comm(ctx, comm);
    if (s != DS_OK) return s;
    if (!curve || !shard_sizes) return dsi::fail(DS_ERR_INVALID_ARGUMENT, "null argument");
    if (dtype != DS_CONF_F64 && dtype != DS_CONF_F32)
        return dsi::fail(DS_ERR_INVALID_ARGUMENT, "unknown confidence dtype");
    const int R = comm->nranks;
    int64_t nmax = 0, total = 0;
    for (int r = 0; r < R; ++r) {
        if (shard_sizes[r] < 0) return dsi::fail(DS_ERR_INVALID_ARGUMENT, "negative shard size");
        nmax = shard_sizes[r] > nmax ? shard_sizes[r] : nmax;
        total += shard_sizes[r];
    }
    const int64_t mine = shard_sizes[comm->rank];
    if (mine > 0 && !conf_local) return dsi::fail(DS_ERR_INVALID_ARGUMENT, "null conf_local");
    if (total == 0) return DS_OK;
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
    const size_t esz = dtype == DS_CONF_F64 ? 8 : 4;
    const size_t slot = esz * static_cast<size_t>(nmax);
    bool ragged = false;
    for (int r = 0; r < R; ++r) ragged |= shard_sizes[r] != nmax;
    char* d = nullptr;
    const size_t b_send = dsi::align_up(slot, 256), b_all = dsi::align_up(slot * R, 256);
    s = comm_scratch(comm, b_send + 2 * b_all, &d);
    if (s != DS_OK) return s;
    const void* send = conf_local;
    if (mine < nmax) {   // the all-gather sends nmax elements from every rank
        if (mine)
            DS_CUDA_TRY(cudaMemcpyAsync(d, conf_local, esz * mine, cudaMemcpyDeviceToDevice, st));
        send = d;
    }
    char* all = d + b_send;
    s = allgather(comm, send, all, slot, st);
    if (s != DS_OK) return s;
    const void* seq = all;
    if (ragged) {   // back to back in rank (= id) order
        char* packed = all + b_all;
        size_t off = 0;
        for (int r = 0; r < R; ++r) {
            const size_t b = esz * static_cast<size_t>(shard_sizes[r]);
            if (b) DS_CUDA_TRY(cudaMemcpyAsync(packed + off, all + slot * r, b,
                                               cudaMemcpyDeviceToDevice, st));
            off += b;
        }
        seq = packed;
    }
    return ds_curve_observe_device(ctx, curve, seq, dtype, total, decay, st);
}

extern "C" ds_status ds_plan_sharded_device(ds_ctx* ctx, ds_comm* comm, const ds_problem* problems,
                                            int32_t n, const ds_cascade* cascades,
                                            int32_t n_cascades, const double* grid_values,
                                            const int32_t* grid_offsets, int32_t n_grids,
                                            int32_t t_lo, int32_t t_hi, ds_plan* out,
                                            void* stream) {
    ds_status s = check_comm(ctx, comm);
    if (s != DS_OK) return s;
    if (n <= 0) return DS_OK;
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
    char* d = nullptr;
    s = comm_scratch(comm, sizeof(uint64_t) * static_cast<size_t>(n), &d);
    if (s != DS_OK) return s;
    uint64_t* keys = reinterpret_cast<uint64_t*>(d);
    s = ds_plan_keys_device(ctx, problems, n, cascades, n_cascades, grid_values, grid_offsets,
                            n_grids, t_lo, t_hi, keys, st);
    if (s != DS_OK) return s;
    s = allreduce_min_u64(comm, keys, static_cast<size_t>(n), st);
    if (s != DS_OK) return s;
    return ds_plan_from_keys_device(ctx, problems, n, cascades, n_cascades, grid_values,
                                    grid_offsets, n_grids, keys, out, st);
}

extern "C" ds_status ds_comm_gather_device(ds_ctx* ctx, ds_comm* comm, int32_t root,
                                           const void* send, size_t bytes, void* recv,
                                           size_t recv_capacity, size_t* total_bytes,
                                           void* stream) {
    ds_status s = check_comm(ctx, comm);
    if (s != DS_OK) return s;
    if (root < 0 || root >= comm->nranks) return dsi::fail(DS_ERR_INVALID_ARGUMENT, "bad root");
    if (bytes > 0 && !send) return dsi::fail(DS_ERR_INVALID_ARGUMENT, "null send");
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
    const int R = comm->nranks;
    // every rank's byte count (8 bytes each) through the same transport
    char* d = nullptr;
    s = comm_scratch(comm, dsi::align_up(8, 256) + dsi::align_up(8 * R, 256), &d);
    if (s != DS_OK) return s;
    const unsigned long long mine = bytes;
    DS_CUDA_TRY(cudaMemcpyAsync(d, &mine, 8, cudaMemcpyHostToDevice, st));
    s = allgather(comm, d, d + 256, 8, st);
    if (s != DS_OK) return s;
    std::vector<unsigned long long> hs(R);
    DS_CUDA_TRY(cudaMemcpyAsync(hs.data(), d + 256, 8 * R, cudaMemcpyDeviceToHost, st));
    DS_CUDA_TRY(cudaStreamSynchronize(st));
    std::vector<size_t> sizes(R);
    size_t total = 0;
    for (int r = 0; r < R; ++r) total += sizes[r] = static_cast<size_t>(hs[r]);
    if (comm->rank == root) {
        if (total > recv_capacity || (total > 0 && !recv))
            return dsi::fail(DS_ERR_CAPACITY, "ds_comm_gather_device: recv too small");
        if (total_bytes) *total_bytes = total;
    }
    s = gatherv(comm, root, send, recv, sizes, st);
    if (s != DS_OK) return s;
    DS_CUDA_TRY(cudaStreamSynchronize(st));
    return DS_OK;
}
