// ds_multi: the score + route hot path over G GPUs of one node, driven from
// C++ through include/ds_gpu.h only (SURVEY.md 8(b) "NCCL-aware multi-GPU
// variant", 8(e); the reference's host is C++ -- experiment.cpp:76-87 -- and
// would drive the GPUs the same way).
//
// One process, G devices: ds_comm_init_all (ncclCommInitAll) and one host
// thread per device (the sharded calls are collective). Two workloads:
//   config 2 : images_per_gpu synthetic 512x512 images per GPU (contiguous
//              global id shards), discriminator -> route at the 101 grid
//              thresholds k/100 (cluster.cpp:20-28) with the routed-count
//              all-gather -> the global heavy queues assembled at rank 0 ->
//              the deferral curve over the global sequence (decay 0.999,
//              prior = the shipped samples, cascades.profiles:20);
//   config 5 : `queries` queries split over the GPUs, scored from each GPU's
//              resident image pool in chunks, routed at t = 0.5, queue
//              gathered at rank 0.
// --check 1 recomputes both on ONE GPU (rank 0 scores every rank's images
// itself) and requires the G-GPU queues, counts and curve bits to be equal.
// Prints one JSON line.
//
//   ds_multi [--gpus G] [--images-per-gpu N] [--queries Q] [--steps K]
//            [--warmup W] [--check 0|1]
#include <cuda_runtime.h>

#include <algorithm>
#include <barrier>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "ds_gpu.h"

namespace {

constexpr int kH = 512, kW = 512;
constexpr uint64_t kImgSeed = 1, kWeightSeed = 2024;
constexpr double kDecay = 0.999;
constexpr int64_t kPool = 5000;   // resident images per GPU for config 5

#define CK(x)                                                                          \
    do {                                                                               \
        ds_status s_ = (x);                                                            \
        if (s_ != DS_OK) {                                                             \
            std::fprintf(stderr, "%s:%d %s -> %d (%s)\n", __FILE__, __LINE__, #x,      \
                         static_cast<int>(s_), ds_last_error());                       \
            std::exit(1);                                                              \
        }                                                                              \
    } while (0)
#define CU(x)                                                                          \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess) {                                                       \
            std::fprintf(stderr, "%s:%d %s -> %s\n", __FILE__, __LINE__, #x,           \
                         cudaGetErrorString(e_));                                      \
            std::exit(1);                                                              \
        }                                                                              \
    } while (0)

std::vector<double> make_grid(double step) {   // cluster.cpp:20-28
    const int n = static_cast<int>(std::lround(1.0 / step));
    std::vector<double> g;
    for (int k = 0; k <= n; ++k) g.push_back(static_cast<double>(k) / n);
    return g;
}

ds_curve shipped_prior(ds_ctx* ctx) {
    // DeferralCurve::from_samples of the shipped 32 samples (profiles.cpp:75-83,
    // cascades.profiles:20) = observe_confidence at decay 1 from empty
    std::vector<double> s;
    for (int i = 0; i < 32; ++i) {
        char buf[32];
        std::snprintf(buf, sizeof buf, "%.4f", 0.2125 + 0.025 * i);
        s.push_back(std::strtod(buf, nullptr));
    }
    ds_curve c{};
    CK(ds_curve_observe(ctx, &c, s.data(), DS_CONF_F64, static_cast<int64_t>(s.size()), 1.0));
    return c;
}

template <typename T>
T* dalloc(size_t n) {
    T* p = nullptr;
    CU(cudaMalloc(&p, sizeof(T) * (n ? n : 1)));
    return p;
}

struct Result {
    double ms_step = 0, ms_scale = 0;
    bool queues_equal = true, counts_equal = true, curve_equal = true, scale_equal = true;
    long long routed50 = 0, scale_routed = 0;
};

}  // namespace

int main(int argc, char** argv) {
    int G = 0, steps = 10, warmup = 3, check = 1;
    int64_t per_gpu = 5000, queries = 1000000;
    for (int i = 1; i + 1 < argc; i += 2) {
        const std::string k = argv[i];
        const long long v = std::atoll(argv[i + 1]);
        if (k == "--gpus") G = static_cast<int>(v);
        else if (k == "--images-per-gpu") per_gpu = v;
        else if (k == "--queries") queries = v;
        else if (k == "--steps") steps = static_cast<int>(v);
        else if (k == "--warmup") warmup = static_cast<int>(v);
        else if (k == "--check") check = static_cast<int>(v);
        else {
            std::fprintf(stderr, "unknown argument %s\n", k.c_str());
            return 2;
        }
    }
    int avail = 0;
    CU(cudaGetDeviceCount(&avail));
    if (G <= 0) G = avail;
    if (G > avail) {
        std::fprintf(stderr, "--gpus %d > %d visible devices\n", G, avail);
        return 2;
    }
    std::vector<ds_ctx*> ctxs(G);
    for (int g = 0; g < G; ++g) CK(ds_ctx_create(g, &ctxs[g]));
    std::vector<ds_comm*> comms(G);
    CK(ds_comm_init_all(ctxs.data(), G, comms.data()));

    const std::vector<double> grid = make_grid(0.01);
    const int NT = static_cast<int>(grid.size());
    const int64_t N = per_gpu * G;
    const size_t img_bytes = static_cast<size_t>(kH) * kW * 3;
    std::barrier sync(G);
    std::vector<Result> res(G);
    std::vector<int64_t> sizes(G);
    for (int r = 0; r < G; ++r) sizes[r] = per_gpu;

    auto worker = [&](int r) {
        ds_ctx* ctx = ctxs[r];
        ds_comm* comm = comms[r];
        CU(cudaSetDevice(r));
        cudaStream_t st = static_cast<cudaStream_t>(ds_ctx_stream(ctx));
        ds_disc* disc = nullptr;
        CK(ds_disc_create(ctx, kWeightSeed, &disc));
        const int64_t id0 = r * per_gpu;
        uint8_t* images = dalloc<uint8_t>(img_bytes * std::max<int64_t>(per_gpu, kPool));
        CK(ds_synth_images_device(ctx, kImgSeed, id0, per_gpu, kH, kW, images, st));
        double* thr = dalloc<double>(NT);
        CU(cudaMemcpyAsync(thr, grid.data(), sizeof(double) * NT, cudaMemcpyHostToDevice, st));
        float* conf = dalloc<float>(per_gpu);
        int64_t* heavy = dalloc<int64_t>(static_cast<size_t>(NT) * per_gpu);
        int64_t* counts = dalloc<int64_t>(NT);
        int64_t* offs = dalloc<int64_t>(NT);
        int64_t* totals = dalloc<int64_t>(NT);
        const bool root = r == 0;
        int64_t* gq = root ? dalloc<int64_t>(static_cast<size_t>(NT) * N) : nullptr;
        int64_t* gc = root ? dalloc<int64_t>(NT) : nullptr;
        const ds_curve prior = shipped_prior(ctx);
        ds_curve* curve = dalloc<ds_curve>(1);

        auto step = [&] {
            CK(ds_disc_score_device(disc, images, per_gpu, kH, kW, conf, st));
            CK(ds_route_sharded_device(ctx, comm, conf, DS_CONF_F32, per_gpu, thr, NT, id0, heavy,
                                       counts, offs, totals, st));
            CK(ds_queue_gather_device(ctx, comm, 0, heavy, per_gpu, counts, NT, gq, N, gc, st));
            CU(cudaMemcpyAsync(curve, &prior, sizeof(ds_curve), cudaMemcpyHostToDevice, st));
            CK(ds_curve_observe_sharded_device(ctx, comm, curve, conf, DS_CONF_F32, sizes.data(),
                                               kDecay, st));
        };
        for (int i = 0; i < warmup; ++i) step();
        CU(cudaStreamSynchronize(st));
        sync.arrive_and_wait();
        cudaEvent_t a, b;
        CU(cudaEventCreate(&a));
        CU(cudaEventCreate(&b));
        CU(cudaEventRecord(a, st));
        for (int i = 0; i < steps; ++i) step();
        CU(cudaEventRecord(b, st));
        CU(cudaEventSynchronize(b));
        float ms = 0;
        CU(cudaEventElapsedTime(&ms, a, b));
        res[r].ms_step = ms / steps;
        sync.arrive_and_wait();

        // config 5: `queries` split over the GPUs, scored from the resident pool
        int64_t lo = 0, hi = 0;
        ds_shard_range(queries, G, r, &lo, &hi);
        const int64_t n5 = hi - lo;
        if (per_gpu < kPool)
            CK(ds_synth_images_device(ctx, kImgSeed, id0, kPool, kH, kW, images, st));
        float* conf5 = dalloc<float>(n5);
        int64_t* heavy5 = dalloc<int64_t>(n5);
        int64_t* cnt5 = dalloc<int64_t>(1);
        double* t5 = dalloc<double>(1);
        const double half = 0.5;
        CU(cudaMemcpyAsync(t5, &half, sizeof(double), cudaMemcpyHostToDevice, st));
        int64_t* gq5 = root ? dalloc<int64_t>(queries) : nullptr;
        int64_t* gc5 = root ? dalloc<int64_t>(1) : nullptr;
        auto scale_step = [&] {
            for (int64_t off = 0; off < n5; off += kPool) {
                const int64_t m = std::min(kPool, n5 - off);
                CK(ds_disc_score_device(disc, images, m, kH, kW, conf5 + off, st));
            }
            CK(ds_route_sharded_device(ctx, comm, conf5, DS_CONF_F32, n5, t5, 1, lo, heavy5, cnt5,
                                       nullptr, nullptr, st));
            CK(ds_queue_gather_device(ctx, comm, 0, heavy5, n5, cnt5, 1, gq5, queries, gc5, st));
        };
        scale_step();
        CU(cudaStreamSynchronize(st));
        sync.arrive_and_wait();
        CU(cudaEventRecord(a, st));
        scale_step();
        CU(cudaEventRecord(b, st));
        CU(cudaEventSynchronize(b));
        CU(cudaEventElapsedTime(&ms, a, b));
        res[r].ms_scale = ms;
        sync.arrive_and_wait();

        if (root && check) {
            // the same work on ONE GPU: every rank's images scored here
            float* call = dalloc<float>(std::max<int64_t>(N, kPool));
            for (int q = 0; q < G; ++q) {
                CK(ds_synth_images_device(ctx, kImgSeed, q * per_gpu, per_gpu, kH, kW, images, st));
                CK(ds_disc_score_device(disc, images, per_gpu, kH, kW, call + q * per_gpu, st));
            }
            int64_t* h1 = dalloc<int64_t>(static_cast<size_t>(NT) * N);
            int64_t* c1 = dalloc<int64_t>(NT);
            CK(ds_route_device(ctx, call, DS_CONF_F32, N, thr, NT, 0, h1, c1, st));
            ds_curve* cur1 = dalloc<ds_curve>(1);
            CU(cudaMemcpyAsync(cur1, &prior, sizeof(ds_curve), cudaMemcpyHostToDevice, st));
            CK(ds_curve_observe_device(ctx, cur1, call, DS_CONF_F32, N, kDecay, st));
            std::vector<int64_t> cg(NT), cs(NT), qg(static_cast<size_t>(NT) * N),
                qs(static_cast<size_t>(NT) * N);
            ds_curve vg, vs;
            CU(cudaMemcpyAsync(cg.data(), gc, 8 * NT, cudaMemcpyDeviceToHost, st));
            CU(cudaMemcpyAsync(cs.data(), c1, 8 * NT, cudaMemcpyDeviceToHost, st));
            CU(cudaMemcpyAsync(qg.data(), gq, 8 * qg.size(), cudaMemcpyDeviceToHost, st));
            CU(cudaMemcpyAsync(qs.data(), h1, 8 * qs.size(), cudaMemcpyDeviceToHost, st));
            CU(cudaMemcpyAsync(&vg, curve, sizeof vg, cudaMemcpyDeviceToHost, st));
            CU(cudaMemcpyAsync(&vs, cur1, sizeof vs, cudaMemcpyDeviceToHost, st));
            CU(cudaStreamSynchronize(st));
            res[r].counts_equal = cg == cs;
            for (int k = 0; k < NT && res[r].queues_equal; ++k)
                res[r].queues_equal = std::equal(qg.begin() + k * N, qg.begin() + k * N + cg[k],
                                                 qs.begin() + k * N);
            res[r].curve_equal = std::memcmp(&vg, &vs, sizeof vg) == 0;
            res[r].routed50 = cg[50];
            // config 5 on one GPU: every id's image is pool[id mod per-rank pool]
            // of ITS rank's pool; recompute rank by rank from the id ranges
            std::vector<int64_t> q5(queries), want;
            int64_t c5 = 0;
            CU(cudaMemcpyAsync(&c5, gc5, 8, cudaMemcpyDeviceToHost, st));
            CU(cudaMemcpyAsync(q5.data(), gq5, 8 * queries, cudaMemcpyDeviceToHost, st));
            CU(cudaStreamSynchronize(st));
            std::vector<float> pool_conf(kPool);
            for (int q = 0; q < G; ++q) {
                CK(ds_synth_images_device(ctx, kImgSeed, q * per_gpu, kPool, kH, kW, images, st));
                CK(ds_disc_score_device(disc, images, kPool, kH, kW, call, st));
                CU(cudaMemcpyAsync(pool_conf.data(), call, 4 * kPool, cudaMemcpyDeviceToHost, st));
                CU(cudaStreamSynchronize(st));
                int64_t qlo = 0, qhi = 0;
                ds_shard_range(queries, G, q, &qlo, &qhi);
                for (int64_t i = qlo; i < qhi; ++i)
                    if (static_cast<double>(pool_conf[(i - qlo) % kPool]) < 0.5) want.push_back(i);
            }
            res[r].scale_routed = c5;
            res[r].scale_equal = c5 == static_cast<int64_t>(want.size()) &&
                                 std::equal(want.begin(), want.end(), q5.begin());
            CU(cudaFree(call));
            CU(cudaFree(h1));
            CU(cudaFree(c1));
            CU(cudaFree(cur1));
        }
        CU(cudaStreamSynchronize(st));
        for (void* p : {static_cast<void*>(images), static_cast<void*>(thr),
                        static_cast<void*>(conf), static_cast<void*>(heavy),
                        static_cast<void*>(counts), static_cast<void*>(offs),
                        static_cast<void*>(totals), static_cast<void*>(curve),
                        static_cast<void*>(conf5), static_cast<void*>(heavy5),
                        static_cast<void*>(cnt5), static_cast<void*>(t5)})
            CU(cudaFree(p));
        if (gq) CU(cudaFree(gq));
        if (gc) CU(cudaFree(gc));
        if (gq5) CU(cudaFree(gq5));
        if (gc5) CU(cudaFree(gc5));
        CK(ds_disc_destroy(disc));
    };
    std::vector<std::thread> th;
    for (int r = 0; r < G; ++r) th.emplace_back(worker, r);
    for (auto& t : th) t.join();
    double ms = 0, ms5 = 0;
    for (const Result& x : res) {
        ms = std::max(ms, x.ms_step);
        ms5 = std::max(ms5, x.ms_scale);
    }
    const Result& r0 = res[0];
    std::printf(
        "{\"driver\": \"ds_multi (C++, one thread per GPU, ncclCommInitAll)\", \"gpus\": %d, "
        "\"config2\": {\"images\": %lld, \"images_per_gpu\": %lld, \"ms_per_step\": %.4f, "
        "\"images_per_s\": %.1f, \"routed_at_0.5\": %lld}, "
        "\"config5\": {\"queries\": %lld, \"ms\": %.3f, \"images_per_s\": %.1f, "
        "\"routed_at_0.5\": %lld}, "
        "\"check\": %s}\n",
        G, static_cast<long long>(N), static_cast<long long>(per_gpu), ms, N / (ms / 1e3),
        r0.routed50, static_cast<long long>(queries), ms5, queries / (ms5 / 1e3), r0.scale_routed,
        check ? (std::string("{\"global_queues_equal_1gpu\": ") +
                 (r0.queues_equal ? "true" : "false") + ", \"global_counts_equal_1gpu\": " +
                 (r0.counts_equal ? "true" : "false") + ", \"global_curve_bits_equal_1gpu\": " +
                 (r0.curve_equal ? "true" : "false") + ", \"config5_queue_equal_1gpu\": " +
                 (r0.scale_equal ? "true" : "false") + "}")
                    .c_str()
              : "null");
    for (int g = 0; g < G; ++g) {
        CK(ds_comm_destroy(comms[g]));
        CK(ds_ctx_destroy(ctxs[g]));
    }
    const bool ok = !check || (r0.queues_equal && r0.counts_equal && r0.curve_equal &&
                               r0.scale_equal);
    return ok ? 0 : 1;
}
