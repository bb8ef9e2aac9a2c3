/*
 * ds_gpu.h -- C ABI of the B200-native DiffServe hot path.
 *
 * Plain C: POD structs, pointers and sizes, integer status codes. No CUDA,
 * torch or C++ types appear in any signature, so the reference's C++ host
 * (or a ctypes / cgo / JNI stub) can bind it directly.
 *
 * Two halves, mirroring the reference hot path:
 *   planner  : ds_plan_batch*        replaces diffserve::solve and variants
 *                                    (reference proj/src/allocator.cpp:153-313)
 *   score    : ds_score_latent*      replaces diffserve::sample_query
 *                                    (reference proj/src/workload.cpp:108-129)
 *              ds_disc_score*        discriminator network (no reference;
 *                                    SURVEY 8a row S9)
 *   route    : ds_route*             replaces the Policy::defers loop
 *                                    (reference proj/src/cluster.cpp:290-306,
 *                                     proj/src/policies.cpp:37-39)
 *   curve    : ds_curve_observe*     replaces diffserve::observe_confidence
 *                                    (reference proj/src/profiles.cpp:108-120)
 *   workload : ds_generate_arrivals* replaces diffserve::generate_arrivals
 *                                    (reference proj/src/workload.cpp:82-106)
 *              ds_sample_queries*    replaces the sample_query loop of
 *                                    run_experiment (experiment.cpp:76-79)
 *   output   : ds_format_*_csv*      replaces diffserve::write_csv's row
 *                                    formatting (metrics.cpp:67-127)
 *
 * Functions without the _device suffix take HOST buffers and copy in/out
 * inside the call (the reference-facing drop-in). The _device variants take
 * device pointers and a cudaStream_t passed as void*; they are stream-ordered
 * and do not synchronize.
 *
 * Errors: the reference throws C++ exceptions (allocator.cpp:12-36,
 * profiles.cpp:20-26,98-100,108-112). Across this ABI each exception type maps
 * to one status code; ds_last_error() returns the reference's message text
 * for the calling thread. Infeasibility is NOT an error (plan.feasible = 0).
 */
#ifndef DS_GPU_H
#define DS_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DS_ABI_VERSION 1
#define DS_MAX_BATCHES 64   /* profiled batch sizes per model               */
#define DS_CURVE_BINS 101   /* DeferralCurve::kBins, profiles.hpp:50         */

typedef enum {
    DS_OK = 0,
    DS_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument                  */
    DS_ERR_DOMAIN = 2,           /* std::domain_error                      */
    DS_ERR_INVARIANT = 3,        /* diffserve::InvariantError              */
    DS_ERR_OUT_OF_RANGE = 4,     /* std::out_of_range (unprofiled batch)   */
    DS_ERR_CUDA = 5,             /* CUDA runtime / launch failure          */
    DS_ERR_NO_DEVICE = 6,        /* no sm_100 device visible               */
    DS_ERR_CAPACITY = 7,         /* input exceeds a compiled-in ABI limit  */
    DS_ERR_COMM = 8              /* collective transport (NCCL / host ops) */
} ds_status;

typedef enum {
    DS_QUEUING_LITTLES_LAW = 0, /* QueuingModel::littles_law, allocator.hpp:23 */
    DS_QUEUING_TWICE_EXEC = 1   /* QueuingModel::twice_exec,  allocator.hpp:24 */
} ds_queuing;

/* Which reference entry point a planner problem runs (allocator.hpp:64-91). */
typedef enum {
    DS_SOLVE = 0,               /* solve()                  allocator.cpp:153 */
    DS_SOLVE_PINNED = 1,        /* solve_pinned_threshold() allocator.cpp:176 */
    DS_SOLVE_FIXED_BATCHES = 2, /* solve_fixed_batches()    allocator.cpp:213 */
    DS_SOLVE_EVEN_SPLIT = 3,    /* solve_even_split()       allocator.cpp:270 */
    DS_SOLVE_SINGLE_LIGHT = 4,  /* solve_single_model(light) allocator.cpp:232 */
    DS_SOLVE_SINGLE_HEAVY = 5   /* solve_single_model(heavy) allocator.cpp:232 */
} ds_solve_mode;
/* solve_static_peak (allocator.cpp:171) is DS_SOLVE with demand := peak. */

/* ModelProfile (profiles.hpp:11-19): batch sizes strictly ascending. */
typedef struct {
    int32_t n;
    int32_t _pad;
    int32_t batch[DS_MAX_BATCHES];
    double latency[DS_MAX_BATCHES];
} ds_model_profile;

/* DeferralCurve (profiles.hpp:35-48); bin lower edges are implicitly k/100. */
typedef struct {
    double bin_mass[DS_CURVE_BINS];
    double total_mass;
} ds_curve;

/* CascadeProfile (profiles.hpp:62-68). */
typedef struct {
    ds_model_profile light;
    ds_model_profile heavy;
    ds_curve deferral;
    double slo_seconds;
} ds_cascade;

/* AllocationProblem (allocator.hpp:27-37) plus the variant selector. */
typedef struct {
    double demand_qps;
    double overprovision_lambda;
    double queue_sentinel_seconds;
    double light_rate;        /* light_queue.arrival_rate */
    double heavy_rate;        /* heavy_queue.arrival_rate */
    int64_t light_len;        /* light_queue.queue_length */
    int64_t heavy_len;        /* heavy_queue.queue_length */
    double fixed_threshold;   /* DS_SOLVE_PINNED                    */
    int32_t fixed_b1;         /* DS_SOLVE_FIXED_BATCHES             */
    int32_t fixed_b2;
    int32_t total_servers;
    int32_t queuing;          /* ds_queuing                         */
    int32_t cascade;          /* index into the cascades array      */
    int32_t grid;             /* index into the grid table          */
    int32_t mode;             /* ds_solve_mode                      */
    int32_t _pad;
} ds_problem;

/* AllocationPlan (allocator.hpp:39-46). */
typedef struct {
    int32_t x1, x2, b1, b2;
    double threshold;
    int32_t feasible;
    int32_t _pad;
} ds_plan;

/* QueryOutcomeModel (workload.hpp:52-58). */
typedef struct {
    double easy_fraction;
    double quality_gap_scale;
    double confidence_fidelity;
    double noise_sigma;
    uint64_t seed;
} ds_query_model;

typedef struct ds_ctx ds_ctx;

/* ---- context -------------------------------------------------------- */
const char* ds_version(void);
const char* ds_last_error(void);
ds_status ds_ctx_create(int device, ds_ctx** out);
ds_status ds_ctx_destroy(ds_ctx* ctx);
ds_status ds_ctx_synchronize(ds_ctx* ctx);
/* Number of device kernels this context launched so far (for bench audits). */
int64_t ds_ctx_launch_count(const ds_ctx* ctx);
void* ds_ctx_stream(ds_ctx* ctx); /* the context's cudaStream_t */
/* The _device variants do not synchronize, so they cannot return the
 * reference's std::domain_error for a confidence outside [0, 1]
 * (profiles.cpp:108-112) at launch time. They stop the curve replay at the
 * first invalid observation, as the reference's throw does (a light batch of
 * <= 2048 images in ds_disc_batch_complete_device also routes only the
 * queries before it, as the throw out of handle_batch_complete would), and
 * record its index in the context. ds_ctx_take_error synchronizes `stream`
 * (NULL: the context's stream), returns DS_ERR_DOMAIN with *first_bad = that
 * index if any device call recorded one since the last call (and clears it),
 * else DS_OK with *first_bad = -1. */
ds_status ds_ctx_take_error(ds_ctx* ctx, void* stream, int64_t* first_bad);

/* ---- planner (K1 plan_sweep) ---------------------------------------- */
/* Validates every problem with the reference's checks (allocator.cpp:22-36,
 * profiles.cpp:20-26), then solves all n problems in one launch.
 * grid_offsets has n_grids+1 entries; grid g is
 * grid_values[grid_offsets[g] .. grid_offsets[g+1]). */
ds_status ds_plan_batch(ds_ctx* ctx, const ds_problem* problems, int32_t n,
                        const ds_cascade* cascades, int32_t n_cascades,
                        const double* grid_values, const int32_t* grid_offsets,
                        int32_t n_grids, ds_plan* out);
/* Same, all pointers on the device, no validation, no sync. */
ds_status ds_plan_batch_device(ds_ctx* ctx, const ds_problem* problems, int32_t n,
                               const ds_cascade* cascades, int32_t n_cascades,
                               const double* grid_values, const int32_t* grid_offsets,
                               int32_t n_grids, ds_plan* out, void* stream);
/* Threshold-range sharding of the planner ("shard t-ranges
 * ... ncclAllReduce(uint64 key, ncclMin) per problem"). ds_plan_keys searches
 * only grid indices [t_lo, t_hi) of each grid-mode problem (DS_SOLVE,
 * DS_SOLVE_FIXED_BATCHES) and returns its packed selection key
 *   (G-1-t_idx)<<40 | (x1+x2)<<28 | (255-b1_idx)<<20 | (255-b2_idx)<<12 | x1
 * (UINT64_MAX: no valid candidate in the range; always for the other modes),
 * whose unsigned order is the reference's choice order (allocator.cpp:57-67,
 * 91-121), so the minimum over disjoint ranges -- one per GPU -- equals the
 * full search's key. ds_plan_from_keys turns the reduced keys into the plans
 * ds_plan_batch returns (decode, or the reference's fallbacks; non-grid modes
 * are solved whole). Same validation and errors as ds_plan_batch. */
ds_status ds_plan_keys(ds_ctx* ctx, const ds_problem* problems, int32_t n,
                       const ds_cascade* cascades, int32_t n_cascades, const double* grid_values,
                       const int32_t* grid_offsets, int32_t n_grids, int32_t t_lo, int32_t t_hi,
                       uint64_t* keys);
ds_status ds_plan_keys_device(ds_ctx* ctx, const ds_problem* problems, int32_t n,
                              const ds_cascade* cascades, int32_t n_cascades,
                              const double* grid_values, const int32_t* grid_offsets,
                              int32_t n_grids, int32_t t_lo, int32_t t_hi, uint64_t* keys,
                              void* stream);
ds_status ds_plan_from_keys(ds_ctx* ctx, const ds_problem* problems, int32_t n,
                            const ds_cascade* cascades, int32_t n_cascades,
                            const double* grid_values, const int32_t* grid_offsets,
                            int32_t n_grids, const uint64_t* keys, ds_plan* out);
ds_status ds_plan_from_keys_device(ds_ctx* ctx, const ds_problem* problems, int32_t n,
                                   const ds_cascade* cascades, int32_t n_cascades,
                                   const double* grid_values, const int32_t* grid_offsets,
                                   int32_t n_grids, const uint64_t* keys, ds_plan* out,
                                   void* stream);
/* Host-side validation only (the checks ds_plan_batch runs before launch). */
ds_status ds_plan_validate(const ds_problem* problems, int32_t n, const ds_cascade* cascades,
                           int32_t n_cascades, const double* grid_values,
                           const int32_t* grid_offsets, int32_t n_grids);

/* ---- latent scorer (K4 latent_score) ---------------------------------- */
/* conf[i] / quality_light[i] of query id0+i, bit-identical streams to
 * sample_query (workload.cpp:108-129). quality_light may be NULL. */
ds_status ds_score_latent(ds_ctx* ctx, const ds_query_model* model, uint64_t id0, int64_t n,
                          double* conf, double* quality_light);
ds_status ds_score_latent_device(ds_ctx* ctx, const ds_query_model* model, uint64_t id0,
                                 int64_t n, double* conf, double* quality_light, void* stream);

/* ---- router (K2 route_compact) ---------------------------------------- */
/* For every threshold t_k: heavy list k = ascending indices i with
 * conf[i] < t_k (strict, policies.cpp:37-39), written to
 * heavy_idx[k*n .. k*n + counts[k]). conf is f64 (dtype 0) or f32 (dtype 1).
 * index_base is added to every written index (global ids of a shard). */
#define DS_CONF_F64 0
#define DS_CONF_F32 1
ds_status ds_route(ds_ctx* ctx, const void* conf, int32_t dtype, int64_t n,
                   const double* thresholds, int32_t n_thresholds, int64_t index_base,
                   int64_t* heavy_idx, int64_t* counts);
ds_status ds_route_device(ds_ctx* ctx, const void* conf, int32_t dtype, int64_t n,
                          const double* thresholds, int32_t n_thresholds, int64_t index_base,
                          int64_t* heavy_idx, int64_t* counts, void* stream);
/* Caller scratch ds_route_device needs for n queries and nt thresholds: 0
 * (kept for ABI stability; K2 is one pass and keeps its look-back flags in
 * the context). */
size_t ds_route_scratch_bytes(int64_t n, int32_t n_thresholds);

/* ---- deferral curve (K3 curve_observe) -------------------------------- */
/* Applies observe_confidence(curve, conf[i], decay) for i = 0..n-1 in order;
 * bit-identical to the reference's sequential loop. */
ds_status ds_curve_observe(ds_ctx* ctx, ds_curve* curve, const void* conf, int32_t dtype,
                           int64_t n, double decay);
ds_status ds_curve_observe_device(ds_ctx* ctx, ds_curve* curve, const void* conf,
                                  int32_t dtype, int64_t n, double decay, void* stream);

/* ---- workload synthesis (K8 arrivals, K4 query records) --------------- */
/* ArrivalMode (workload.hpp:26). */
typedef enum {
    DS_ARRIVALS_POISSON = 0,
    DS_ARRIVALS_UNIFORM = 1
} ds_arrival_mode;

/* Query (workload.hpp:39-46), 48 bytes. */
typedef struct {
    uint64_t id;
    double arrival;
    double deadline;
    double quality_light;
    double quality_heavy;
    double confidence;
} ds_query;

/* generate_arrivals(Trace{interval_seconds, rates[0..n_rates)}, seed, mode)
 * (workload.cpp:82-106): bit-identical timestamps. *count receives the number
 * of arrivals. arrivals may be NULL (count only); otherwise it must hold
 * *count entries, else DS_ERR_CAPACITY (with *count set). Rates must be
 * finite and >= 0 and interval_seconds > 0 (what load_trace admits,
 * workload.cpp:21-22,44-45), else DS_ERR_DOMAIN. */
ds_status ds_generate_arrivals(ds_ctx* ctx, const double* rates, int32_t n_rates,
                               double interval_seconds, uint64_t seed, int32_t mode,
                               double* arrivals, int64_t capacity, int64_t* count);
/* Same with arrivals on the device (rates and count stay host memory). The
 * output length is data-dependent, so this call synchronizes its stream once
 * to read the count; the copy into arrivals is stream-ordered after it. */
ds_status ds_generate_arrivals_device(ds_ctx* ctx, const double* rates, int32_t n_rates,
                                      double interval_seconds, uint64_t seed, int32_t mode,
                                      double* arrivals, int64_t capacity, int64_t* count,
                                      void* stream);
/* out[i] = sample_query(model, id0 + i, arrivals[i], slo_seconds)
 * (workload.cpp:108-129): the Query records run_experiment builds
 * (experiment.cpp:76-79) with ids id0.. in arrival order. */
ds_status ds_sample_queries(ds_ctx* ctx, const ds_query_model* model, uint64_t id0,
                            const double* arrivals, int64_t n, double slo_seconds,
                            ds_query* out);
ds_status ds_sample_queries_device(ds_ctx* ctx, const ds_query_model* model, uint64_t id0,
                                   const double* arrivals, int64_t n, double slo_seconds,
                                   ds_query* out, void* stream);

/* ---- CSV output (K9 csv_format) ---------------------------------------- */
/* Outcome (metrics.hpp:12-17). */
typedef enum {
    DS_OUTCOME_SERVED_LIGHT = 0,
    DS_OUTCOME_SERVED_HEAVY = 1,
    DS_OUTCOME_DROPPED = 2,
    DS_OUTCOME_LATE = 3
} ds_outcome;

/* QueryRecord (metrics.hpp:22-36); std::optional fields are engaged when the
 * matching DS_REC_* bit of `present` is set. */
#define DS_REC_LIGHT_START 0x01u
#define DS_REC_LIGHT_END 0x02u
#define DS_REC_HEAVY_START 0x04u
#define DS_REC_HEAVY_END 0x08u
#define DS_REC_COMPLETION 0x10u
#define DS_REC_OUTCOME 0x20u
#define DS_REC_DELIVERED_QUALITY 0x40u
typedef struct {
    uint64_t id;
    double arrival;
    double deadline;
    double confidence;
    double quality_light;
    double quality_heavy;
    double light_start;
    double light_end;
    double heavy_start;
    double heavy_end;
    double completion;
    double delivered_quality;
    uint32_t present;
    int32_t outcome; /* ds_outcome */
} ds_query_record;

/* IntervalSnapshot (metrics.hpp:42-54). */
typedef struct {
    double interval_start;
    double demand_observed;
    double demand_estimated;
    ds_plan plan;
    uint64_t arrived;
    uint64_t served_light;
    uint64_t served_heavy;
    uint64_t dropped;
    uint64_t late;
    double threshold;
    double mean_delivered_quality;
    int32_t has_mean_delivered_quality;
    int32_t _pad;
} ds_interval_snapshot;

/* PlanLogEntry (metrics.hpp:57-62). */
typedef struct {
    int32_t tick;
    int32_t _pad;
    double time;
    double demand_estimated;
    ds_plan plan;
} ds_plan_log_entry;

/* The bytes write_csv puts in queries.csv / intervals.csv / plans.csv
 * (metrics.cpp:91-127, header line included), byte-identical: every real goes
 * through an exact "%.6g" (fmt6, metrics.cpp:67-71). *bytes receives the file
 * size; out may be NULL (size only), else it must hold *bytes bytes, else
 * DS_ERR_CAPACITY. Host buffers in and out. */
ds_status ds_format_queries_csv(ds_ctx* ctx, const ds_query_record* records, int64_t n,
                                char* out, int64_t capacity, int64_t* bytes);
ds_status ds_format_intervals_csv(ds_ctx* ctx, const ds_interval_snapshot* rows, int64_t n,
                                  char* out, int64_t capacity, int64_t* bytes);
ds_status ds_format_plans_csv(ds_ctx* ctx, const ds_plan_log_entry* rows, int64_t n, char* out,
                              int64_t capacity, int64_t* bytes);
/* Same for queries.csv with device records and a device output buffer; reads
 * the size back once (one stream synchronization). */
ds_status ds_format_queries_csv_device(ds_ctx* ctx, const ds_query_record* records, int64_t n,
                                       char* out, int64_t capacity, int64_t* bytes,
                                       void* stream);
/* fmt6 of n doubles into 16-byte slots (NUL-padded), for tests and callers
 * that assemble their own rows. */
ds_status ds_format_g6(ds_ctx* ctx, const double* values, int64_t n, char* out16);

/* ---- discriminator (K5-K7: ingest + fused tcgen05 MLP + head) --------- */
/* PatchDisc: u8 NHWC image -> 16x16 patches -> 768->256 GELU -> 256->1024
 * ReLU -> 1024->256 ReLU -> mean over patches -> dot(256)+b -> sigmoid.
 * Layer 1 is u8 pixels x int8 weights with an exact s32 accumulator
 * (h1_pre = s1 * acc + b1); layers 2-3 are bf16 x bf16 -> f32. Weights are
 * generated deterministically from weight_seed. */
#define DS_DISC_PATCH 16
#define DS_DISC_D0 768
#define DS_DISC_D1 256
#define DS_DISC_D2 1024
#define DS_DISC_D3 256
typedef struct ds_disc ds_disc;
ds_status ds_disc_create(ds_ctx* ctx, uint64_t weight_seed, ds_disc** out);
ds_status ds_disc_destroy(ds_disc* disc);
/* Host copies of the weights in the kernel's logical layout (row = input
 * feature): q1 [768][256] int8 with its scale s1 (one f32), w2 [256][1024]
 * and w3 [1024][256] as raw bf16 bit patterns; b1/b2/b3 f32; head w
 * f32[256]; head bias f32. Any pointer may be NULL. */
ds_status ds_disc_export(const ds_disc* disc, int8_t* q1, float* s1, uint16_t* w2, uint16_t* w3,
                         float* b1, float* b2, float* b3, float* head_w, float* head_b);
/* Scores n images (host buffer, n*h*w*3 bytes; h, w multiples of 128). */
ds_status ds_disc_score(ds_disc* disc, const uint8_t* nhwc, int64_t n, int32_t h, int32_t w,
                        float* conf);
ds_status ds_disc_score_device(ds_disc* disc, const uint8_t* nhwc, int64_t n, int32_t h,
                               int32_t w, float* conf, void* stream);

/* One light batch as Simulation::handle_batch_complete (cluster.cpp:288-307)
 * handles it: score the n images into conf, apply observe_confidence(curve,
 * conf[i], decay) in batch order (profiles.cpp:108-120), then route every
 * image at each threshold with Policy::defers (policies.cpp:37-39, strict <)
 * into ordered heavy lists (row k of heavy_idx holds counts[k] ids, stride n).
 * All pointers are device memory, stream-ordered. Bit-identical to
 * ds_disc_score_device + ds_curve_observe_device + ds_route_device. Batches of
 * <= 2048 images are ONE launch whose last CTA runs the tail, and consecutive
 * calls on a stream overlap (programmatic dependent launch): the next call's
 * pair tiles start on the SMs this batch's last round leaves idle, reading
 * only its images before it waits for this call to complete. The images of a
 * call must therefore be written by stream work that completes before the
 * call (copies, ordinary kernels) -- not by a kernel that itself lets its
 * dependents start early. Calls on one stream complete in order; the tail's
 * state lives per (disc, stream). DS_DISC_NO_CHAIN=1 at the first call of a
 * disc selects two plain launches per batch. */
ds_status ds_disc_batch_complete_device(ds_disc* disc, const uint8_t* nhwc, int64_t n,
                                        int32_t h, int32_t w, float* conf, ds_curve* curve,
                                        double decay, const double* thresholds,
                                        int32_t n_thresholds, int64_t index_base,
                                        int64_t* heavy_idx, int64_t* counts, void* stream);

/* A backlog of light batches in one call: batch b is images
 * [batch_offsets[b], batch_offsets[b+1]) (device array of n_batches + 1
 * nondecreasing offsets, 0 .. n_images), completed in order as
 * handle_batch_complete (cluster.cpp:288-307) completes them one by one:
 * every confidence observed into the curve in order, batch b routed at ITS
 * threshold thresholds[b] (device, one per batch: the plan in force when it
 * completes) into heavy_idx[batch_offsets[b] .. + counts[b]) (global ids
 * index_base + image index). Bit-identical to n_batches calls of
 * ds_disc_batch_complete_device (the discriminator's confidences do not
 * depend on the batch split), but one discriminator launch streams all the
 * batches' tiles, so small batches keep every SM busy (config 1: batches of
 * 32). A confidence outside [0, 1] stops the curve and the routing at that
 * query (later batches: counts 0) and is recorded as in ds_ctx_take_error. */
ds_status ds_disc_batches_complete_device(ds_disc* disc, const uint8_t* nhwc, int64_t n_images,
                                          const int64_t* batch_offsets, int32_t n_batches,
                                          int32_t h, int32_t w, float* conf, ds_curve* curve,
                                          double decay, const double* thresholds,
                                          int64_t index_base, int64_t* heavy_idx,
                                          int64_t* counts, void* stream);

/* Synthetic image pool: pixel bytes are a pure
 * function of (seed, image id, pixel index); generated on the device. */
ds_status ds_synth_images_device(ds_ctx* ctx, uint64_t seed, uint64_t id0, int64_t n,
                                 int32_t h, int32_t w, uint8_t* out, void* stream);

/* ---- multi-GPU: the sharded hot path (SURVEY.md 8(b) "NCCL-aware
 * multi-GPU variant", 8(e)) ---------------------------------------------- */
/* One rank per GPU. Queries shard by contiguous id range, planner problems by
 * index or one batch by threshold range. The reference is single-process
 * (SPEC.md:330); these entry points make an N-GPU run return exactly what one
 * GPU -- and therefore the reference -- returns:
 *   heavy queues : routed-count all-gather + exclusive scan (each rank's
 *                  offset in every global queue), then the ordered ids of all
 *                  ranks gathered into the global queues at a root rank
 *                  (cluster.cpp:290-306 id order);
 *   curve        : the ordered confidences all-gathered, every rank replays
 *                  the whole sequence (observe_confidence is order-dependent
 *                  through the decay, profiles.cpp:108-120);
 *   planner      : packed selection keys MIN-all-reduced over threshold
 *                  ranges (allocator.cpp:57-67,91-121).
 * All calls below are COLLECTIVE: every rank of the communicator makes the
 * same call with matching scalar arguments, in the same order. Device
 * pointers, stream-ordered on `stream` (NULL: the context's stream); calls
 * that must size a transfer from device counts synchronize `stream` once. */
typedef struct ds_comm ds_comm;
#define DS_NCCL_UNIQUE_ID_BYTES 128

/* Host transport for callers without NCCL (and for tests that run several
 * ranks on one GPU, which NCCL refuses): the library copies to host, calls
 * these, copies back. Each returns 0 on success. */
typedef struct {
    /* recv gets nranks*bytes bytes: rank r's `bytes` bytes at offset r*bytes */
    int (*allgather)(const void* send, void* recv, size_t bytes, void* user);
    /* element-wise unsigned minimum over ranks, in place */
    int (*allreduce_min_u64)(uint64_t* buf, size_t count, void* user);
    /* rank r contributes bytes[r] bytes; root receives them back to back in
     * rank order (recv is NULL on the other ranks) */
    int (*gatherv)(const void* send, void* recv, const size_t* bytes, int32_t root, void* user);
} ds_comm_ops;

/* NCCL (loaded at run time: libnccl.so.2, the process's own if one is
 * already loaded -- a host that links its own NCCL, e.g. torch, must load it
 * before the first ds_comm call, or the system copy takes the soname). Rank 0 makes the id and distributes it out of band (MPI,
 * torch.distributed, a file), then every rank calls ds_comm_init_nccl with
 * its context -- ncclCommInitRank on the context's device. */
ds_status ds_comm_nccl_unique_id(uint8_t id[DS_NCCL_UNIQUE_ID_BYTES]);
ds_status ds_comm_init_nccl(ds_ctx* ctx, int32_t nranks, int32_t rank,
                            const uint8_t id[DS_NCCL_UNIQUE_ID_BYTES], ds_comm** out);
/* Wraps a caller's ncclComm_t (not owned; its device must be ctx's). */
ds_status ds_comm_wrap_nccl(ds_ctx* ctx, void* nccl_comm, ds_comm** out);
/* One process driving n GPUs (ncclCommInitAll over ctxs[i]'s devices): drive
 * each comms[i] from its own host thread (the calls are collective and some
 * synchronize, so one thread issuing all ranks' calls would deadlock). */
ds_status ds_comm_init_all(ds_ctx* const* ctxs, int32_t n, ds_comm** comms);
ds_status ds_comm_create_host(ds_ctx* ctx, int32_t nranks, int32_t rank, const ds_comm_ops* ops,
                              void* user, ds_comm** out);
ds_status ds_comm_destroy(ds_comm* comm);
int32_t ds_comm_rank(const ds_comm* comm);
int32_t ds_comm_size(const ds_comm* comm);
/* [lo, hi) of a contiguous balanced split of n items: lo = n*rank/nranks. */
void ds_shard_range(int64_t n, int32_t nranks, int32_t rank, int64_t* lo, int64_t* hi);

/* Route this rank's shard (ds_route_device with index_base = its first global
 * id), then all-gather the routed counts: rank_offsets[k] = this rank's start
 * inside global heavy queue k (sum of lower ranks' counts), global_counts[k] =
 * the global queue's length. Either output may be NULL. */
ds_status ds_route_sharded_device(ds_ctx* ctx, ds_comm* comm, const void* conf, int32_t dtype,
                                  int64_t n_local, const double* thresholds, int32_t n_thresholds,
                                  int64_t index_base, int64_t* heavy_local, int64_t* counts_local,
                                  int64_t* rank_offsets, int64_t* global_counts, void* stream);
/* Assemble the global heavy queues at `root`: row k of global_heavy (stride
 * global_stride >= the global count) receives every rank's counts_local[k]
 * ids from heavy_local row k (stride n_local) at that rank's offset, i.e.
 * rank order = global id order. global_heavy / global_counts are written on
 * root only (may be NULL elsewhere). Synchronizes `stream` once (the
 * transfer sizes come from the counts). */
ds_status ds_queue_gather_device(ds_ctx* ctx, ds_comm* comm, int32_t root,
                                 const int64_t* heavy_local, int64_t n_local,
                                 const int64_t* counts_local, int32_t n_thresholds,
                                 int64_t* global_heavy, int64_t global_stride,
                                 int64_t* global_counts, void* stream);
/* observe_confidence over the GLOBAL sequence: the ranks' shards (sizes
 * shard_sizes[0..nranks), host memory, rank order = id order) are
 * all-gathered and every rank replays all of them into its `curve`, so every
 * rank ends with the curve one GPU (and the reference) computes. An invalid
 * confidence is recorded as in ds_curve_observe_device (global index). */
ds_status ds_curve_observe_sharded_device(ds_ctx* ctx, ds_comm* comm, ds_curve* curve,
                                          const void* conf_local, int32_t dtype,
                                          const int64_t* shard_sizes, double decay,
                                          void* stream);
/* Threshold-range sharded planning of ONE problem batch (every rank passes the
 * same problems): this rank searches grid indices [t_lo, t_hi) (ds_plan_keys),
 * the keys are MIN-all-reduced (uint64; "none" is UINT64_MAX), and every rank
 * decodes the plans ds_plan_batch would return (ds_plan_from_keys). */
ds_status ds_plan_sharded_device(ds_ctx* ctx, ds_comm* comm, const ds_problem* problems, int32_t n,
                                 const ds_cascade* cascades, int32_t n_cascades,
                                 const double* grid_values, const int32_t* grid_offsets,
                                 int32_t n_grids, int32_t t_lo, int32_t t_hi, ds_plan* out,
                                 void* stream);
/* Generic ordered gather (problem-sharded plans, per-rank results): rank r
 * contributes `bytes` bytes (may differ per rank); root receives all of them
 * back to back in rank order and *total_bytes their sum (root only). recv
 * needs room for the sum. Synchronizes `stream` once. */
ds_status ds_comm_gather_device(ds_ctx* ctx, ds_comm* comm, int32_t root, const void* send,
                                size_t bytes, void* recv, size_t recv_capacity,
                                size_t* total_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DS_GPU_H */
