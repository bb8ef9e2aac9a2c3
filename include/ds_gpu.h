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
    DS_ERR_CAPACITY = 7          /* input exceeds a compiled-in ABI limit  */
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
/* Scratch bytes ds_route_device needs for n queries and nt thresholds. */
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
 * ds_disc_score_device + ds_curve_observe_device + ds_route_device; batches of
 * <= 2048 images run as the discriminator plus one fused tail launch. */
ds_status ds_disc_batch_complete_device(ds_disc* disc, const uint8_t* nhwc, int64_t n,
                                        int32_t h, int32_t w, float* conf, ds_curve* curve,
                                        double decay, const double* thresholds,
                                        int32_t n_thresholds, int64_t index_base,
                                        int64_t* heavy_idx, int64_t* counts, void* stream);

/* Synthetic image pool: pixel bytes are a pure
 * function of (seed, image id, pixel index); generated on the device. */
ds_status ds_synth_images_device(ds_ctx* ctx, uint64_t seed, uint64_t id0, int64_t n,
                                 int32_t h, int32_t w, uint8_t* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DS_GPU_H */
