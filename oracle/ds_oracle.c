/*
 * TEST INFRASTRUCTURE ONLY -- the CPU oracle (checker), never the product.
 *
 * Plain-C restatement of the reference hot path, function by function, on the
 * POD types of include/ds_gpu.h. Parity of this restatement is PINNED against
 * the reference itself: tests/test_oracle.py checks it against the golden
 * vectors in tests/golden/ (generated from the reference's own generators and
 * solver by oracle/make_golden.py) and, where oracle/_ref/libdsref.so exists,
 * directly against the reference library on fresh random inputs.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
 * --impl reference) may load this library.
 *
 * Build: gcc -std=c11 -O2 at the default -march (no FMA contraction), see
 * oracle/Makefile.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "ds_gpu.h"

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

/* ---------------------------------------------------------------------- */
/* RNG primitives: rng.cpp:8-36, rng.hpp:17-40                             */

uint64_t dso_splitmix64(uint64_t x) { /* rng.cpp:8-13 */
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

uint64_t dso_hash_name(const char* s) { /* rng.cpp:15-22, FNV-1a */
    uint64_t h = 0xcbf29ce484222325ULL;
    for (; *s; ++s) {
        h ^= (unsigned char)*s;
        h *= 0x100000001b3ULL;
    }
    return h;
}

/* std::mt19937_64 (ISO C++ [rand.predef]); full-state textbook version. */
typedef struct {
    uint64_t mt[312];
    int idx;
} dso_mt64;

static void mt64_seed(dso_mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
}

static uint64_t mt64_next(dso_mt64* g) {
    if (g->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            uint64_t y = (g->mt[i] & 0xFFFFFFFF80000000ULL) | (g->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t v = g->mt[(i + 156) % 312] ^ (y >> 1);
            if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
            g->mt[i] = v;
        }
        g->idx = 0;
    }
    uint64_t z = g->mt[g->idx++];
    z ^= (z >> 29) & 0x5555555555555555ULL;
    z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
    z ^= (z << 37) & 0xFFF7EEE000000000ULL;
    z ^= z >> 43;
    return z;
}

/* RandomStream(seed, name): eng_(splitmix64(seed ^ splitmix64(hash_name(name)))) */
static void stream_init(dso_mt64* g, uint64_t seed, const char* name) {
    mt64_seed(g, dso_splitmix64(seed ^ dso_splitmix64(dso_hash_name(name))));
}
static double stream_uniform(dso_mt64* g) { /* rng.hpp:26 */
    return (double)(mt64_next(g) >> 11) * 0x1.0p-53;
}
static double stream_normal(dso_mt64* g) { /* rng.cpp:30-36 */
    double u1 = stream_uniform(g);
    double u2 = stream_uniform(g);
    if (u1 <= 0.0) u1 = 0x1.0p-53;
    return sqrt(-2.0 * log(u1)) * cos(2.0 * M_PI * u2);
}

/* First k raw outputs of the mt19937_64 engine a RandomStream(seed, name)
 * would produce (used to pin the GPU's streamed-state shortcut). */
void dso_stream_raw(uint64_t seed, const char* name, int k, uint64_t* out) {
    dso_mt64 g;
    stream_init(&g, seed, name);
    for (int i = 0; i < k; ++i) out[i] = mt64_next(&g);
}

/* sample_query (workload.cpp:108-129): confidence and quality_light of id. */
int dso_sample_query(const ds_query_model* m, uint64_t id, double* conf, double* quality_light) {
    if (!(m->easy_fraction >= 0.0) || !(m->easy_fraction <= 1.0)) return DS_ERR_DOMAIN;
    dso_mt64 g;
    stream_init(&g, dso_splitmix64(m->seed) ^ dso_splitmix64(id), "query");
    int easy = stream_uniform(&g) < m->easy_fraction;
    double gap = m->quality_gap_scale * fabs(stream_normal(&g));
    double dq = easy ? gap : -gap;
    double noise = 0.0 + m->noise_sigma * stream_normal(&g);
    double c = 0.5 + m->confidence_fidelity * dq + noise;
    if (c < 0.0) c = 0.0;
    if (c > 1.0) c = 1.0;
    *conf = c;
    if (quality_light) *quality_light = 1.0 + dq;
    return DS_OK;
}

typedef struct {
    const ds_query_model* m;
    uint64_t id0;
    int64_t lo, hi;
    double *conf, *ql;
} sq_job;

static void* sq_worker(void* arg) {
    sq_job* j = (sq_job*)arg;
    for (int64_t i = j->lo; i < j->hi; ++i)
        dso_sample_query(j->m, j->id0 + (uint64_t)i, &j->conf[i], j->ql ? &j->ql[i] : NULL);
    return NULL;
}

int dso_sample_queries(const ds_query_model* m, uint64_t id0, int64_t n, double* conf,
                       double* quality_light, int threads) {
    if (!(m->easy_fraction >= 0.0) || !(m->easy_fraction <= 1.0)) return DS_ERR_DOMAIN;
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pthread_t tid[256];
    sq_job jobs[256];
    for (int k = 0; k < threads; ++k) {
        jobs[k] = (sq_job){m, id0, n * k / threads, n * (k + 1) / threads, conf, quality_light};
        if (threads == 1) sq_worker(&jobs[0]);
        else pthread_create(&tid[k], NULL, sq_worker, &jobs[k]);
    }
    if (threads > 1)
        for (int k = 0; k < threads; ++k) pthread_join(tid[k], NULL);
    return DS_OK;
}

/* ---------------------------------------------------------------------- */
/* Workload synthesis: workload.cpp:82-106                                 */

/* generate_arrivals on Trace{dt, rates[0..n)}: returns the count and writes
 * min(count, cap) timestamps. mode 0 = poisson, 1 = uniform. The Exp(1)
 * draws are RandomStream::exponential(1.0) = -log1p(-U) / 1.0 through the
 * host libm, as in the reference (rng.cpp:24-28). */
int64_t dso_generate_arrivals(const double* rates, int32_t n, double dt, uint64_t seed,
                              int32_t mode, double* out, int64_t cap) {
    dso_mt64 g;
    stream_init(&g, seed, "arrivals");
    const double duration = dt * (double)n;
    double target = mode == 1 ? 0.0 : -log1p(-stream_uniform(&g)) / 1.0;
    double cum = 0.0, last = 0.0;
    int64_t c = 0;
    for (int32_t k = 0; k < n; ++k) {
        double rate = rates[k];
        double start = dt * (double)k;
        double cum_end = cum + rate * dt;
        while (rate > 0.0 && target < cum_end - 1e-12) {
            double t = start + (target - cum) / rate;
            if (c > 0 && t <= last) t = nextafter(last, INFINITY);
            if (t >= duration) break;
            if (c < cap) out[c] = t;
            last = t;
            ++c;
            target += mode == 1 ? 1.0 : -log1p(-stream_uniform(&g)) / 1.0;
        }
        cum = cum_end;
    }
    return c;
}

/* ---------------------------------------------------------------------- */
/* CSV rows: metrics.cpp:67-127 (write_csv), fmt6 = snprintf("%.6g")       */

/* fmt6 of n doubles into 16-byte NUL-padded slots (metrics.cpp:67-71). */
void dso_fmt6(const double* v, int64_t n, char* out16) {
    for (int64_t i = 0; i < n; ++i) {
        char buf[40];
        memset(out16 + 16 * i, 0, 16);
        snprintf(buf, sizeof buf, "%.6g", v[i]);
        memcpy(out16 + 16 * i, buf, strlen(buf));
    }
}

typedef struct {
    char* p;
    int64_t n, cap;
} sbuf;

static void sb_put(sbuf* b, const char* s, size_t k) {
    if (b->p && b->n + (int64_t)k <= b->cap) memcpy(b->p + b->n, s, k);
    b->n += (int64_t)k;
}
static void sb_str(sbuf* b, const char* s) { sb_put(b, s, strlen(s)); }
static void sb_g6(sbuf* b, double v) {
    char t[40];
    snprintf(t, sizeof t, "%.6g", v);
    sb_str(b, t);
}
static void sb_opt6(sbuf* b, int present, double v) { /* metrics.cpp:75 */
    if (present) sb_g6(b, v);
}
static void sb_i64(sbuf* b, long long v) {
    char t[32];
    snprintf(t, sizeof t, "%lld", v);
    sb_str(b, t);
}
static void sb_u64(sbuf* b, unsigned long long v) {
    char t[32];
    snprintf(t, sizeof t, "%llu", v);
    sb_str(b, t);
}

/* queries.csv bytes (metrics.cpp:104-115); returns the size, writes at most cap. */
int64_t dso_format_queries_csv(const ds_query_record* r, int64_t n, char* out, int64_t cap) {
    static const char* outcome[] = {"served_light", "served_heavy", "dropped", "late"};
    sbuf b = {out, 0, cap};
    sb_str(&b, "id,arrival,confidence,quality_light,quality_heavy,deadline,light_start,"
               "light_end,heavy_start,heavy_end,completion,outcome,delivered_quality\n");
    for (int64_t i = 0; i < n; ++i) {
        const ds_query_record* q = &r[i];
        sb_u64(&b, q->id); sb_str(&b, ",");
        sb_g6(&b, q->arrival); sb_str(&b, ",");
        sb_g6(&b, q->confidence); sb_str(&b, ",");
        sb_g6(&b, q->quality_light); sb_str(&b, ",");
        sb_g6(&b, q->quality_heavy); sb_str(&b, ",");
        sb_g6(&b, q->deadline); sb_str(&b, ",");
        sb_opt6(&b, q->present & DS_REC_LIGHT_START, q->light_start); sb_str(&b, ",");
        sb_opt6(&b, q->present & DS_REC_LIGHT_END, q->light_end); sb_str(&b, ",");
        sb_opt6(&b, q->present & DS_REC_HEAVY_START, q->heavy_start); sb_str(&b, ",");
        sb_opt6(&b, q->present & DS_REC_HEAVY_END, q->heavy_end); sb_str(&b, ",");
        sb_opt6(&b, q->present & DS_REC_COMPLETION, q->completion); sb_str(&b, ",");
        if (q->present & DS_REC_OUTCOME)
            sb_str(&b, (q->outcome >= 0 && q->outcome < 4) ? outcome[q->outcome] : "?");
        sb_str(&b, ",");
        sb_opt6(&b, q->present & DS_REC_DELIVERED_QUALITY, q->delivered_quality);
        sb_str(&b, "\n");
    }
    return b.n;
}

/* intervals.csv bytes (metrics.cpp:92-103). */
int64_t dso_format_intervals_csv(const ds_interval_snapshot* s, int64_t n, char* out,
                                 int64_t cap) {
    sbuf b = {out, 0, cap};
    sb_str(&b, "interval_start,demand_observed,demand_estimated,threshold,x1,x2,b1,b2,"
               "feasible,arrived,served_light,served_heavy,dropped,late,"
               "mean_delivered_quality\n");
    for (int64_t i = 0; i < n; ++i) {
        const ds_interval_snapshot* r = &s[i];
        sb_g6(&b, r->interval_start); sb_str(&b, ",");
        sb_g6(&b, r->demand_observed); sb_str(&b, ",");
        sb_g6(&b, r->demand_estimated); sb_str(&b, ",");
        sb_g6(&b, r->threshold); sb_str(&b, ",");
        sb_i64(&b, r->plan.x1); sb_str(&b, ",");
        sb_i64(&b, r->plan.x2); sb_str(&b, ",");
        sb_i64(&b, r->plan.b1); sb_str(&b, ",");
        sb_i64(&b, r->plan.b2); sb_str(&b, ",");
        sb_str(&b, r->plan.feasible ? "1" : "0"); sb_str(&b, ",");
        sb_u64(&b, r->arrived); sb_str(&b, ",");
        sb_u64(&b, r->served_light); sb_str(&b, ",");
        sb_u64(&b, r->served_heavy); sb_str(&b, ",");
        sb_u64(&b, r->dropped); sb_str(&b, ",");
        sb_u64(&b, r->late); sb_str(&b, ",");
        sb_opt6(&b, r->has_mean_delivered_quality, r->mean_delivered_quality);
        sb_str(&b, "\n");
    }
    return b.n;
}

/* plans.csv bytes (metrics.cpp:117-126). */
int64_t dso_format_plans_csv(const ds_plan_log_entry* e, int64_t n, char* out, int64_t cap) {
    sbuf b = {out, 0, cap};
    sb_str(&b, "tick,time,demand_estimated,threshold,x1,x2,b1,b2,feasible\n");
    for (int64_t i = 0; i < n; ++i) {
        const ds_plan_log_entry* r = &e[i];
        sb_i64(&b, r->tick); sb_str(&b, ",");
        sb_g6(&b, r->time); sb_str(&b, ",");
        sb_g6(&b, r->demand_estimated); sb_str(&b, ",");
        sb_g6(&b, r->plan.threshold); sb_str(&b, ",");
        sb_i64(&b, r->plan.x1); sb_str(&b, ",");
        sb_i64(&b, r->plan.x2); sb_str(&b, ",");
        sb_i64(&b, r->plan.b1); sb_str(&b, ",");
        sb_i64(&b, r->plan.b2); sb_str(&b, ",");
        sb_str(&b, r->plan.feasible ? "1" : "0");
        sb_str(&b, "\n");
    }
    return b.n;
}

/* ---------------------------------------------------------------------- */
/* Deferral curve: profiles.cpp:60-71, 75-120                              */

static int bin_of(double c) { /* profiles.cpp:60-65 */
    int idx = (int)floor(c * 100.0 + 1e-9);
    return idx < 0 ? 0 : (idx > DS_CURVE_BINS - 1 ? DS_CURVE_BINS - 1 : idx);
}
static int bins_below(double t) { /* profiles.cpp:67-71 */
    int k = (int)ceil(t * 100.0 - 1e-9);
    return k < 0 ? 0 : (k > DS_CURVE_BINS ? DS_CURVE_BINS : k);
}
int dso_bin_of(double c) { return bin_of(c); }
int dso_bins_below(double t) { return bins_below(t); }

int dso_deferral_fraction(const ds_curve* c, double t, double* out) { /* profiles.cpp:98-106 */
    if (!(t >= 0.0) || !(t <= 1.0)) return DS_ERR_DOMAIN;
    if (c->total_mass <= 0.0) {
        *out = 0.0;
        return DS_OK;
    }
    int k = bins_below(t);
    double below = 0.0;
    for (int i = 0; i < k; ++i) below += c->bin_mass[i];
    *out = below / c->total_mass;
    return DS_OK;
}

int dso_observe(ds_curve* c, double conf, double decay) { /* profiles.cpp:108-120 */
    if (!(conf >= 0.0) || !(conf <= 1.0)) return DS_ERR_DOMAIN;
    if (!(decay > 0.0) || !(decay <= 1.0)) return DS_ERR_DOMAIN;
    if (decay != 1.0) {
        for (int i = 0; i < DS_CURVE_BINS; ++i) c->bin_mass[i] *= decay;
        c->total_mass *= decay;
    }
    c->bin_mass[bin_of(conf)] += 1.0;
    c->total_mass += 1.0;
    return DS_OK;
}

int dso_curve_observe(ds_curve* c, const double* conf, int64_t n, double decay) {
    for (int64_t i = 0; i < n; ++i) {
        int s = dso_observe(c, conf[i], decay);
        if (s) return s;
    }
    return DS_OK;
}

/* Strict-threshold routing (policies.cpp:37-39) with order-preserving
 * compaction, for nt thresholds; heavy list k at heavy_idx[k*n ..]. */
void dso_route(const double* conf, int64_t n, const double* t, int nt, int64_t index_base,
               int64_t* heavy_idx, int64_t* counts) {
    for (int k = 0; k < nt; ++k) {
        int64_t m = 0;
        for (int64_t i = 0; i < n; ++i)
            if (conf[i] < t[k]) heavy_idx[(int64_t)k * n + m++] = index_base + i;
        counts[k] = m;
    }
}

/* cluster.cpp:290-306 minus the DES: observe then defers, per query. */
int dso_route_loop(const double* conf, int64_t n, double t, int observe, double decay,
                   ds_curve* curve, int64_t* heavy_idx, int64_t* count) {
    int64_t m = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (observe) {
            int s = dso_observe(curve, conf[i], decay);
            if (s) return s;
        }
        if (conf[i] < t) heavy_idx[m++] = i;
    }
    *count = m;
    return DS_OK;
}

/* ---------------------------------------------------------------------- */
/* Planner: allocator.cpp:12-313                                           */

static int find_batch(const ds_model_profile* m, int b) {
    for (int i = 0; i < m->n; ++i)
        if (m->batch[i] == b) return i;
    return -1;
}
static double exec_latency(const ds_model_profile* m, int b, int* err) { /* profiles.cpp:20-26 */
    int i = find_batch(m, b);
    if (i < 0) {
        *err = DS_ERR_OUT_OF_RANGE;
        return 0.0;
    }
    return m->latency[i];
}
static double tput(const ds_model_profile* m, int b, int* err) { /* profiles.cpp:28-30 */
    return (double)b / exec_latency(m, b, err);
}

static double queuing_delay(int64_t len, double rate, double sentinel) { /* allocator.cpp:12-18 */
    if (len == 0) return 0.0;
    if (rate == 0.0) return sentinel;
    return (double)len / rate;
}

static int check_problem(const ds_problem* p) { /* allocator.cpp:22-28 */
    if (p->total_servers < 1) return DS_ERR_DOMAIN;
    if (!(p->demand_qps >= 0.0)) return DS_ERR_DOMAIN;
    if (!(p->overprovision_lambda >= 1.0)) return DS_ERR_DOMAIN;
    return DS_OK;
}
static int check_grid(const double* g, int n) { /* allocator.cpp:30-36 */
    if (n == 0 || g[0] != 0.0) return DS_ERR_INVARIANT;
    for (int i = 1; i < n; ++i)
        if (!(g[i] > g[i - 1])) return DS_ERR_INVARIANT;
    return DS_OK;
}

/* allocator.cpp:45-51. x86 cvttsd2si gives INT_MIN for out-of-range values;
 * (int)ceil(q) is restated with that behaviour so huge quotients behave as in
 * the reference build (x := 1, then the bounded while loop). */
static int min_servers(double need, double per, int cap) {
    if (need <= 0.0) return 0;
    double q = ceil(need / per);
    int x = (q >= -2147483648.0 && q < 2147483648.0) ? (int)q : (int)0x80000000u;
    if (x < 1) x = 1;
    while (x <= cap && x * per < need) ++x;
    return x;
}

static int latency_ok(const ds_problem* p, const ds_cascade* c, int b1, int b2, int* err) {
    /* allocator.cpp:129-142 */
    double e1 = exec_latency(&c->light, b1, err);
    double e2 = exec_latency(&c->heavy, b2, err);
    double q1, q2;
    if (p->queuing == DS_QUEUING_TWICE_EXEC) {
        q1 = 2.0 * e1;
        q2 = 2.0 * e2;
    } else {
        q1 = queuing_delay(p->light_len, p->light_rate, p->queue_sentinel_seconds);
        q2 = queuing_delay(p->heavy_len, p->heavy_rate, p->queue_sentinel_seconds);
    }
    return e1 + q1 + e2 + q2 <= c->slo_seconds;
}

typedef struct {
    ds_plan plan;
    int valid;
} cand;

static int better_than(const cand* a, const cand* o) { /* allocator.cpp:57-67 */
    if (!o->valid) return a->valid;
    if (!a->valid) return 0;
    int t = a->plan.x1 + a->plan.x2, ot = o->plan.x1 + o->plan.x2;
    if (t != ot) return t < ot;
    if (a->plan.b1 != o->plan.b1) return a->plan.b1 > o->plan.b1;
    if (a->plan.b2 != o->plan.b2) return a->plan.b2 > o->plan.b2;
    return a->plan.x1 < o->plan.x1;
}

static ds_plan best_effort_light(const ds_problem* p, const ds_cascade* c) { /* allocator.cpp:70-88 */
    int err = 0;
    int best_b = c->light.batch[0];
    double best_T = tput(&c->light, best_b, &err);
    for (int i = 0; i < c->light.n; ++i) {
        double T = tput(&c->light, c->light.batch[i], &err);
        if (T >= best_T) {
            best_T = T;
            best_b = c->light.batch[i];
        }
    }
    ds_plan plan = {0};
    plan.x1 = p->total_servers;
    plan.x2 = 0;
    plan.b1 = best_b;
    plan.b2 = c->heavy.batch[0];
    plan.threshold = 0.0;
    plan.feasible = 0;
    return plan;
}

/* allocator.cpp:91-121 over the descending threshold list `td`. */
static cand search(const ds_problem* p, const ds_cascade* c, const double* td, int nt,
                   const int* b1s, int n1, const int* b2s, int n2, int* err) {
    const double need_light = p->overprovision_lambda * p->demand_qps;
    int pb1[DS_MAX_BATCHES * DS_MAX_BATCHES], pb2[DS_MAX_BATCHES * DS_MAX_BATCHES];
    int np = 0;
    for (int i = 0; i < n1; ++i)
        for (int j = 0; j < n2; ++j)
            if (latency_ok(p, c, b1s[i], b2s[j], err)) {
                pb1[np] = b1s[i];
                pb2[np] = b2s[j];
                ++np;
            }
    for (int k = 0; k < nt; ++k) {
        double t = td[k], f = 0.0;
        int s = dso_deferral_fraction(&c->deferral, t, &f);
        if (s) {
            *err = s;
            return (cand){{0}, 0};
        }
        double need_heavy = need_light * f;
        cand best = {{0}, 0};
        for (int q = 0; q < np; ++q) {
            double T1 = tput(&c->light, pb1[q], err);
            double T2 = tput(&c->heavy, pb2[q], err);
            int x1 = min_servers(need_light, T1, p->total_servers);
            if (x1 < 1) x1 = 1;
            if (x1 > p->total_servers) continue;
            int x2 = min_servers(need_heavy, T2, p->total_servers);
            if (x1 + x2 > p->total_servers) continue;
            cand cd = {{x1, x2, pb1[q], pb2[q], t, 1, 0}, 1};
            if (better_than(&cd, &best)) best = cd;
        }
        if (best.valid) return best;
    }
    return (cand){{0}, 0};
}

static int single_model(const ds_model_profile* m, int is_light, int S, double demand,
                        double lambda, double slo, ds_plan* plan) { /* allocator.cpp:232-268 */
    if (S < 1) return DS_ERR_DOMAIN;
    int err = 0;
    double need = lambda * demand;
    int adm[DS_MAX_BATCHES], na = 0;
    for (int i = 0; i < m->n; ++i)
        if (2.0 * m->latency[i] <= slo) adm[na++] = m->batch[i];
    memset(plan, 0, sizeof(*plan));
    plan->threshold = 0.0;
#define ASSIGN(b, feas)                                                                        \
    do {                                                                                       \
        if (is_light) { plan->x1 = S; plan->x2 = 0; plan->b1 = (b); plan->b2 = 0; }           \
        else { plan->x1 = 0; plan->x2 = S; plan->b1 = 0; plan->b2 = (b); }                     \
        plan->feasible = (feas);                                                               \
    } while (0)
    for (int i = 0; i < na; ++i)
        if (S * tput(m, adm[i], &err) >= need) {
            ASSIGN(adm[i], 1);
            return DS_OK;
        }
    if (na > 0) {
        int best_b = adm[0];
        for (int i = 0; i < na; ++i)
            if (tput(m, adm[i], &err) >= tput(m, best_b, &err)) best_b = adm[i];
        ASSIGN(best_b, 0);
        return DS_OK;
    }
    ASSIGN(m->batch[0], 0);
#undef ASSIGN
    return DS_OK;
}

static void cheapest(const ds_model_profile* m, double slo, double side_need, int cap, int* bx,
                     int* bb) { /* allocator.cpp:283-291 */
    int err = 0;
    int best_x = cap + 1, best_b = 0;
    for (int i = 0; i < m->n; ++i) {
        if (!(2.0 * m->latency[i] <= slo)) continue;
        int b = m->batch[i];
        int x = min_servers(side_need, tput(m, b, &err), cap);
        if (x < 1) x = 1;
        if (x < best_x || (x == best_x && b > best_b)) {
            best_x = x;
            best_b = b;
        }
    }
    *bx = best_x;
    *bb = best_b;
}

int dso_solve_one(const ds_problem* p, const ds_cascade* c, const double* grid, int g,
                  ds_plan* out) {
    /* solve_single_model (allocator.cpp:232-236) checks only S >= 1; every
     * other entry point runs check_problem first. */
    int err = 0;
    if (p->mode != DS_SOLVE_SINGLE_LIGHT && p->mode != DS_SOLVE_SINGLE_HEAVY &&
        (err = check_problem(p)))
        return err;
    double td[4096];
    int b1s[DS_MAX_BATCHES], b2s[DS_MAX_BATCHES];
    for (int i = 0; i < c->light.n; ++i) b1s[i] = c->light.batch[i];
    for (int i = 0; i < c->heavy.n; ++i) b2s[i] = c->heavy.batch[i];
    memset(out, 0, sizeof(*out));
    switch (p->mode) {
    case DS_SOLVE: { /* allocator.cpp:153-169 */
        if ((err = check_grid(grid, g))) return err;
        if (g > 4096) return DS_ERR_CAPACITY;
        for (int i = 0; i < g; ++i) td[i] = grid[g - 1 - i];
        cand best = search(p, c, td, g, b1s, c->light.n, b2s, c->heavy.n, &err);
        if (err) return err;
        *out = best.valid ? best.plan : best_effort_light(p, c);
        return DS_OK;
    }
    case DS_SOLVE_PINNED: { /* allocator.cpp:176-211 */
        double ft = p->fixed_threshold;
        if (!(ft >= 0.0) || !(ft <= 1.0)) return DS_ERR_DOMAIN;
        cand best = search(p, c, &ft, 1, b1s, c->light.n, b2s, c->heavy.n, &err);
        if (err) return err;
        if (best.valid) {
            *out = best.plan;
            return DS_OK;
        }
        double need = p->overprovision_lambda * p->demand_qps, f = 0.0;
        dso_deferral_fraction(&c->deferral, ft, &f);
        double need_heavy = need * f;
        cand pick = {{0}, 0};
        for (int i = 0; i < c->light.n; ++i)
            for (int j = 0; j < c->heavy.n; ++j) {
                int b1 = b1s[i], b2 = b2s[j];
                double T1 = tput(&c->light, b1, &err), T2 = tput(&c->heavy, b2, &err);
                int x1 = min_servers(need, T1, p->total_servers);
                if (x1 < 1) x1 = 1;
                if (x1 > p->total_servers) x1 = p->total_servers;
                int x2 = min_servers(need_heavy, T2, p->total_servers);
                if (x2 > p->total_servers - x1) x2 = p->total_servers - x1;
                double d1 = need - x1 * T1, d2 = need_heavy - x2 * T2;
                double deficit = (d1 > 0.0 ? d1 : 0.0) + (d2 > 0.0 ? d2 : 0.0);
                cand cd = {{x1, x2, b1, b2, ft, 0, 0}, 1};
                double best_deficit = INFINITY;
                if (pick.valid) {
                    double e1 = need - pick.plan.x1 * tput(&c->light, pick.plan.b1, &err);
                    double e2 = need_heavy - pick.plan.x2 * tput(&c->heavy, pick.plan.b2, &err);
                    best_deficit = (e1 > 0.0 ? e1 : 0.0) + (e2 > 0.0 ? e2 : 0.0);
                }
                if (deficit < best_deficit || (deficit == best_deficit && better_than(&cd, &pick)))
                    pick = cd;
            }
        *out = pick.plan;
        return DS_OK;
    }
    case DS_SOLVE_FIXED_BATCHES: { /* allocator.cpp:213-230 */
        if ((err = check_grid(grid, g))) return err;
        if (g > 4096) return DS_ERR_CAPACITY;
        int b1 = p->fixed_b1, b2 = p->fixed_b2;
        if (find_batch(&c->light, b1) < 0 || find_batch(&c->heavy, b2) < 0)
            return DS_ERR_OUT_OF_RANGE;
        for (int i = 0; i < g; ++i) td[i] = grid[g - 1 - i];
        cand best = search(p, c, td, g, &b1, 1, &b2, 1, &err);
        if (err) return err;
        if (best.valid) {
            *out = best.plan;
            return DS_OK;
        }
        double need = p->overprovision_lambda * p->demand_qps;
        double T1 = tput(&c->light, b1, &err);
        int x1 = min_servers(need, T1, p->total_servers);
        if (x1 < 1) x1 = 1;
        out->x1 = x1 < p->total_servers ? x1 : p->total_servers;
        out->x2 = 0;
        out->b1 = b1;
        out->b2 = b2;
        out->threshold = 0.0;
        out->feasible = 0;
        return DS_OK;
    }
    case DS_SOLVE_EVEN_SPLIT: { /* allocator.cpp:270-313 */
        double need = p->overprovision_lambda * p->demand_qps;
        int xh, bh;
        cheapest(&c->heavy, c->slo_seconds, need, p->total_servers, &xh, &bh);
        if (bh != 0 && xh <= p->total_servers) {
            *out = (ds_plan){0, xh, 0, bh, 0.0, 1, 0};
            return DS_OK;
        }
        int x1, b1, x2, b2;
        cheapest(&c->light, c->slo_seconds, need / 2.0, p->total_servers, &x1, &b1);
        cheapest(&c->heavy, c->slo_seconds, need / 2.0, p->total_servers, &x2, &b2);
        if (b1 != 0 && b2 != 0 && x1 + x2 <= p->total_servers) {
            *out = (ds_plan){x1, x2, b1, b2, 0.0, 1, 0};
            return DS_OK;
        }
        single_model(&c->light, 1, p->total_servers, p->demand_qps, p->overprovision_lambda,
                     c->slo_seconds, out);
        out->b2 = c->heavy.batch[0];
        return DS_OK;
    }
    case DS_SOLVE_SINGLE_LIGHT:
    case DS_SOLVE_SINGLE_HEAVY:
        return single_model(p->mode == DS_SOLVE_SINGLE_LIGHT ? &c->light : &c->heavy,
                            p->mode == DS_SOLVE_SINGLE_LIGHT, p->total_servers, p->demand_qps,
                            p->overprovision_lambda, c->slo_seconds, out);
    }
    return DS_ERR_INVALID_ARGUMENT;
}

/* Threshold-range restatement of search (allocator.cpp:91-121) for the
 * t-sharded planner: grid indices [t_lo, t_hi) walked from the top, the
 * winner encoded as the packed key whose unsigned order is the reference's
 * choice order (first valid t from the top, then better_than):
 *   (G-1-t_idx)<<40 | (x1+x2)<<28 | (255-b1_idx)<<20 | (255-b2_idx)<<12 | x1.
 * UINT64_MAX when the slice has no valid candidate or the mode is not a grid
 * mode (DS_SOLVE, DS_SOLVE_FIXED_BATCHES). Inputs are assumed valid. */
int dso_plan_keys(const ds_problem* problems, int32_t n, const ds_cascade* cascades,
                  const double* grid_values, const int32_t* grid_offsets, int32_t t_lo,
                  int32_t t_hi, uint64_t* keys) {
    for (int i = 0; i < n; ++i) {
        const ds_problem* p = &problems[i];
        const ds_cascade* c = &cascades[p->cascade];
        keys[i] = UINT64_MAX;
        if (p->mode != DS_SOLVE && p->mode != DS_SOLVE_FIXED_BATCHES) continue;
        const double* g = grid_values + grid_offsets[p->grid];
        const int G = grid_offsets[p->grid + 1] - grid_offsets[p->grid];
        int b1s[DS_MAX_BATCHES], b2s[DS_MAX_BATCHES], n1 = 0, n2 = 0;
        for (int k = 0; k < c->light.n; ++k)
            if (p->mode == DS_SOLVE || c->light.batch[k] == p->fixed_b1) b1s[n1++] = c->light.batch[k];
        for (int k = 0; k < c->heavy.n; ++k)
            if (p->mode == DS_SOLVE || c->heavy.batch[k] == p->fixed_b2) b2s[n2++] = c->heavy.batch[k];
        const int hi = t_hi < G ? t_hi : G, lo = t_lo > 0 ? t_lo : 0;
        int err = 0;
        for (int t = hi - 1; t >= lo; --t) {
            cand best = search(p, c, &g[t], 1, b1s, n1, b2s, n2, &err);
            if (err) return err;
            if (!best.valid) continue;
            const int bi = find_batch(&c->light, best.plan.b1), bj = find_batch(&c->heavy, best.plan.b2);
            keys[i] = ((uint64_t)(G - 1 - t) << 40) | ((uint64_t)(best.plan.x1 + best.plan.x2) << 28) |
                      ((uint64_t)(255 - bi) << 20) | ((uint64_t)(255 - bj) << 12) |
                      (uint64_t)best.plan.x1;
            break;
        }
    }
    return DS_OK;
}

typedef struct {
    const ds_problem* p;
    const ds_cascade* c;
    const double* gv;
    const int32_t* go;
    ds_plan* out;
    int32_t* status;
    int lo, hi;
} plan_job;

static void* plan_worker(void* arg) {
    plan_job* j = (plan_job*)arg;
    for (int i = j->lo; i < j->hi; ++i) {
        const ds_problem* p = &j->p[i];
        j->status[i] = dso_solve_one(p, &j->c[p->cascade], j->gv + j->go[p->grid],
                                     j->go[p->grid + 1] - j->go[p->grid], &j->out[i]);
    }
    return NULL;
}

/* Solves n problems on `threads` POSIX threads; per-problem status codes. */
int dso_plan_batch(const ds_problem* problems, int32_t n, const ds_cascade* cascades,
                   const double* grid_values, const int32_t* grid_offsets, ds_plan* out,
                   int32_t* status, int threads) {
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pthread_t tid[256];
    plan_job jobs[256];
    for (int k = 0; k < threads; ++k) {
        jobs[k] = (plan_job){problems, cascades, grid_values, grid_offsets, out, status,
                             (int)((int64_t)n * k / threads), (int)((int64_t)n * (k + 1) / threads)};
        if (threads == 1) plan_worker(&jobs[0]);
        else pthread_create(&tid[k], NULL, plan_worker, &jobs[k]);
    }
    if (threads > 1)
        for (int k = 0; k < threads; ++k) pthread_join(tid[k], NULL);
    for (int i = 0; i < n; ++i)
        if (status[i]) return status[i];
    return DS_OK;
}
