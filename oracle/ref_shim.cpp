// TEST INFRASTRUCTURE ONLY -- the checker, never the product.
//
// extern "C" shim over the UNMODIFIED reference library compiled from
// /root/reference/proj/src/*.cpp by oracle/Makefile into oracle/_ref/libdsref.so.
// It lets the Python tests and bench.py's reference arm call the reference's
// own solve / sample_query / observe_confidence / defers through ctypes, on
// the POD types of include/ds_gpu.h. Only tests/, __graft_entry__.smoke() and
// bench.py (cpu_baseline leg and --impl reference) may load it.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "diffserve/allocator.hpp"
#include "diffserve/errors.hpp"
#include "diffserve/metrics.hpp"
#include "diffserve/policies.hpp"
#include "diffserve/profiles.hpp"
#include "diffserve/rng.hpp"
#include "diffserve/workload.hpp"
#include "ds_gpu.h"

using namespace diffserve;

namespace {

thread_local std::string g_err;

int map_exception() {
    try {
        throw;
    } catch (const InvariantError& e) {
        g_err = e.what();
        return DS_ERR_INVARIANT;
    } catch (const std::domain_error& e) {
        g_err = e.what();
        return DS_ERR_DOMAIN;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return DS_ERR_INVALID_ARGUMENT;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return DS_ERR_OUT_OF_RANGE;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 99;
    }
}

ModelProfile to_model(const ds_model_profile& m, const char* name) {
    ModelProfile out;
    out.name = name;
    for (int i = 0; i < m.n; ++i) out.latency_table[m.batch[i]] = m.latency[i];
    return out;
}

CascadeProfile to_cascade(const ds_cascade& c) {
    CascadeProfile out;
    out.name = "shim";
    out.light = to_model(c.light, "light");
    out.heavy = to_model(c.heavy, "heavy");
    out.deferral = DeferralCurve::empty();
    for (int i = 0; i < DS_CURVE_BINS; ++i) out.deferral.bin_mass[i] = c.deferral.bin_mass[i];
    out.deferral.total_mass = c.deferral.total_mass;
    out.slo_seconds = c.slo_seconds;
    return out;
}

void from_model(const ModelProfile& m, ds_model_profile& out) {
    std::memset(&out, 0, sizeof(out));
    int i = 0;
    for (const auto& [b, e] : m.latency_table) {
        out.batch[i] = b;
        out.latency[i] = e;
        ++i;
    }
    out.n = i;
}

void from_cascade(const CascadeProfile& c, ds_cascade& out) {
    std::memset(&out, 0, sizeof(out));
    from_model(c.light, out.light);
    from_model(c.heavy, out.heavy);
    for (int i = 0; i < DS_CURVE_BINS; ++i) out.deferral.bin_mass[i] = c.deferral.bin_mass[i];
    out.deferral.total_mass = c.deferral.total_mass;
    out.slo_seconds = c.slo_seconds;
}

AllocationProblem to_problem(const ds_problem& p, const CascadeProfile* c, const double* grid,
                             int g) {
    AllocationProblem out;
    out.demand_qps = p.demand_qps;
    out.total_servers = p.total_servers;
    out.cascade = c;
    out.overprovision_lambda = p.overprovision_lambda;
    out.threshold_grid.assign(grid, grid + g);
    out.light_queue = QueueState{p.light_len, p.light_rate};
    out.heavy_queue = QueueState{p.heavy_len, p.heavy_rate};
    out.queuing = p.queuing == DS_QUEUING_TWICE_EXEC ? QueuingModel::twice_exec
                                                     : QueuingModel::littles_law;
    out.queue_sentinel_seconds = p.queue_sentinel_seconds;
    return out;
}

void from_problem(const AllocationProblem& p, ds_problem& out) {
    std::memset(&out, 0, sizeof(out));
    out.demand_qps = p.demand_qps;
    out.overprovision_lambda = p.overprovision_lambda;
    out.queue_sentinel_seconds = p.queue_sentinel_seconds;
    out.light_rate = p.light_queue.arrival_rate;
    out.heavy_rate = p.heavy_queue.arrival_rate;
    out.light_len = p.light_queue.queue_length;
    out.heavy_len = p.heavy_queue.queue_length;
    out.total_servers = p.total_servers;
    out.queuing = p.queuing == QueuingModel::twice_exec ? DS_QUEUING_TWICE_EXEC
                                                        : DS_QUEUING_LITTLES_LAW;
}

ds_plan from_plan(const AllocationPlan& p) {
    ds_plan out{};
    out.x1 = p.x1;
    out.x2 = p.x2;
    out.b1 = p.b1;
    out.b2 = p.b2;
    out.threshold = p.threshold;
    out.feasible = p.feasible ? 1 : 0;
    return out;
}

AllocationPlan run_mode(const ds_problem& dp, const AllocationProblem& p) {
    switch (dp.mode) {
    case DS_SOLVE: return solve(p);
    case DS_SOLVE_PINNED: return solve_pinned_threshold(p, dp.fixed_threshold);
    case DS_SOLVE_FIXED_BATCHES: return solve_fixed_batches(p, dp.fixed_b1, dp.fixed_b2);
    case DS_SOLVE_EVEN_SPLIT: return solve_even_split(p);
    case DS_SOLVE_SINGLE_LIGHT:
        return solve_single_model(p.cascade->light, true, p.total_servers, p.demand_qps,
                                  p.overprovision_lambda, p.cascade->slo_seconds);
    case DS_SOLVE_SINGLE_HEAVY:
        return solve_single_model(p.cascade->heavy, false, p.total_servers, p.demand_qps,
                                  p.overprovision_lambda, p.cascade->slo_seconds);
    }
    throw std::invalid_argument("unknown solve mode");
}

} // namespace

extern "C" {

const char* dsref_last_error(void) { return g_err.c_str(); }

// diffserve::solve and variants over n problems; threads > 1 splits problem
// indices across std::threads (solve is pure). Returns the first
// failing problem's status (its plan slot is left zeroed).
int dsref_plan_batch(const ds_problem* problems, int32_t n, const ds_cascade* cascades,
                     int32_t n_cascades, const double* grid_values, const int32_t* grid_offsets,
                     int32_t n_grids, ds_plan* out, int32_t threads) {
    std::vector<CascadeProfile> cs;
    cs.reserve(static_cast<size_t>(n_cascades));
    for (int i = 0; i < n_cascades; ++i) cs.push_back(to_cascade(cascades[i]));
    std::vector<int> status(static_cast<size_t>(n), 0);
    std::vector<std::string> errs(static_cast<size_t>(n));
    auto work = [&](int lo, int hi) {
        for (int i = lo; i < hi; ++i) {
            const ds_problem& dp = problems[i];
            try {
                const int g = dp.grid;
                if (g < 0 || g >= n_grids) throw std::invalid_argument("grid index");
                if (dp.cascade < 0 || dp.cascade >= n_cascades)
                    throw std::invalid_argument("cascade index");
                AllocationProblem p = to_problem(dp, &cs[static_cast<size_t>(dp.cascade)],
                                                 grid_values + grid_offsets[g],
                                                 grid_offsets[g + 1] - grid_offsets[g]);
                out[i] = from_plan(run_mode(dp, p));
            } catch (...) {
                status[static_cast<size_t>(i)] = map_exception();
                errs[static_cast<size_t>(i)] = g_err;
                out[i] = ds_plan{};
            }
        }
    };
    if (threads <= 1 || n < 2) {
        work(0, n);
    } else {
        std::vector<std::thread> pool;
        const int t = std::min<int>(threads, n);
        for (int k = 0; k < t; ++k) {
            const int lo = static_cast<int>(static_cast<int64_t>(n) * k / t);
            const int hi = static_cast<int>(static_cast<int64_t>(n) * (k + 1) / t);
            pool.emplace_back(work, lo, hi);
        }
        for (auto& th : pool) th.join();
    }
    for (int i = 0; i < n; ++i)
        if (status[static_cast<size_t>(i)]) {
            g_err = errs[static_cast<size_t>(i)];
            return status[static_cast<size_t>(i)];
        }
    return 0;
}

// One run of a Policy from make_policy (policies.cpp:198-219) -- the
// reference's per-kind control logic -- over n ticks: tick i calls
// plan(problems[i]) -> out[i], then observe_batch(ev_model[i] (0 light,
// 1 heavy), ev_timeout[i]) and records live_batch(light/heavy) ->
// live[2i], live[2i+1], and entry_stage(out[i], rng) -> entry[i] (0 light,
// 1 heavy) from RandomStream(seed, "entry").
int dsref_policy_run(int32_t kind, double peak, double fixed_t, int32_t add_step, double mult,
                     const ds_problem* problems, int32_t n, const ds_cascade* cascade,
                     const double* grid, int32_t g, const int32_t* ev_model,
                     const int32_t* ev_timeout, uint64_t seed, ds_plan* out, int32_t* live,
                     int32_t* entry) {
    try {
        PolicyParams pp;
        pp.kind = static_cast<PolicyKind>(kind);
        pp.peak_demand_qps = peak;
        pp.fixed_threshold = fixed_t;
        pp.aimd_add_step = add_step;
        pp.aimd_mult_factor = mult;
        std::unique_ptr<Policy> pol = make_policy(pp);
        CascadeProfile c = to_cascade(*cascade);
        RandomStream rng(seed, "entry");
        for (int i = 0; i < n; ++i) {
            AllocationProblem p = to_problem(problems[i], &c, grid, g);
            AllocationPlan pl = pol->plan(p);
            out[i] = from_plan(pl);
            pol->observe_batch(ev_model[i] ? ModelKind::heavy : ModelKind::light,
                               ev_timeout[i] != 0);
            live[2 * i] = pol->live_batch(ModelKind::light);
            live[2 * i + 1] = pol->live_batch(ModelKind::heavy);
            entry[i] = pol->entry_stage(pl, rng) == ModelKind::heavy ? 1 : 0;
        }
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// Predicates, for property tests (allocator.cpp:129-151).
int dsref_latency_feasible(const ds_problem* dp, const ds_cascade* c, const double* grid, int g,
                           int b1, int b2, int* out) {
    try {
        CascadeProfile cp = to_cascade(*c);
        AllocationProblem p = to_problem(*dp, &cp, grid, g);
        *out = latency_feasible(p, b1, b2) ? 1 : 0;
        return 0;
    } catch (...) {
        return map_exception();
    }
}

int dsref_throughput_feasible(const ds_problem* dp, const ds_cascade* c, const double* grid,
                              int g, const ds_plan* plan, int* out) {
    try {
        CascadeProfile cp = to_cascade(*c);
        AllocationProblem p = to_problem(*dp, &cp, grid, g);
        AllocationPlan ap{plan->x1, plan->x2, plan->b1, plan->b2, plan->threshold,
                          plan->feasible != 0};
        *out = throughput_feasible(p, ap) ? 1 : 0;
        return 0;
    } catch (...) {
        return map_exception();
    }
}

double dsref_deferral_fraction(const ds_curve* curve, double t, int* status) {
    try {
        DeferralCurve c = DeferralCurve::empty();
        for (int i = 0; i < DS_CURVE_BINS; ++i) c.bin_mass[i] = curve->bin_mass[i];
        c.total_mass = curve->total_mass;
        *status = 0;
        return deferral_fraction(c, t);
    } catch (...) {
        *status = map_exception();
        return 0.0;
    }
}

// Curve constructors (profiles.cpp:75-96).
void dsref_curve_empty(ds_curve* out) {
    DeferralCurve c = DeferralCurve::empty();
    for (int i = 0; i < DS_CURVE_BINS; ++i) out->bin_mass[i] = c.bin_mass[i];
    out->total_mass = c.total_mass;
}
void dsref_curve_uniform_prior(ds_curve* out) {
    DeferralCurve c = DeferralCurve::uniform_prior();
    for (int i = 0; i < DS_CURVE_BINS; ++i) out->bin_mass[i] = c.bin_mass[i];
    out->total_mass = c.total_mass;
}
int dsref_curve_from_samples(const double* s, int64_t n, ds_curve* out) {
    try {
        DeferralCurve c = DeferralCurve::from_samples(std::vector<double>(s, s + n));
        for (int i = 0; i < DS_CURVE_BINS; ++i) out->bin_mass[i] = c.bin_mass[i];
        out->total_mass = c.total_mass;
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// observe_confidence over a sequence, in order (profiles.cpp:108-120).
int dsref_curve_observe(ds_curve* curve, const double* conf, int64_t n, double decay) {
    try {
        DeferralCurve c = DeferralCurve::empty();
        for (int i = 0; i < DS_CURVE_BINS; ++i) c.bin_mass[i] = curve->bin_mass[i];
        c.total_mass = curve->total_mass;
        for (int64_t i = 0; i < n; ++i) observe_confidence(c, conf[i], decay);
        for (int i = 0; i < DS_CURVE_BINS; ++i) curve->bin_mass[i] = c.bin_mass[i];
        curve->total_mass = c.total_mass;
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// sample_query over ids id0..id0+n-1 (workload.cpp:108-129), threads split ids.
int dsref_sample_queries(const ds_query_model* m, uint64_t id0, int64_t n, double slo,
                         double* conf, double* quality_light, int32_t threads) {
    QueryOutcomeModel qm;
    qm.easy_fraction = m->easy_fraction;
    qm.quality_gap_scale = m->quality_gap_scale;
    qm.confidence_fidelity = m->confidence_fidelity;
    qm.noise_sigma = m->noise_sigma;
    qm.seed = m->seed;
    try {
        (void)sample_query(qm, id0, 0.0, slo); // validate once on this thread
    } catch (...) {
        return map_exception();
    }
    auto work = [&](int64_t lo, int64_t hi) {
        for (int64_t i = lo; i < hi; ++i) {
            Query q = sample_query(qm, id0 + static_cast<uint64_t>(i), 0.0, slo);
            conf[i] = q.confidence;
            if (quality_light) quality_light[i] = q.quality_light;
        }
    };
    if (threads <= 1 || n < 1024) {
        work(0, n);
    } else {
        std::vector<std::thread> pool;
        for (int k = 0; k < threads; ++k)
            pool.emplace_back(work, n * k / threads, n * (k + 1) / threads);
        for (auto& th : pool) th.join();
    }
    return 0;
}

// The light-batch completion loop of cluster.cpp:290-306 with the DES enqueue
// replaced by an append: per query in order, observe into the curve (when
// observe != 0), then Policy::defers(c, t) -> append id to the heavy list.
int dsref_route_loop(const double* conf, int64_t n, double t, int32_t observe, double decay,
                     ds_curve* curve, int64_t* heavy_idx, int64_t* count) {
    try {
        auto policy = make_policy(PolicyParams{});
        DeferralCurve c = DeferralCurve::empty();
        for (int i = 0; i < DS_CURVE_BINS; ++i) c.bin_mass[i] = curve->bin_mass[i];
        c.total_mass = curve->total_mass;
        int64_t k = 0;
        for (int64_t i = 0; i < n; ++i) {
            if (observe) observe_confidence(c, conf[i], decay);
            if (policy->defers(conf[i], t)) heavy_idx[k++] = i;
        }
        *count = k;
        for (int i = 0; i < DS_CURVE_BINS; ++i) curve->bin_mass[i] = c.bin_mass[i];
        curve->total_mass = c.total_mass;
        return 0;
    } catch (...) {
        return map_exception();
    }
}

int dsref_defers(double c, double t) {
    auto policy = make_policy(PolicyParams{});
    return policy->defers(c, t) ? 1 : 0;
}

// Loads a cascade from a profile file (profiles.cpp:262-355).
int dsref_load_cascade(const char* path, const char* name, ds_cascade* out) {
    try {
        from_cascade(load_cascade(path, name), *out);
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// Exposed for the golden generators in ref_tests_*.cpp.
void dsref_from_cascade(const void* c, ds_cascade* out) {
    from_cascade(*static_cast<const CascadeProfile*>(c), *out);
}
void dsref_from_problem(const void* p, ds_problem* out) {
    from_problem(*static_cast<const AllocationProblem*>(p), *out);
}

// RNG primitives (rng.cpp:8-36) for the oracle's own checks.
// generate_arrivals (workload.cpp:82-106) on Trace{dt, rates}. Returns the
// arrival count and copies min(count, cap) timestamps; -1 on an exception.
int64_t dsref_generate_arrivals(const double* rates, int32_t n, double dt, uint64_t seed,
                                int32_t mode, double* out, int64_t cap) {
    try {
        Trace t;
        t.interval_seconds = dt;
        t.rates.assign(rates, rates + n);
        const auto a = generate_arrivals(t, seed, mode == 1 ? ArrivalMode::uniform
                                                            : ArrivalMode::poisson);
        const int64_t c = static_cast<int64_t>(a.size());
        for (int64_t i = 0; i < c && i < cap; ++i) out[i] = a[i];
        return c;
    } catch (...) {
        map_exception();
        return -1;
    }
}

// The run_experiment query loop (experiment.cpp:76-79) with ids id0.. :
// full Query records.
int dsref_sample_query_records(const ds_query_model* m, uint64_t id0, const double* arrivals,
                               int64_t n, double slo, ds_query* out) {
    QueryOutcomeModel qm;
    qm.easy_fraction = m->easy_fraction;
    qm.quality_gap_scale = m->quality_gap_scale;
    qm.confidence_fidelity = m->confidence_fidelity;
    qm.noise_sigma = m->noise_sigma;
    qm.seed = m->seed;
    try {
        for (int64_t i = 0; i < n; ++i) {
            const Query q = sample_query(qm, id0 + static_cast<uint64_t>(i), arrivals[i], slo);
            out[i] = ds_query{q.id, q.arrival, q.deadline, q.quality_light, q.quality_heavy,
                              q.confidence};
        }
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// The reference's write_csv (metrics.cpp:91-127) on POD rows, into dir.
static AllocationPlan to_plan(const ds_plan& p) {
    AllocationPlan a;
    a.x1 = p.x1;
    a.x2 = p.x2;
    a.b1 = p.b1;
    a.b2 = p.b2;
    a.threshold = p.threshold;
    a.feasible = p.feasible != 0;
    return a;
}

int dsref_write_csv(const char* dir, const ds_interval_snapshot* iv, int64_t ni,
                    const ds_query_record* qr, int64_t nq, const ds_plan_log_entry* pl,
                    int64_t np) {
    try {
        std::vector<IntervalSnapshot> ivs(static_cast<size_t>(ni));
        for (int64_t i = 0; i < ni; ++i) {
            IntervalSnapshot& s = ivs[static_cast<size_t>(i)];
            s.interval_start = iv[i].interval_start;
            s.demand_observed = iv[i].demand_observed;
            s.demand_estimated = iv[i].demand_estimated;
            s.plan = to_plan(iv[i].plan);
            s.arrived = iv[i].arrived;
            s.served_light = iv[i].served_light;
            s.served_heavy = iv[i].served_heavy;
            s.dropped = iv[i].dropped;
            s.late = iv[i].late;
            s.threshold = iv[i].threshold;
            if (iv[i].has_mean_delivered_quality) s.mean_delivered_quality = iv[i].mean_delivered_quality;
        }
        std::vector<QueryRecord> rs(static_cast<size_t>(nq));
        for (int64_t i = 0; i < nq; ++i) {
            const ds_query_record& q = qr[i];
            QueryRecord& r = rs[static_cast<size_t>(i)];
            r.id = q.id;
            r.arrival = q.arrival;
            r.deadline = q.deadline;
            r.confidence = q.confidence;
            r.quality_light = q.quality_light;
            r.quality_heavy = q.quality_heavy;
            if (q.present & DS_REC_LIGHT_START) r.light_start = q.light_start;
            if (q.present & DS_REC_LIGHT_END) r.light_end = q.light_end;
            if (q.present & DS_REC_HEAVY_START) r.heavy_start = q.heavy_start;
            if (q.present & DS_REC_HEAVY_END) r.heavy_end = q.heavy_end;
            if (q.present & DS_REC_COMPLETION) r.completion = q.completion;
            if (q.present & DS_REC_OUTCOME) r.outcome = static_cast<Outcome>(q.outcome);
            if (q.present & DS_REC_DELIVERED_QUALITY) r.delivered_quality = q.delivered_quality;
        }
        std::vector<PlanLogEntry> ps(static_cast<size_t>(np));
        for (int64_t i = 0; i < np; ++i) {
            ps[static_cast<size_t>(i)].tick = pl[i].tick;
            ps[static_cast<size_t>(i)].time = pl[i].time;
            ps[static_cast<size_t>(i)].demand_estimated = pl[i].demand_estimated;
            ps[static_cast<size_t>(i)].plan = to_plan(pl[i].plan);
        }
        write_csv(dir, ivs, rs, ps);
        return 0;
    } catch (...) {
        return map_exception();
    }
}

uint64_t dsref_splitmix64(uint64_t x) { return splitmix64(x); }
uint64_t dsref_hash_name(const char* s) { return hash_name(s); }
void dsref_stream_raw(uint64_t seed, const char* name, int k, uint64_t* out) {
    RandomStream rs(seed, name);
    for (int i = 0; i < k; ++i) out[i] = rs.next_u64();
}

} // extern "C"
