// Reference-side drop-in for the DiffServe simulator (the binding a maintainer
// of /root/reference/proj would add).
//
// ds_b200::GpuPlannerPolicy is a diffserve::Policy (policies.hpp:30-60) whose
// plan() runs on the B200 planner (K1 plan_sweep) through the C ABI
// (include/ds_gpu.h), for every policy kind make_policy() knows
// (policies.cpp:63-219): the control logic around the solver (frozen Clipper
// plans, Proteus fix-ups, AIMD state) mirrors policies.cpp; only the solves
// move to the GPU. score_queries() replaces run_experiment's per-query
// sample_query loop (experiment.cpp:76-79) with one K4 launch.
//
// Header-only; compiles against the reference headers and links libds_b200.so.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "diffserve/allocator.hpp"
#include "diffserve/errors.hpp"
#include "diffserve/metrics.hpp"
#include "diffserve/policies.hpp"
#include "diffserve/profiles.hpp"
#include "diffserve/workload.hpp"
#include "ds_gpu.h"

namespace ds_b200 {

// Status -> the exception type the reference throws for the same condition.
inline void throw_status(ds_status s) {
    if (s == DS_OK) return;
    const std::string msg = ds_last_error();
    switch (s) {
    case DS_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case DS_ERR_DOMAIN: throw std::domain_error(msg);
    case DS_ERR_INVARIANT: throw diffserve::InvariantError(msg);
    case DS_ERR_OUT_OF_RANGE: throw std::out_of_range(msg);
    default: throw std::runtime_error("ds_b200: " + msg);
    }
}

inline void to_pod(const diffserve::ModelProfile& m, ds_model_profile& out) {
    std::memset(&out, 0, sizeof(out));
    if (m.latency_table.size() > DS_MAX_BATCHES)
        throw std::length_error("ds_b200: more than DS_MAX_BATCHES profiled batch sizes");
    int i = 0;
    for (const auto& [b, e] : m.latency_table) {
        out.batch[i] = b;
        out.latency[i] = e;
        ++i;
    }
    out.n = i;
}

inline ds_cascade to_pod(const diffserve::CascadeProfile& c) {
    ds_cascade out;
    std::memset(&out, 0, sizeof(out));
    to_pod(c.light, out.light);
    to_pod(c.heavy, out.heavy);
    for (int i = 0; i < DS_CURVE_BINS && i < static_cast<int>(c.deferral.bin_mass.size()); ++i)
        out.deferral.bin_mass[i] = c.deferral.bin_mass[i];
    out.deferral.total_mass = c.deferral.total_mass;
    out.slo_seconds = c.slo_seconds;
    return out;
}

// One planner call (n = 1) of `mode` on the GPU.
inline diffserve::AllocationPlan gpu_plan(ds_ctx* ctx, const diffserve::AllocationProblem& p,
                                          int mode, double fixed_t = 0.0, int fb1 = 0,
                                          int fb2 = 0) {
    if (!p.cascade) throw std::invalid_argument("allocation problem has no cascade");
    ds_cascade c = to_pod(*p.cascade);
    ds_problem q;
    std::memset(&q, 0, sizeof(q));
    q.demand_qps = p.demand_qps;
    q.overprovision_lambda = p.overprovision_lambda;
    q.queue_sentinel_seconds = p.queue_sentinel_seconds;
    q.light_rate = p.light_queue.arrival_rate;
    q.heavy_rate = p.heavy_queue.arrival_rate;
    q.light_len = p.light_queue.queue_length;
    q.heavy_len = p.heavy_queue.queue_length;
    q.fixed_threshold = fixed_t;
    q.fixed_b1 = fb1;
    q.fixed_b2 = fb2;
    q.total_servers = p.total_servers;
    q.queuing = p.queuing == diffserve::QueuingModel::twice_exec ? DS_QUEUING_TWICE_EXEC
                                                                 : DS_QUEUING_LITTLES_LAW;
    q.mode = mode;
    const int32_t offs[2] = {0, static_cast<int32_t>(p.threshold_grid.size())};
    ds_plan out;
    std::memset(&out, 0, sizeof(out));
    throw_status(ds_plan_batch(ctx, &q, 1, &c, 1, p.threshold_grid.data(), offs, 1, &out));
    return diffserve::AllocationPlan{out.x1, out.x2, out.b1, out.b2, out.threshold,
                                     out.feasible != 0};
}

class GpuPlannerPolicy : public diffserve::Policy {
public:
    GpuPlannerPolicy(ds_ctx* ctx, const diffserve::PolicyParams& params)
        : ctx_(ctx), p_(params) {}

    diffserve::PolicyKind kind() const override { return p_.kind; }

    diffserve::ModelKind entry_stage(const diffserve::AllocationPlan& plan,
                                     diffserve::RandomStream& rng) override {
        using diffserve::ModelKind;
        using diffserve::PolicyKind;
        switch (p_.kind) {
        case PolicyKind::clipper_light: return ModelKind::light;          // policies.cpp:92-94
        case PolicyKind::clipper_heavy: return ModelKind::heavy;
        case PolicyKind::proteus_like:                                    // policies.cpp:123-128
            if (plan.x1 > 0 && plan.x2 > 0)
                return rng.bernoulli(0.5) ? ModelKind::heavy : ModelKind::light;
            return plan.x2 > 0 ? ModelKind::heavy : ModelKind::light;
        default: return ModelKind::light;
        }
    }

    bool defers(double confidence, double threshold) const override {
        return discriminator() ? confidence < threshold : false;          // policies.cpp:37-39
    }
    bool uses_discriminator() const override { return discriminator(); }

    diffserve::AllocationPlan plan(const diffserve::AllocationProblem& p) override {
        using diffserve::PolicyKind;
        switch (p_.kind) {
        case PolicyKind::diffserve: return gpu_plan(ctx_, p, DS_SOLVE);
        case PolicyKind::diffserve_static: {                              // allocator.cpp:171-174
            diffserve::AllocationProblem q = p;
            q.demand_qps = p_.peak_demand_qps;
            return gpu_plan(ctx_, q, DS_SOLVE);
        }
        case PolicyKind::clipper_light:
        case PolicyKind::clipper_heavy: {                                 // policies.cpp:98-110
            if (!solved_) {
                const bool light = p_.kind == PolicyKind::clipper_light;
                diffserve::AllocationProblem q = p;
                q.demand_qps = p_.peak_demand_qps;
                frozen_ = gpu_plan(ctx_, q, light ? DS_SOLVE_SINGLE_LIGHT : DS_SOLVE_SINGLE_HEAVY);
                if (light) frozen_.b2 = p.cascade->heavy.min_batch();
                else frozen_.b1 = p.cascade->light.min_batch();
                solved_ = true;
            }
            return frozen_;
        }
        case PolicyKind::proteus_like: {                                  // policies.cpp:132-137
            diffserve::AllocationPlan out = gpu_plan(ctx_, p, DS_SOLVE_EVEN_SPLIT);
            if (out.b1 == 0) out.b1 = p.cascade->light.min_batch();
            if (out.b2 == 0) out.b2 = p.cascade->heavy.min_batch();
            return out;
        }
        case PolicyKind::abl_static_threshold:                            // policies.cpp:145-147
            return gpu_plan(ctx_, p, DS_SOLVE_PINNED, p_.fixed_threshold);
        case PolicyKind::abl_aimd_batching:                               // policies.cpp:157-164
            cascade_ = p.cascade;
            if (b1_ == 0) {
                b1_ = p.cascade->light.min_batch();
                b2_ = p.cascade->heavy.min_batch();
            }
            return gpu_plan(ctx_, p, DS_SOLVE_FIXED_BATCHES, 0.0, b1_, b2_);
        case PolicyKind::abl_no_queuing_model: {                          // policies.cpp:188-192
            diffserve::AllocationProblem q = p;
            q.queuing = diffserve::QueuingModel::twice_exec;
            return gpu_plan(ctx_, q, DS_SOLVE);
        }
        }
        throw std::invalid_argument("unhandled policy kind");
    }

    void observe_batch(diffserve::ModelKind model, bool slo_timeout) override {
        if (p_.kind != diffserve::PolicyKind::abl_aimd_batching || !cascade_ || b1_ == 0) return;
        if (model == diffserve::ModelKind::light)                         // policies.cpp:166-172
            b1_ = diffserve::aimd_update(cascade_->light, b1_, slo_timeout, p_.aimd_add_step,
                                         p_.aimd_mult_factor);
        else
            b2_ = diffserve::aimd_update(cascade_->heavy, b2_, slo_timeout, p_.aimd_add_step,
                                         p_.aimd_mult_factor);
    }

    int live_batch(diffserve::ModelKind model) const override {
        if (p_.kind != diffserve::PolicyKind::abl_aimd_batching) return 0;
        return model == diffserve::ModelKind::light ? b1_ : b2_;
    }

private:
    bool discriminator() const {
        return p_.kind != diffserve::PolicyKind::clipper_light &&
               p_.kind != diffserve::PolicyKind::clipper_heavy &&
               p_.kind != diffserve::PolicyKind::proteus_like;
    }

    ds_ctx* ctx_;
    diffserve::PolicyParams p_;
    bool solved_ = false;
    diffserve::AllocationPlan frozen_;
    const diffserve::CascadeProfile* cascade_ = nullptr;
    int b1_ = 0, b2_ = 0;
};

// generate_arrivals (workload.cpp:82-106) on the GPU (K8), bit-identical.
inline std::vector<double> generate_arrivals(ds_ctx* ctx, const diffserve::Trace& trace,
                                             uint64_t seed, diffserve::ArrivalMode mode) {
    const int32_t m = mode == diffserve::ArrivalMode::uniform ? DS_ARRIVALS_UNIFORM
                                                              : DS_ARRIVALS_POISSON;
    const int32_t nr = static_cast<int32_t>(trace.rates.size());
    int64_t n = 0;
    throw_status(ds_generate_arrivals(ctx, trace.rates.data(), nr, trace.interval_seconds, seed,
                                      m, nullptr, 0, &n));
    std::vector<double> out(static_cast<size_t>(n));
    throw_status(ds_generate_arrivals(ctx, trace.rates.data(), nr, trace.interval_seconds, seed,
                                      m, out.data(), n, &n));
    return out;
}

// run_experiment's query construction (experiment.cpp:70-79): one K4 launch
// writes the Query records instead of a sample_query call per query.
inline std::vector<diffserve::Query> score_queries(ds_ctx* ctx,
                                                   const diffserve::QueryOutcomeModel& m,
                                                   const std::vector<double>& arrivals,
                                                   double slo_seconds) {
    static_assert(sizeof(diffserve::Query) == sizeof(ds_query), "Query layout");
    static_assert(offsetof(diffserve::Query, arrival) == offsetof(ds_query, arrival), "layout");
    static_assert(offsetof(diffserve::Query, deadline) == offsetof(ds_query, deadline), "");
    static_assert(offsetof(diffserve::Query, quality_light) == offsetof(ds_query, quality_light),
                  "");
    static_assert(offsetof(diffserve::Query, quality_heavy) == offsetof(ds_query, quality_heavy),
                  "");
    static_assert(offsetof(diffserve::Query, confidence) == offsetof(ds_query, confidence), "");
    ds_query_model qm{m.easy_fraction, m.quality_gap_scale, m.confidence_fidelity,
                      m.noise_sigma, m.seed};
    const int64_t n = static_cast<int64_t>(arrivals.size());
    std::vector<diffserve::Query> out(static_cast<size_t>(n));
    throw_status(ds_sample_queries(ctx, &qm, 0, arrivals.data(), n, slo_seconds,
                                   reinterpret_cast<ds_query*>(out.data())));
    return out;
}

inline ds_plan to_plan_pod(const diffserve::AllocationPlan& p) {
    ds_plan out{};
    out.x1 = p.x1;
    out.x2 = p.x2;
    out.b1 = p.b1;
    out.b2 = p.b2;
    out.threshold = p.threshold;
    out.feasible = p.feasible ? 1 : 0;
    return out;
}

// write_csv (metrics.cpp:91-127) with the rows formatted on the GPU (K9);
// byte-identical files.
inline void write_csv(ds_ctx* ctx, const std::string& out_dir,
                      const std::vector<diffserve::IntervalSnapshot>& intervals,
                      const std::vector<diffserve::QueryRecord>& records,
                      const std::vector<diffserve::PlanLogEntry>& plans) {
    std::vector<ds_interval_snapshot> iv(intervals.size());
    for (size_t i = 0; i < intervals.size(); ++i) {
        const auto& s = intervals[i];
        ds_interval_snapshot& o = iv[i];
        o = ds_interval_snapshot{};
        o.interval_start = s.interval_start;
        o.demand_observed = s.demand_observed;
        o.demand_estimated = s.demand_estimated;
        o.plan = to_plan_pod(s.plan);
        o.arrived = s.arrived;
        o.served_light = s.served_light;
        o.served_heavy = s.served_heavy;
        o.dropped = s.dropped;
        o.late = s.late;
        o.threshold = s.threshold;
        o.has_mean_delivered_quality = s.mean_delivered_quality.has_value();
        o.mean_delivered_quality = s.mean_delivered_quality.value_or(0.0);
    }
    std::vector<ds_query_record> qr(records.size());
    for (size_t i = 0; i < records.size(); ++i) {
        const auto& r = records[i];
        ds_query_record& o = qr[i];
        o = ds_query_record{};
        o.id = r.id;
        o.arrival = r.arrival;
        o.deadline = r.deadline;
        o.confidence = r.confidence;
        o.quality_light = r.quality_light;
        o.quality_heavy = r.quality_heavy;
        auto opt = [&o](const std::optional<double>& v, double* dst, uint32_t bit) {
            if (v) {
                *dst = *v;
                o.present |= bit;
            }
        };
        opt(r.light_start, &o.light_start, DS_REC_LIGHT_START);
        opt(r.light_end, &o.light_end, DS_REC_LIGHT_END);
        opt(r.heavy_start, &o.heavy_start, DS_REC_HEAVY_START);
        opt(r.heavy_end, &o.heavy_end, DS_REC_HEAVY_END);
        opt(r.completion, &o.completion, DS_REC_COMPLETION);
        opt(r.delivered_quality, &o.delivered_quality, DS_REC_DELIVERED_QUALITY);
        if (r.outcome) {
            o.outcome = static_cast<int32_t>(*r.outcome);
            o.present |= DS_REC_OUTCOME;
        }
    }
    std::vector<ds_plan_log_entry> pl(plans.size());
    for (size_t i = 0; i < plans.size(); ++i) {
        pl[i] = ds_plan_log_entry{};
        pl[i].tick = plans[i].tick;
        pl[i].time = plans[i].time;
        pl[i].demand_estimated = plans[i].demand_estimated;
        pl[i].plan = to_plan_pod(plans[i].plan);
    }
    std::filesystem::create_directories(out_dir);
    auto emit = [&](const char* name, auto fn, const auto& rows) {
        int64_t bytes = 0;
        const int64_t n = static_cast<int64_t>(rows.size());
        throw_status(fn(ctx, rows.data(), n, nullptr, 0, &bytes));
        std::string buf(static_cast<size_t>(bytes), '\0');
        throw_status(fn(ctx, rows.data(), n, buf.data(), bytes, &bytes));
        const std::string path = out_dir + "/" + name;
        std::ofstream out(path, std::ios::binary);
        if (!out) throw std::runtime_error("cannot write " + path);
        out.write(buf.data(), static_cast<std::streamsize>(buf.size()));
    };
    emit("intervals.csv", ds_format_intervals_csv, iv);
    emit("queries.csv", ds_format_queries_csv, qr);
    emit("plans.csv", ds_format_plans_csv, pl);
}

} // namespace ds_b200
