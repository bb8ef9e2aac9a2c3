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

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "diffserve/allocator.hpp"
#include "diffserve/errors.hpp"
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

// run_experiment's query construction (experiment.cpp:70-79) with one K4
// launch instead of a sample_query call per query.
inline std::vector<diffserve::Query> score_queries(ds_ctx* ctx,
                                                   const diffserve::QueryOutcomeModel& m,
                                                   const std::vector<double>& arrivals,
                                                   double slo_seconds) {
    if (!(slo_seconds > 0.0)) throw std::domain_error("slo_seconds must be positive");
    ds_query_model qm{m.easy_fraction, m.quality_gap_scale, m.confidence_fidelity,
                      m.noise_sigma, m.seed};
    const int64_t n = static_cast<int64_t>(arrivals.size());
    std::vector<double> conf(static_cast<size_t>(n)), ql(static_cast<size_t>(n));
    throw_status(ds_score_latent(ctx, &qm, 0, n, conf.data(), ql.data()));
    std::vector<diffserve::Query> out(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) {
        diffserve::Query& q = out[static_cast<size_t>(i)];
        q.id = static_cast<uint64_t>(i);
        q.arrival = arrivals[static_cast<size_t>(i)];
        q.deadline = q.arrival + slo_seconds;
        q.quality_light = ql[static_cast<size_t>(i)];
        q.quality_heavy = 1.0;
        q.confidence = conf[static_cast<size_t>(i)];
    }
    return out;
}

} // namespace ds_b200
