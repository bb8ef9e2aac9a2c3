// The reference simulator run end to end with the B200 hot path plugged in
// (SURVEY.md 8(f) rows 1, 3, 4): run_experiment (experiment.cpp:60-159)
// restated with (a) the arrival timestamps generated on the GPU (K8) instead
// of generate_arrivals, (b) one K4 launch writing every Query record instead
// of the sample_query loop, (c) ds_b200::GpuPlannerPolicy as the Policy and
// (d) the three CSV files formatted on the GPU (K9) instead of write_csv;
// everything else -- config, trace, the DES (Simulation) -- the reference's
// own code. --mode cpu runs the stock reference run_experiment for comparison.
//
//   des_gpu --config cfg --out dir [--mode gpu|cpu] [--policy name] [--seed s]
//
// Built by `make -C oracle des` (needs /root/reference and libds_b200.so).
#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <string>

#include "diffserve/cluster.hpp"
#include "diffserve/config.hpp"
#include "diffserve/experiment.hpp"
#include "diffserve/metrics.hpp"
#include "diffserve/policies.hpp"
#include "gpu_planner_policy.hpp"

using namespace diffserve;

int main(int argc, char** argv) {
    std::string config, out_dir, mode = "gpu", policy_name;
    long long seed = -1;
    for (int i = 1; i + 1 < argc; i += 2) {
        const std::string k = argv[i], v = argv[i + 1];
        if (k == "--config") config = v;
        else if (k == "--out") out_dir = v;
        else if (k == "--mode") mode = v;
        else if (k == "--policy") policy_name = v;
        else if (k == "--seed") seed = std::stoll(v);
        else {
            std::fprintf(stderr, "unknown argument %s\n", k.c_str());
            return 2;
        }
    }
    if (config.empty() || out_dir.empty()) {
        std::fprintf(stderr, "usage: des_gpu --config cfg --out dir [--mode gpu|cpu]\n");
        return 2;
    }
    try {
        ExperimentConfig cfg = load_config(config);
        cfg.out_dir = out_dir;
        if (!policy_name.empty()) cfg.policy = policy_name;
        if (seed >= 0) cfg.seed = static_cast<uint64_t>(seed);
        if (mode == "cpu") {
            ExperimentResult res = run_experiment(cfg, true);
            std::printf("%s\n", res.summary_line.c_str());
            return 0;
        }
        validate_config(cfg);
        CascadeProfile cascade = load_cascade(cfg.profiles_path, cfg.cascade);
        Trace trace = load_trace(cfg.trace_path);
        if (cfg.trace_scale_min) trace = scale_trace(trace, *cfg.trace_scale_min, *cfg.trace_scale_max);
        ds_ctx* ctx = nullptr;
        ds_b200::throw_status(ds_ctx_create(0, &ctx));
        const std::vector<double> arrivals = ds_b200::generate_arrivals(
            ctx, trace, cfg.seed, parse_arrival_mode(cfg.arrival_mode));
        QueryOutcomeModel qmodel;
        qmodel.easy_fraction = cfg.easy_fraction;
        qmodel.quality_gap_scale = cfg.quality_gap_scale;
        qmodel.confidence_fidelity = cfg.confidence_fidelity;
        qmodel.noise_sigma = cfg.noise_sigma;
        qmodel.seed = cfg.seed;

        std::vector<Query> queries =
            ds_b200::score_queries(ctx, qmodel, arrivals, cascade.slo_seconds);

        PolicyParams pp;
        pp.kind = parse_policy_kind(cfg.policy);
        pp.peak_demand_qps = trace.peak();
        pp.fixed_threshold = cfg.fixed_threshold;
        pp.aimd_add_step = cfg.aimd_add_step;
        pp.aimd_mult_factor = cfg.aimd_mult_factor;
        ds_b200::GpuPlannerPolicy policy(ctx, pp);

        ClusterConfig cc;
        cc.servers = cfg.servers;
        cc.control_interval_seconds = cfg.control_interval_seconds;
        cc.ewma_alpha = cfg.ewma_alpha;
        cc.overprovision_lambda = cfg.overprovision_lambda;
        cc.threshold_grid_step = cfg.threshold_grid_step;
        cc.deferral_decay = cfg.deferral_decay;
        cc.queue_sentinel_seconds = cfg.queue_sentinel_seconds;
        cc.bill_formed_batch = cfg.bill_formed_batch;
        cc.switch_delay_seconds = cfg.switch_delay_seconds;
        cc.seed = cfg.seed;

        Simulation sim(cascade, trace, std::move(queries), policy, cc);
        const auto t0 = std::chrono::steady_clock::now();
        RunOutput out = sim.run();
        const auto t1 = std::chrono::steady_clock::now();
        ds_b200::write_csv(ctx, cfg.out_dir, out.intervals, out.records, out.plans);
        uint64_t arrived = 0, light = 0, heavy = 0, dropped = 0, late = 0;
        for (const QueryRecord& r : out.records) {
            ++arrived;
            if (r.outcome == Outcome::served_light) ++light;
            else if (r.outcome == Outcome::served_heavy) ++heavy;
            else if (r.outcome == Outcome::dropped) ++dropped;
            else if (r.outcome == Outcome::late) ++late;
        }
        double solve_us = 0.0;
        for (double us : out.solve_micros) solve_us += us;
        if (!out.solve_micros.empty()) solve_us /= static_cast<double>(out.solve_micros.size());
        std::printf("policy=%s mode=gpu arrived=%llu served_light=%llu served_heavy=%llu "
                    "dropped=%llu late=%llu forced_light=%llu ticks=%zu solve_mean_us=%s "
                    "wall_s=%s gpu_launches=%lld\n",
                    cfg.policy.c_str(), (unsigned long long)arrived, (unsigned long long)light,
                    (unsigned long long)heavy, (unsigned long long)dropped,
                    (unsigned long long)late, (unsigned long long)out.forced_light,
                    out.plans.size(), fmt6(solve_us).c_str(),
                    fmt6(std::chrono::duration<double>(t1 - t0).count()).c_str(),
                    (long long)ds_ctx_launch_count(ctx));
        ds_ctx_destroy(ctx);
        return 0;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "des_gpu: %s\n", e.what());
        return 1;
    }
}
