// TEST INFRASTRUCTURE ONLY -- golden-vector generator, never the product.
//
// Compiles the reference's acceptance binary source in place
// (/root/reference/proj/tests/acceptance_main.cpp, via -I, not copied; its
// main() is renamed) and exposes its instance generators and the brute-force
// reference_max_threshold (acceptance_main.cpp:46-144) through extern "C":
//   * C1: 200 instances seeded mt19937_64(20260825) (acceptance_main.cpp:146-173)
//   * C2: the solve-speed problem recipe, seeded mt19937_64(7)
//         (acceptance_main.cpp:175-190), generalised to any cascade and S --
//         the SURVEY 8(d) config-4 planner batch.
#define main reference_acceptance_main
#include "acceptance_main.cpp"
#undef main
#include "ds_gpu.h"

extern "C" void dsref_from_cascade(const void* c, ds_cascade* out);
extern "C" void dsref_from_problem(const void* p, ds_problem* out);

extern "C" int dsref_gen_accept_c1(uint64_t seed, int n, ds_cascade* cascades,
                                   ds_problem* problems, double* grids, int32_t* glen,
                                   double* want_t, int32_t* want_has, ds_plan* want_solve) {
    std::mt19937_64 rng(seed);
    for (int i = 0; i < n; ++i) {
        CascadeProfile c = random_cascade(rng);
        AllocationProblem p = random_problem(rng, c);
        dsref_from_cascade(&c, &cascades[i]);
        dsref_from_problem(&p, &problems[i]);
        problems[i].cascade = i;
        problems[i].grid = i;
        glen[i] = static_cast<int32_t>(p.threshold_grid.size());
        for (size_t k = 0; k < p.threshold_grid.size(); ++k) grids[i * 101 + k] = p.threshold_grid[k];
        std::optional<double> want = reference_max_threshold(p);
        want_has[i] = want.has_value() ? 1 : 0;
        want_t[i] = want.value_or(-1.0);
        AllocationPlan got = solve(p);
        want_solve[i].x1 = got.x1; want_solve[i].x2 = got.x2;
        want_solve[i].b1 = got.b1; want_solve[i].b2 = got.b2;
        want_solve[i].threshold = got.threshold;
        want_solve[i].feasible = got.feasible ? 1 : 0;
    }
    return 0;
}

// acceptance_main.cpp:177-190 for an arbitrary cascade and server count:
// D = 1.2*u*S*T1(max b1); light queue {floor(20u), D+0.1}; heavy queue
// {floor(8u), 0.3D+0.1}; lambda 1.05 (AllocationProblem default); grid is the
// caller's (problems[i].grid = 0).
extern "C" int dsref_gen_c2_recipe(const ds_cascade* dc, int servers, uint64_t seed, int n,
                                   ds_problem* problems) {
    CascadeProfile c;
    c.name = "c2";
    for (int i = 0; i < dc->light.n; ++i) c.light.latency_table[dc->light.batch[i]] = dc->light.latency[i];
    for (int i = 0; i < dc->heavy.n; ++i) c.heavy.latency_table[dc->heavy.batch[i]] = dc->heavy.latency[i];
    c.slo_seconds = dc->slo_seconds;
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> u(0.0, 1.0);
    double light_capacity = servers * throughput(c.light, c.light.max_batch());
    for (int i = 0; i < n; ++i) {
        AllocationProblem p;
        p.cascade = &c;
        p.total_servers = servers;
        p.demand_qps = 1.2 * u(rng) * light_capacity;
        p.light_queue = {static_cast<long long>(20.0 * u(rng)), p.demand_qps + 0.1};
        p.heavy_queue = {static_cast<long long>(8.0 * u(rng)), 0.3 * p.demand_qps + 0.1};
        dsref_from_problem(&p, &problems[i]);
        problems[i].cascade = 0;
        problems[i].grid = 0;
    }
    return 0;
}
