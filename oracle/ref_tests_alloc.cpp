// TEST INFRASTRUCTURE ONLY -- golden-vector generator, never the product.
//
// Compiles the reference's own allocator unit suite in place
// (/root/reference/proj/tests/test_allocator.cpp, via -I, not copied) and
// exposes its instance generators and exhaustive oracle (random_cascade,
// random_problem, oracle_solve: test_allocator.cpp:33-166) through extern "C",
// so tests/golden/ can pin the reference's own random-equivalence case
// ("solve agrees with exhaustive enumeration", test_allocator.cpp:266-276).
#include "test_allocator.cpp"
#include "ds_gpu.h"

extern "C" void dsref_from_cascade(const void* c, ds_cascade* out);
extern "C" void dsref_from_problem(const void* p, ds_problem* out);

namespace {
ds_plan to_ds(const AllocationPlan& p) {
    ds_plan o{};
    o.x1 = p.x1; o.x2 = p.x2; o.b1 = p.b1; o.b2 = p.b2;
    o.threshold = p.threshold;
    o.feasible = p.feasible ? 1 : 0;
    return o;
}
} // namespace

// Replays test_allocator.cpp:266-276 with seed `seed` for n trials. Grid of
// trial i goes to grids[i*101 ..] with length glen[i]; want_oracle is
// oracle_solve's plan, want_solve is diffserve::solve's plan.
extern "C" int dsref_gen_alloc_random(uint64_t seed, int n, ds_cascade* cascades,
                                      ds_problem* problems, double* grids, int32_t* glen,
                                      ds_plan* want_oracle, ds_plan* want_solve) {
    std::mt19937_64 rng(seed);
    for (int i = 0; i < n; ++i) {
        CascadeProfile c = random_cascade(rng);
        AllocationProblem p = random_problem(c, rng);
        dsref_from_cascade(&c, &cascades[i]);
        dsref_from_problem(&p, &problems[i]);
        problems[i].cascade = i;
        problems[i].grid = i;
        glen[i] = static_cast<int32_t>(p.threshold_grid.size());
        for (size_t k = 0; k < p.threshold_grid.size(); ++k) grids[i * 101 + k] = p.threshold_grid[k];
        want_oracle[i] = to_ds(oracle_solve(p));
        want_solve[i] = to_ds(solve(p));
    }
    return 0;
}
