"""GPU parity: K1 plan_sweep vs the reference planner (exact plan equality).

Goldens come from the reference itself (tests/golden/, oracle/make_golden.py);
known-answer cases re-host proj/tests/test_allocator.cpp:172-457 through the
reference-shaped API (paper_2411_15381_b200/api.py)."""
import numpy as np
import pytest

from oracle import lib
from paper_2411_15381_b200 import abi, workloads
from paper_2411_15381_b200.api import (AllocationPlan, AllocationProblem, CascadeProfile,
                                       DeferralCurve, DomainError, InvalidArgument,
                                       InvariantError, ModelProfile, OutOfRange, QueueState,
                                       solve, solve_even_split, solve_fixed_batches,
                                       solve_pinned_threshold, solve_single_model,
                                       solve_static_peak)
from tests.helpers import assert_plans_equal, planner_set

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2411_15381_b200.api import default_context
    return default_context()


@pytest.mark.parametrize("name,key", [("alloc_random_2024", "want_oracle"),
                                      ("alloc_random_2024", "want_solve"),
                                      ("accept_c1", "want_solve"),
                                      ("config4", "want_solve"),
                                      ("config4_bench", "want_solve"),
                                      ("wide_random", "want")])
def test_planner_matches_reference_goldens(ctx, golden, name, key):
    g = golden(name)
    got = ctx.plan_batch(*planner_set(g))
    assert_plans_equal(got, g[key], name)


def test_accept_c1_max_threshold(ctx, golden):
    """acceptance C1 (acceptance_main.cpp:146-173)."""
    g = golden("accept_c1")
    got = ctx.plan_batch(*planner_set(g))
    has = g["want_has"].astype(bool)
    assert np.array_equal(got["feasible"].astype(bool), has)
    assert np.array_equal(got["threshold"][has], g["want_max_t"][has])


def test_planner_matches_port_on_fresh_instances(ctx):
    """Fresh random config-4 style batches vs the C restatement (and the
    reference itself when oracle/_ref exists)."""
    port = lib.port()
    rng = np.random.default_rng(77)
    cas = np.zeros(3, abi.CASCADE)
    for i, name in enumerate(["cascade1", "cascade2", "cascade3"]):
        light, heavy, slo = workloads.fitted_tables(name)
        samples = rng.random(int(rng.integers(10, 2000)))
        curve = np.zeros((), abi.CURVE)
        port.dso_curve_observe(abi.ptr(curve), abi.ptr(samples), len(samples), 0.999)
        cas[i] = workloads.make_cascade(light, heavy, slo, curve)
    probs = []
    for ci in range(3):
        for s in (16, 48, 128):
            p = workloads.c2_problems(cas[ci], s, 200, seed=int(rng.integers(1 << 30)))
            p["cascade"] = ci
            probs.append(p)
    pro = np.concatenate(probs)
    grid = workloads.make_grid(0.01)
    offs = np.array([0, len(grid)], np.int32)
    got = ctx.plan_batch(pro, cas, grid, offs)
    want = np.zeros(len(pro), abi.PLAN)
    st = np.zeros(len(pro), np.int32)
    port.dso_plan_batch(abi.ptr(pro), len(pro), abi.ptr(cas), abi.ptr(grid), abi.ptr(offs),
                        abi.ptr(want), abi.ptr(st), 8)
    assert not st.any()
    assert_plans_equal(got, want, "fresh")
    if lib.ref_available():
        ref = np.zeros(len(pro), abi.PLAN)
        assert lib.ref().dsref_plan_batch(abi.ptr(pro), len(pro), abi.ptr(cas), len(cas),
                                          abi.ptr(grid), abi.ptr(offs), 1, abi.ptr(ref), 8) == 0
        assert_plans_equal(got, ref, "fresh-vs-reference")


def test_planner_server_counts_at_integer_quotients(ctx):
    """Demands whose heavy-side server count need / T2 lands ON or one ulp
    beside an integer for most thresholds (uniform prior: f(k/100) = k/100;
    T2 in {4, 3, 2.5, 10/3, ...}; lambda * D = 400 -> need ~ 4k): every
    x2 entry of these problems takes min_servers' exact-division fallback or
    sits at its edge (plan_sweep.cu min_servers_r). Plans equal the C
    restatement's (and the reference's when oracle/_ref exists). Mixed batch
    counts (32 and 7 heavy sizes) cover both x2 table layouts."""
    port = lib.port()
    heavy32 = {b: b / 4.0 for b in range(1, 33)}                       # T2 = 4
    heavy32.update({b: b / 3.0 for b in range(2, 33, 3)})              # T2 = 3
    heavy32.update({b: b / 2.5 for b in range(3, 33, 5)})              # T2 = 2.5
    heavy7 = {1: 0.3, 2: 0.6, 3: 0.9, 5: 1.25, 8: 2.4, 12: 3.0, 20: 6.0}   # T2 = 10/3, 4, ...
    light = {b: b / 40.0 for b in (1, 2, 4, 8, 16, 32)}                # T1 = 40
    # extreme profiles: T2 near 1e308 makes 1/T2 subnormal (the fast path's
    # accuracy bound does not hold there: it must take the exact division)
    heavy_x = {1: 1e-308, 2: 3e-308, 4: 5e-300, 8: 1e-3}
    cas = np.zeros(3, abi.CASCADE)
    cas[0] = workloads.make_cascade(light, heavy32, 1e3)
    cas[1] = workloads.make_cascade(light, heavy7, 1e3)
    cas[2] = workloads.make_cascade(light, heavy_x, 1e3)
    probs = []
    for ci in range(3):
        for s in (3, 8, 16, 64, 128, 1000):
            for d in (100.0, 300.0, 400.0, 1000.0, 1234.5, 4000.0, 12.0):
                for lam in (1.0, 1.05):
                    p = np.zeros(1, abi.PROBLEM)
                    p["demand_qps"] = d
                    p["overprovision_lambda"] = lam
                    p["queue_sentinel_seconds"] = 1e6
                    p["total_servers"] = s
                    p["cascade"] = ci
                    p["mode"] = abi.SOLVE
                    probs.append(p)
    pro = np.concatenate(probs)
    grid = workloads.make_grid(0.01)
    offs = np.array([0, len(grid)], np.int32)
    got = ctx.plan_batch(pro, cas, grid, offs)
    want = np.zeros(len(pro), abi.PLAN)
    st = np.zeros(len(pro), np.int32)
    port.dso_plan_batch(abi.ptr(pro), len(pro), abi.ptr(cas), abi.ptr(grid), abi.ptr(offs),
                        abi.ptr(want), abi.ptr(st), 8)
    assert not st.any()
    assert want["feasible"].any() and not want["feasible"].all()
    assert_plans_equal(got, want, "integer-quotients")
    if lib.ref_available():
        ref = np.zeros(len(pro), abi.PLAN)
        assert lib.ref().dsref_plan_batch(abi.ptr(pro), len(pro), abi.ptr(cas), len(cas),
                                          abi.ptr(grid), abi.ptr(offs), 1, abi.ptr(ref), 8) == 0
        assert_plans_equal(got, ref, "integer-quotients-vs-reference")


# ---- test_allocator.cpp known answers, through the reference-shaped API ---------

def toy_cascade(slo=100.0):      # helpers.hpp:53-61
    return CascadeProfile("toy", ModelProfile("toy-light", {1: 0.1}),
                          ModelProfile("toy-heavy", {1: 1.0}), DeferralCurve.uniform_prior(), slo)


def batched_cascade(slo=5.0):    # helpers.hpp:64-72
    return CascadeProfile("batched",
                          ModelProfile("b-light", {1: 0.10, 2: 0.13, 4: 0.18, 8: 0.30, 16: 0.52}),
                          ModelProfile("b-heavy", {1: 1.78, 2: 1.90}),
                          DeferralCurve.uniform_prior(), slo)


def make_problem(c, demand, servers, grid=None):
    return AllocationProblem(demand, servers, c, threshold_grid=list(
        workloads.full_grid() if grid is None else grid))


def test_solve_maximizes_threshold_subject_to_capacity():        # :227-241
    p = make_problem(toy_cascade(), 10.0, 4)
    p.overprovision_lambda = 1.0
    plan = solve(p)
    assert plan.feasible
    assert plan.threshold == pytest.approx(0.30)
    assert (plan.x1, plan.x2, plan.b1, plan.b2) == (1, 3, 1, 1)


def test_zero_demand_threshold_one_largest_batches():            # :243-253
    plan = solve(make_problem(batched_cascade(), 0.0, 8))
    assert plan.feasible and plan.threshold == 1.0
    assert (plan.x1, plan.x2, plan.b1, plan.b2) == (1, 0, 16, 2)


def test_overload_returns_all_light_best_effort():                # :255-264
    plan = solve(make_problem(batched_cascade(), 100000.0, 4))
    assert not plan.feasible
    assert (plan.threshold, plan.x1, plan.x2, plan.b1) == (0.0, 4, 0, 16)


def test_threshold_falls_monotonically_with_demand():             # :278-287
    prev = 2.0
    for k in range(1, 21):
        t = solve(make_problem(batched_cascade(), k * 12.0, 16)).threshold
        assert t <= prev
        prev = t


def test_acceptance_c3_threshold_vs_demand():
    """acceptance C3 (acceptance_main.cpp:200-219; test_output.txt:23):
    t falls 1.00 -> 0.26 over 6..120 qps on cascade 1, never rising."""
    lt, ht, slo = (workloads.SHIPPED["cascade1"][k] for k in ("light", "heavy", "slo"))
    c = CascadeProfile("cascade1", ModelProfile("l", lt), ModelProfile("h", ht),
                       DeferralCurve.from_samples(workloads.SHIPPED_PRIOR_SAMPLES), slo)
    ts = [solve(make_problem(c, 6.0 * k, 16)).threshold for k in range(1, 21)]
    assert ts[0] == 1.0 and round(ts[-1], 2) == 0.26
    assert all(b <= a for a, b in zip(ts, ts[1:]))


def test_lower_deferral_curve_admits_higher_threshold():          # :289-300
    low = batched_cascade()
    low.deferral = DeferralCurve.from_samples([0.8, 0.9])
    high = batched_cascade()
    high.deferral = DeferralCurve.from_samples([0.1, 0.2])
    for d in (20.0, 60.0, 120.0):
        assert solve(make_problem(low, d, 16)).threshold >= solve(make_problem(high, d, 16)).threshold


def test_validation_mirrors_reference_exceptions():               # :318-339
    c = toy_cascade()
    p = make_problem(c, 10.0, 4)
    with pytest.raises(InvalidArgument):
        solve(AllocationProblem(10.0, 4, None, threshold_grid=[0.0, 1.0]))
    with pytest.raises(DomainError):
        solve(make_problem(c, 10.0, 0))
    with pytest.raises(InvariantError):
        solve(make_problem(c, 10.0, 4, grid=[0.5, 1.0]))
    with pytest.raises(InvariantError):
        solve(make_problem(c, 10.0, 4, grid=[0.0, 0.5, 0.5]))
    with pytest.raises(DomainError):
        solve(make_problem(c, -1.0, 4))
    q = make_problem(c, 10.0, 4)
    q.light_queue = QueueState(-1, 5.0)
    with pytest.raises(DomainError):
        solve(q)
    assert solve(p).feasible


def test_static_peak_equals_solve_at_peak():                      # :341-347
    c = batched_cascade()
    assert solve_static_peak(make_problem(c, 4.0, 16), 32.0) == solve(make_problem(c, 32.0, 16))


def test_pinned_threshold_variants():                             # :349-374
    c = toy_cascade()
    p = make_problem(c, 10.0, 4)
    p.overprovision_lambda = 1.0
    opt = solve(p)
    assert solve_pinned_threshold(p, opt.threshold) == opt
    q = make_problem(c, 30.0, 4)
    q.overprovision_lambda = 1.0
    plan = solve_pinned_threshold(q, 1.0)
    assert not plan.feasible and plan.x1 >= 1 and plan.x1 + plan.x2 <= 4
    assert plan.threshold == 1.0
    zero = solve_pinned_threshold(q, 0.0)
    assert zero.x2 == 0 and zero.feasible
    with pytest.raises(DomainError):
        solve_pinned_threshold(q, 1.5)


def test_fixed_batches_variants():                                # :376-394
    c = batched_cascade()
    p = make_problem(c, 50.0, 16)
    free = solve(p)
    assert solve_fixed_batches(p, free.b1, free.b2) == free
    tiny = solve_fixed_batches(p, 1, 1)
    assert (tiny.b1, tiny.b2) == (1, 1) and tiny.threshold <= free.threshold
    over = solve_fixed_batches(make_problem(c, 10000.0, 4), 1, 1)
    assert not over.feasible and over.x2 == 0
    with pytest.raises(OutOfRange):
        solve_fixed_batches(p, 3, 1)


def test_single_model_variants():                                 # :396-432
    light = ModelProfile("l", {1: 0.10, 2: 0.13, 4: 0.18, 8: 0.30, 16: 0.52})
    plan = solve_single_model(light, True, 16, 200.0, 1.05, 5.0)
    assert plan.feasible and (plan.x1, plan.x2, plan.b1) == (16, 0, 2)
    assert solve_single_model(light, True, 16, 100.0, 1.05, 5.0).b1 == 1
    over = solve_single_model(light, True, 16, 50000.0, 1.05, 5.0)
    assert not over.feasible and over.b1 == 16
    tight = solve_single_model(light, True, 16, 50000.0, 1.05, 0.5)
    assert not tight.feasible and tight.b1 == 4
    hopeless = solve_single_model(light, True, 16, 10.0, 1.05, 0.15)
    assert not hopeless.feasible and hopeless.b1 == 1
    heavy = ModelProfile("h", {1: 1.78, 2: 1.90})
    hv = solve_single_model(heavy, False, 16, 8.0, 1.05, 5.0)
    assert hv.feasible and (hv.x1, hv.x2, hv.b1, hv.b2) == (0, 16, 0, 1)


def test_even_split_variants():                                   # :434-457
    c = toy_cascade()
    heavy_only = solve_even_split(make_problem(c, 3.0, 4))
    assert heavy_only.feasible and (heavy_only.x1, heavy_only.x2) == (0, 4)
    p = make_problem(c, 4.5, 4)
    p.overprovision_lambda = 1.0
    split = solve_even_split(p)
    assert split.feasible and (split.x1, split.x2) == (1, 3)
    q = make_problem(c, 10.0, 4)
    q.overprovision_lambda = 1.0
    lo = solve_even_split(q)
    assert lo.feasible and (lo.x1, lo.x2) == (4, 0)


def test_empty_and_large_batches(ctx, golden):
    g = golden("config4")
    pro, cas, gv, go = planner_set(g)
    assert len(ctx.plan_batch(pro[:0], cas, gv, go)) == 0
    big = np.tile(pro, 6)          # 18432 problems in one launch
    got = ctx.plan_batch(big, cas, gv, go)
    assert_plans_equal(got, np.tile(g["want_solve"], 6), "tiled")


@pytest.mark.parametrize("name,key,shards", [("config4", "want_solve", 4),
                                             ("wide_random", "want", 3),
                                             ("alloc_random_2024", "want_solve", 2),
                                             ("accept_c1", "want_solve", 8)])
def test_t_sharded_keys_min_then_decode_equals_reference(ctx, golden, name, key, shards):
    """ds_plan_keys over disjoint threshold slices (one per GPU in the sharded
    planner), element-wise MIN (the all-reduce), ds_plan_from_keys -> exactly
    the reference's plans; every slice's keys equal the C restatement's."""
    from paper_2411_15381_b200 import dist as ddist
    g = golden(name)
    pro, cas, gv, go = planner_set(g)
    G = int(max(go[1:] - go[:-1]))
    port = lib.port()
    red = np.full(len(pro), ddist.KEY_NONE, np.uint64)
    for r in range(shards):
        lo, hi = ddist.shard_range(G, shards, r)
        k = ctx.plan_keys(pro, cas, gv, go, lo, hi)
        want_k = np.zeros(len(pro), np.uint64)
        port.dso_plan_keys(abi.ptr(pro), len(pro), abi.ptr(cas), abi.ptr(gv), abi.ptr(go),
                           lo, hi, abi.ptr(want_k))
        assert np.array_equal(k, want_k), (name, r)
        red = np.minimum(red, k)
    assert np.array_equal(red, ctx.plan_keys(pro, cas, gv, go, 0, G))
    assert_plans_equal(ctx.plan_from_keys(pro, cas, gv, go, red), g[key], name)
