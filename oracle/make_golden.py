"""TEST INFRASTRUCTURE ONLY -- regenerates tests/golden/*.npz from the reference.

Every expected value in the fixtures comes from the UNMODIFIED reference built
by oracle/Makefile (oracle/_ref/libdsref.so): its own instance generators
(test_allocator.cpp:99-166, acceptance_main.cpp:46-113,175-190), its own
solver / exhaustive oracles, sample_query, observe_confidence and the
Policy::defers loop. Run here (where /root/reference exists):

    make -C oracle ref && python oracle/make_golden.py

The fixtures are small and committed; the GPU box reads only them.
"""
from __future__ import annotations

import ctypes
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)

from oracle import lib  # noqa: E402
from paper_2411_15381_b200 import abi, workloads  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")
P = abi.ptr


def _check(rc, what):
    if rc != 0:
        raise RuntimeError(f"{what}: status {rc}: {lib.ref().dsref_last_error()}")


def ref_plan(problems, cascades, gvals, goffs, threads=8):
    r = lib.ref()
    out = np.zeros(len(problems), abi.PLAN)
    _check(r.dsref_plan_batch(P(problems), len(problems), P(cascades), len(cascades), P(gvals),
                              P(goffs), len(goffs) - 1, P(out), threads), "plan_batch")
    return out


def grids_from_fixed(grids, glen):
    offs = np.zeros(len(glen) + 1, np.int32)
    offs[1:] = np.cumsum(glen)
    vals = np.concatenate([grids[i, :glen[i]] for i in range(len(glen))])
    return vals, offs


def gen_alloc_random():
    """test_allocator.cpp:266-276: 60 instances, mt19937_64(2024)."""
    n = 60
    cas = np.zeros(n, abi.CASCADE)
    pro = np.zeros(n, abi.PROBLEM)
    grids = np.zeros((n, 101), np.float64)
    glen = np.zeros(n, np.int32)
    want_o = np.zeros(n, abi.PLAN)
    want_s = np.zeros(n, abi.PLAN)
    _check(lib.ref().dsref_gen_alloc_random(2024, n, P(cas), P(pro), P(grids), P(glen),
                                            P(want_o), P(want_s)), "gen_alloc_random")
    vals, offs = grids_from_fixed(grids, glen)
    np.savez_compressed(os.path.join(OUT, "alloc_random_2024.npz"), cascades=cas, problems=pro,
                        grid_values=vals, grid_offsets=offs, want_oracle=want_o, want_solve=want_s)
    return int(want_s["feasible"].sum())


def gen_accept_c1():
    """acceptance_main.cpp:146-173: 200 instances, mt19937_64(20260825)."""
    n = 200
    cas = np.zeros(n, abi.CASCADE)
    pro = np.zeros(n, abi.PROBLEM)
    grids = np.zeros((n, 101), np.float64)
    glen = np.zeros(n, np.int32)
    want_t = np.zeros(n, np.float64)
    want_has = np.zeros(n, np.int32)
    want_s = np.zeros(n, abi.PLAN)
    _check(lib.ref().dsref_gen_accept_c1(20260825, n, P(cas), P(pro), P(grids), P(glen),
                                         P(want_t), P(want_has), P(want_s)), "gen_accept_c1")
    vals, offs = grids_from_fixed(grids, glen)
    np.savez_compressed(os.path.join(OUT, "accept_c1.npz"), cascades=cas, problems=pro,
                        grid_values=vals, grid_offsets=offs, want_max_t=want_t,
                        want_has=want_has, want_solve=want_s)
    return int(want_has.sum())


def sampled_curve(name="cascade1", n=5000):
    """from_samples of the n sample_query confidences (cascade cfg, seed 1)."""
    r = lib.ref()
    m = workloads.query_model()
    conf = np.zeros(n, np.float64)
    _check(r.dsref_sample_queries(P(m), 0, n, workloads.SHIPPED[name]["slo"], P(conf), None, 8),
           "sample")
    curve = np.zeros((), abi.CURVE)
    _check(r.dsref_curve_from_samples(P(conf), n, P(curve)), "from_samples")
    return curve


def gen_config4(per_combo=256):
    """fitted 32x32 tables, C2 recipe seed 7, S in 16..128."""
    r = lib.ref()
    cas = np.zeros(3, abi.CASCADE)
    for i, name in enumerate(["cascade1", "cascade2", "cascade3"]):
        light, heavy, slo = workloads.fitted_tables(name)
        cas[i] = workloads.make_cascade(light, heavy, slo, sampled_curve(name))
    grid = workloads.make_grid(0.01)
    probs = []
    for ci in range(3):
        for s in (16, 32, 64, 128):
            p = np.zeros(per_combo, abi.PROBLEM)
            one = cas[ci:ci + 1].copy()  # keep alive across the call
            _check(r.dsref_gen_c2_recipe(P(one), s, 7, per_combo, P(p)),
                   "c2 recipe")
            p["cascade"] = ci
            probs.append(p)
    pro = np.concatenate(probs)
    offs = np.array([0, len(grid)], np.int32)
    want = ref_plan(pro, cas, grid, offs)
    np.savez_compressed(os.path.join(OUT, "config4.npz"), cascades=cas, problems=pro,
                        grid_values=grid, grid_offsets=offs, want_solve=want)
    return int(want["feasible"].sum()), len(pro)


def gen_config4_bench(total=4096):
    """BASELINE.md's planner batch: P = 4,096 problems of the acceptance-C2
    recipe (mt19937_64(7), acceptance_main.cpp:177-190) over the 3 fitted 32x32
    cascades x S in {16, 32, 64, 128} (12 combos: 342 or 341 problems each),
    the cascades' curves = from_samples of 5K sample_query confidences (cfg,
    seed 1), grid k/100; want_solve = the reference's solve on each. The
    batch bench.py times (GPU and the reference CPU arm) -- identical inputs."""
    r = lib.ref()
    cas = np.zeros(3, abi.CASCADE)
    for i, name in enumerate(["cascade1", "cascade2", "cascade3"]):
        light, heavy, slo = workloads.fitted_tables(name)
        cas[i] = workloads.make_cascade(light, heavy, slo, sampled_curve(name))
    grid = workloads.make_grid(0.01)
    combos = [(ci, s) for ci in range(3) for s in (16, 32, 64, 128)]
    probs = []
    for j, (ci, s) in enumerate(combos):
        n = total // len(combos) + (1 if j < total % len(combos) else 0)
        p = np.zeros(n, abi.PROBLEM)
        one = cas[ci:ci + 1].copy()
        _check(r.dsref_gen_c2_recipe(P(one), s, 7, n, P(p)), "c2 recipe")
        p["cascade"] = ci
        probs.append(p)
    pro = np.concatenate(probs)
    assert len(pro) == total
    offs = np.array([0, len(grid)], np.int32)
    want = ref_plan(pro, cas, grid, offs)
    np.savez_compressed(os.path.join(OUT, "config4_bench.npz"), cascades=cas, problems=pro,
                        grid_values=grid, grid_offsets=offs, want_solve=want)
    return int(want["feasible"].sum()), len(pro)


def random_table(rng, base, max_sizes, contiguous):
    n = int(rng.integers(1, max_sizes + 1))
    t = {}
    e = base
    if contiguous:
        for b in range(1, n + 1):
            t[b] = e
            # e(b+1) in [e(b), e(b)*(b+1)/b]: non-decreasing latency,
            # non-increasing per-query latency (profiles.cpp:27-48)
            e *= float(rng.uniform(1.0, (b + 1) / b))
    else:
        b = 1
        for _ in range(n):
            t[b] = e
            b *= 2
            e *= float(rng.uniform(1.0, 2.0))
    return t


def gen_wide(n=3000, seed=99):
    """Analogue of SURVEY probe A.3: S in [1, 128], up to 6 (doubling) or 32
    (contiguous) batch sizes, uniform/empty/sampled curves, random queues, 20%
    twice_exec, both grid flavours, and every solve variant. Inputs come from a
    numpy stream; expected plans from the reference solver."""
    rng = np.random.default_rng(seed)
    r = lib.ref()
    cas = np.zeros(n, abi.CASCADE)
    pro = np.zeros(n, abi.PROBLEM)
    grids = [workloads.full_grid(0.01), workloads.full_grid(0.1), workloads.make_grid(0.01),
             workloads.make_grid(0.05)]
    for i in range(n):
        contiguous = rng.random() < 0.25
        light = random_table(rng, float(rng.uniform(0.05, 0.5)), 32 if contiguous else 6,
                             contiguous)
        heavy = random_table(rng, light[1] * float(rng.uniform(2.0, 12.0)),
                             32 if contiguous else 4, contiguous)
        slo = (light[1] + heavy[1]) * float(rng.uniform(1.01, 4.0))
        kind = int(rng.integers(0, 4))
        if kind == 0:
            curve = workloads.uniform_prior()
        elif kind == 1:
            curve = workloads.empty_curve()
        else:
            s = rng.random(int(rng.integers(1, 400)))
            if rng.random() < 0.3:
                s = np.round(s * 100) / 100  # grid-aligned samples exercise bin_of's nudge
            curve = np.zeros((), abi.CURVE)
            _check(r.dsref_curve_from_samples(P(s), len(s), P(curve)), "from_samples")
            if rng.random() < 0.5:
                more = rng.random(int(rng.integers(1, 200)))
                _check(r.dsref_curve_observe(P(curve), P(more), len(more), 0.999), "observe")
        cas[i] = workloads.make_cascade(light, heavy, slo, curve)
        p = pro[i]
        S = int(rng.integers(1, 129))
        p["total_servers"] = S
        tmax = max(b / e for b, e in light.items())
        p["demand_qps"] = float(rng.random()) * 1.5 * S * tmax
        if rng.random() < 0.02:
            p["demand_qps"] = 0.0
        p["overprovision_lambda"] = [1.0, 1.05, 1.1, 1.5][int(rng.integers(0, 4))]
        p["queue_sentinel_seconds"] = 1e6
        for side in ("light", "heavy"):
            q = int(rng.integers(0, 4))
            if q == 1:
                p[f"{side}_len"] = int(rng.integers(1, 11))
            elif q == 2:
                p[f"{side}_len"] = int(rng.integers(1, 11))
                p[f"{side}_rate"] = 1.0 + float(rng.random()) * 30.0
            elif q == 3:
                p[f"{side}_len"] = int(rng.integers(500, 1000))
                p[f"{side}_rate"] = 1.0 + float(rng.random()) * 5.0
        p["queuing"] = abi.QUEUING_TWICE_EXEC if rng.random() < 0.2 else abi.QUEUING_LITTLES_LAW
        p["cascade"] = i
        p["grid"] = int(rng.integers(0, len(grids)))
        mode = int(rng.choice([0, 0, 0, 0, 1, 2, 3, 4, 5]))
        p["mode"] = mode
        if mode == abi.SOLVE_PINNED:
            p["fixed_threshold"] = float(rng.choice([0.0, 1.0, round(float(rng.random()), 2),
                                                     float(rng.random())]))
        if mode == abi.SOLVE_FIXED_BATCHES:
            p["fixed_b1"] = int(rng.choice(list(light.keys())))
            p["fixed_b2"] = int(rng.choice(list(heavy.keys())))
    gvals = np.concatenate(grids)
    offs = np.zeros(len(grids) + 1, np.int32)
    offs[1:] = np.cumsum([len(g) for g in grids])
    want = ref_plan(pro, cas, gvals, offs)
    np.savez_compressed(os.path.join(OUT, "wide_random.npz"), cascades=cas, problems=pro,
                        grid_values=gvals, grid_offsets=offs, want=want)
    return int(want["feasible"].sum()), n


def gen_latent():
    """sample_query streams, routing and curve replay (workload.cpp:108-129,
    cluster.cpp:290-306, profiles.cpp:108-120)."""
    r = lib.ref()
    out = {}
    models = [workloads.query_model(),                               # cascade cfg, seed 1
              workloads.query_model(confidence_fidelity=1.5, noise_sigma=0.15, seed=9),
              workloads.query_model(easy_fraction=1.0, noise_sigma=0.0, seed=5),
              workloads.query_model(confidence_fidelity=0.0, noise_sigma=0.0, seed=0),
              workloads.query_model(seed=0xFFFFFFFFFFFFFFFF)]
    rng = np.random.default_rng(5)
    for k, m in enumerate(models):
        ids = np.arange(5000, dtype=np.uint64) if k == 0 else np.sort(
            rng.choice(1_000_000, 2000, replace=False)).astype(np.uint64)
        conf = np.zeros(len(ids), np.float64)
        ql = np.zeros(len(ids), np.float64)
        if k == 0:
            _check(r.dsref_sample_queries(P(m), 0, len(ids), 5.0, P(conf), P(ql), 8), "sample")
        else:
            c1 = np.zeros(1, np.float64)
            q1 = np.zeros(1, np.float64)
            for j, i in enumerate(ids):
                _check(r.dsref_sample_queries(P(m), int(i), 1, 5.0, P(c1), P(q1), 1), "sample")
                conf[j], ql[j] = c1[0], q1[0]
        out[f"model{k}"] = m
        out[f"ids{k}"] = ids
        out[f"conf{k}"] = conf
        out[f"ql{k}"] = ql
    # Route + observe over the 5K cascade-1 confidences, every grid threshold,
    # starting from the shipped prior (cascades.profiles:20) at decay 0.999.
    conf = out["conf0"]
    grid = workloads.make_grid(0.01)
    prior = np.zeros((), abi.CURVE)
    samples = np.asarray(workloads.SHIPPED_PRIOR_SAMPLES, np.float64)
    _check(r.dsref_curve_from_samples(P(samples), len(samples), P(prior)), "prior")
    counts = np.zeros(len(grid), np.int64)
    digests = np.zeros(len(grid), np.uint64)
    curve_after = None
    for k, t in enumerate(grid):
        curve = prior.copy()
        idx = np.zeros(len(conf), np.int64)
        cnt = np.zeros(1, np.int64)
        _check(r.dsref_route_loop(P(conf), len(conf), float(t), 1, 0.999, P(curve), P(idx),
                                  P(cnt)), "route_loop")
        counts[k] = cnt[0]
        digests[k] = np.uint64(int(np.bitwise_xor.reduce(
            (idx[:cnt[0]].astype(np.uint64) * np.uint64(0x9E3779B97F4A7C15)) ^
            np.arange(cnt[0], dtype=np.uint64)) if cnt[0] else 0))
        curve_after = curve
    out.update(route_grid=grid, route_counts=counts, route_digest=digests, prior=prior,
               curve_after_0999=curve_after)
    for decay in (1.0, 0.5):
        c = prior.copy()
        _check(r.dsref_curve_observe(P(c), P(conf), len(conf), decay), "observe")
        out[f"curve_after_{str(decay).replace('.', '')}"] = c
    raw = np.zeros((4, 8), np.uint64)
    for k, s in enumerate([0, 1, 0x9E3779B97F4A7C15, 123456789]):
        # the engine seed RandomStream(s, "query") uses; first 8 outputs
        g = np.zeros(8, np.uint64)
        lib.ref().dsref_stream_raw(s, b"query", 8, P(g))
        raw[k] = g
    out["raw_seeds"] = np.array([0, 1, 0x9E3779B97F4A7C15, 123456789], np.uint64)
    out["raw_first8"] = raw
    np.savez_compressed(os.path.join(OUT, "latent.npz"), **out)


def gen_des():
    """Inputs + reference CSV digests for the drop-in DES run.
    The digests come from the stock reference run_experiment (des_gpu --mode
    cpu) on inputs re-written by oracle/des_inputs.py; they must equal the
    digests of the reference's own files."""
    import hashlib
    import subprocess
    import tempfile
    from oracle import des_inputs
    ref = "/root/reference/proj"
    g = {}
    for name, d in workloads.SHIPPED.items():
        g[f"{name}_light"] = np.array(sorted(d["light"].items()), np.float64)
        g[f"{name}_heavy"] = np.array(sorted(d["heavy"].items()), np.float64)
        g[f"{name}_slo"] = np.float64(d["slo"])
    g["prior"] = np.asarray(workloads.SHIPPED_PRIOR_SAMPLES, np.float64)
    for t in ("trace_4to32qps", "trace_1to8qps", "trace_8to24qps"):
        with open(f"{ref}/traces/{t}.txt") as f:
            g[t] = np.array([float(x) for x in f.read().split()], np.float64)
    exe = os.path.join(HERE, "_ref", "des_gpu")
    with tempfile.TemporaryDirectory() as tmp:
        cfgs = des_inputs.write_inputs(tmp, g)
        for name, cfg in cfgs.items():
            out = os.path.join(tmp, "out_" + name)
            subprocess.run([exe, "--config", cfg, "--out", out, "--mode", "cpu"], cwd=tmp,
                           check=True, capture_output=True)
            outr = os.path.join(tmp, "outref_" + name)
            subprocess.run([exe, "--config", f"configs/{name}.cfg", "--out", outr, "--mode", "cpu"],
                           cwd=ref, check=True, capture_output=True)
            for csv in ("intervals", "plans", "queries"):
                a = hashlib.md5(open(os.path.join(out, csv + ".csv"), "rb").read()).hexdigest()
                b = hashlib.md5(open(os.path.join(outr, csv + ".csv"), "rb").read()).hexdigest()
                assert a == b, (name, csv, "rewritten inputs change the reference's output")
                g[f"md5_{name}_{csv}"] = np.array(a)
    np.savez_compressed(os.path.join(OUT, "des_inputs.npz"), **g)


def arrival_cases():
    """(name, rates, interval_seconds, seed, mode) for generate_arrivals goldens:
    the reference's own unit/acceptance traces (test_workload.cpp:71-103,
    acceptance_main.cpp:326-336), the shipped traces at the configs' seed, and
    synthetic traces that stress zero-rate gaps, tiny rates, many interval
    boundaries and ~1M arrivals."""
    ref = "/root/reference/proj"
    cases = [
        ("unit_uniform_2", [2.0], 1.0, 0, 1),
        ("unit_uniform_13", [1.0, 3.0], 1.0, 0, 1),
        ("unit_zero", [0.0, 0.0], 1.0, 0, 1),
        ("unit_poisson_42", [10.0] * 600, 1.0, 42, 0),
        ("unit_poisson_43", [10.0] * 600, 1.0, 43, 0),
    ]
    for t, seed in (("trace_4to32qps", 1), ("trace_1to8qps", 1), ("trace_8to24qps", 1),
                    ("trace_4to32qps", 7)):
        with open(f"{ref}/traces/{t}.txt") as f:
            rates = [float(x) for x in f.read().split()]
        cases.append((f"{t}_s{seed}", rates, 1.0, seed, 0))
        cases.append((f"{t}_s{seed}_uniform", rates, 1.0, seed, 1))
    light = workloads.SHIPPED["cascade1"]["light"]
    rate = 0.7 * 2 * (4 / light[4])                 # acceptance_main.cpp:329
    cases.append(("accept_wait", [rate] * 3600, 1.0, 11, 0))
    mixed = [0.0, 0.0, 5.0, 0.001, 0.0, 17.5, 300.0, 0.0, 1e-6, 42.0, 0.0]
    cases.append(("mixed_poisson", mixed, 0.37, 7, 0))
    cases.append(("mixed_uniform", mixed, 0.37, 7, 1))
    rng = np.random.default_rng(9)
    # rates on a 1/64 qps lattice (exact in binary, compresses well)
    cases.append(("boundaries", list(rng.integers(0, 400 * 64, 30000) / 64.0), 0.01, 9, 0))
    cases.append(("boundaries_uniform", list(rng.integers(0, 400 * 64, 8000) / 64.0), 0.013, 9,
                  1))
    cases.append(("dense_1m", [2500.0] * 400, 1.0, 3, 0))
    cases.append(("dense_1m_uniform", [4999.5] * 200, 1.0, 3, 1))
    return cases


def gen_arrivals(full_limit=6000):
    """generate_arrivals goldens from the reference (workload.cpp:82-106):
    count, sha256 of the timestamp bytes, and the timestamps themselves for
    small cases (head/tail/strided samples for large ones). Also the Query
    records of the cascade-1 and cascade-3 runs (experiment.cpp:76-79)."""
    import hashlib
    r = lib.ref()
    out = {}
    names = []
    for name, rates, dt, seed, mode in arrival_cases():
        rates = np.asarray(rates, np.float64)
        n = r.dsref_generate_arrivals(P(rates), len(rates), dt, seed, mode, None, 0)
        a = np.zeros(max(n, 1), np.float64)
        n2 = r.dsref_generate_arrivals(P(rates), len(rates), dt, seed, mode, P(a), len(a))
        assert n == n2 >= 0, name
        a = a[:n]
        names.append(name)
        out[f"{name}__rates"] = rates
        out[f"{name}__meta"] = np.array([dt, seed, mode], np.float64)
        out[f"{name}__count"] = np.int64(n)
        out[f"{name}__sha256"] = np.array(hashlib.sha256(a.tobytes()).hexdigest())
        if n <= full_limit:
            out[f"{name}__arrivals"] = a
        else:
            idx = np.unique(np.concatenate([np.arange(512), np.arange(n - 512, n),
                                            np.linspace(0, n - 1, 1024).astype(np.int64)]))
            out[f"{name}__sample_idx"] = idx
            out[f"{name}__sample"] = a[idx]
    out["names"] = np.array(names)
    for cname, tname in (("cascade3", "trace_1to8qps_s1"),):
        m = np.zeros((), abi.QUERY_MODEL)
        m["easy_fraction"], m["quality_gap_scale"] = 0.3, 1.0
        m["confidence_fidelity"], m["noise_sigma"], m["seed"] = 0.35, 0.12, 1
        slo = workloads.SHIPPED[cname]["slo"]
        a = out.get(f"{tname}__arrivals")
        q = np.zeros(len(a), abi.QUERY)
        _check(r.dsref_sample_query_records(P(m.reshape(1)), 0, P(a), len(a), slo, P(q)),
               "sample_query_records")
        out[f"records_{cname}"] = q
        out[f"records_{cname}_slo"] = np.float64(slo)
    np.savez_compressed(os.path.join(OUT, "arrivals.npz"), **out)
    return {n: int(out[f"{n}__count"]) for n in names}


def gen_csv():
    """write_csv goldens (metrics.cpp:91-127): random QueryRecord /
    IntervalSnapshot / PlanLogEntry rows (with the "%.6g" stress values of
    tests/helpers.special_doubles) and the bytes the reference's own
    write_csv produced for them."""
    import tempfile
    from tests import helpers
    rng = np.random.default_rng(6)
    q = helpers.random_query_records(rng, 3000)
    iv = helpers.random_intervals(rng, 300)
    pl = helpers.random_plan_log(rng, 200)
    out = {"records": q, "intervals": iv, "plans": pl}
    with tempfile.TemporaryDirectory() as tmp:
        _check(lib.ref().dsref_write_csv(tmp.encode(), P(iv), len(iv), P(q), len(q), P(pl),
                                         len(pl)), "write_csv")
        for name in ("queries", "intervals", "plans"):
            with open(os.path.join(tmp, name + ".csv"), "rb") as f:
                out[f"{name}_csv"] = np.frombuffer(f.read(), np.uint8)
    vals = np.concatenate([helpers.special_doubles(), helpers.random_doubles(rng, 6000)])
    g6 = np.zeros(len(vals), "S16")
    lib.port().dso_fmt6(P(vals), len(vals), P(g6))
    out["g6_values"], out["g6_text"] = vals, g6
    np.savez_compressed(os.path.join(OUT, "csv.npz"), **out)
    return {k: len(v) for k, v in out.items()}


def main():
    os.makedirs(OUT, exist_ok=True)
    print("alloc_random_2024: feasible", gen_alloc_random(), "of 60")
    print("accept_c1: feasible", gen_accept_c1(), "of 200")
    print("config4: feasible/total", gen_config4())
    print("config4_bench: feasible/total", gen_config4_bench())
    print("wide_random: feasible/total", gen_wide())
    gen_latent()
    print("latent: ok")
    gen_des()
    print("des: ok")
    print("arrivals:", gen_arrivals())
    print("csv:", gen_csv())


if __name__ == "__main__":
    if len(sys.argv) > 1:
        for name in sys.argv[1:]:
            print(name, globals()[f"gen_{name}"]())
    else:
        main()
