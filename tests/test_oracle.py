"""CPU suite: pins the plain-C oracle restatement (oracle/ds_oracle.c) to the
reference, via the golden vectors the reference itself produced
(tests/golden/, oracle/make_golden.py) and, where the reference library was
built (oracle/_ref), directly against it on fresh inputs."""
import ctypes

import numpy as np
import pytest

from oracle import lib
from paper_2411_15381_b200 import abi, workloads
from tests.helpers import assert_plans_equal, planner_set, route_digest

P = abi.ptr


def port_plan(problems, cascades, gvals, goffs, threads=4):
    out = np.zeros(len(problems), abi.PLAN)
    status = np.zeros(len(problems), np.int32)
    lib.port().dso_plan_batch(P(problems), len(problems), P(cascades), P(gvals), P(goffs), P(out),
                              P(status), threads)
    return out, status


@pytest.mark.parametrize("name,key", [("alloc_random_2024", "want_oracle"),
                                      ("alloc_random_2024", "want_solve"),
                                      ("accept_c1", "want_solve"),
                                      ("config4", "want_solve"),
                                      ("config4_bench", "want_solve"),
                                      ("wide_random", "want")])
def test_port_planner_matches_reference_goldens(golden, name, key):
    g = golden(name)
    got, status = port_plan(*planner_set(g))
    assert not status.any()
    assert_plans_equal(got, g[key], name)


def test_accept_c1_thresholds_match_brute_force(golden):
    """acceptance C1 (acceptance_main.cpp:146-173): max feasible t exactly."""
    g = golden("accept_c1")
    got, _ = port_plan(*planner_set(g))
    has = g["want_has"].astype(bool)
    assert has.sum() == 50
    assert np.array_equal(got["feasible"].astype(bool), has)
    assert np.array_equal(got["threshold"][has], g["want_max_t"][has])


def test_port_latent_matches_reference_bits(golden):
    g = golden("latent")
    for k in range(5):
        m = np.ascontiguousarray(g[f"model{k}"])
        ids = g[f"ids{k}"]
        c1 = np.zeros(1)
        q1 = np.zeros(1)
        conf = np.zeros(len(ids))
        ql = np.zeros(len(ids))
        for j, i in enumerate(ids):
            lib.port().dso_sample_query(P(m), int(i), P(c1), P(q1))
            conf[j], ql[j] = c1[0], q1[0]
        assert np.array_equal(conf.view(np.uint64), g[f"conf{k}"].view(np.uint64)), k
        assert np.array_equal(ql.view(np.uint64), g[f"ql{k}"].view(np.uint64)), k


def test_port_mt19937_64_streams(golden):
    g = golden("latent")
    for s, want in zip(g["raw_seeds"], g["raw_first8"]):
        out = np.zeros(8, np.uint64)
        lib.port().dso_stream_raw(int(s), b"query", 8, P(out))
        assert np.array_equal(out, want)


def test_port_route_and_curve_match_reference(golden):
    g = golden("latent")
    conf = g["conf0"]
    grid = g["route_grid"]
    idx = np.zeros(len(grid) * len(conf), np.int64)
    counts = np.zeros(len(grid), np.int64)
    lib.port().dso_route(P(conf), len(conf), P(grid), len(grid), 0, P(idx), P(counts))
    assert np.array_equal(counts, g["route_counts"])
    for k in range(len(grid)):
        lst = idx[k * len(conf): k * len(conf) + counts[k]]
        assert route_digest(lst) == g["route_digest"][k]
    for key, decay in (("curve_after_0999", 0.999), ("curve_after_10", 1.0),
                       ("curve_after_05", 0.5)):
        c = g["prior"].copy()
        assert lib.port().dso_curve_observe(P(c), P(conf), len(conf), decay) == 0
        want = g[key]
        assert np.array_equal(c["bin_mass"].view(np.uint64), want["bin_mass"].view(np.uint64))
        assert c["total_mass"] == want["total_mass"]


def test_profiles_golden_known_answers():
    """test_profiles.cpp:68-92,128-132 known answers through the port."""
    port = lib.port()
    c = np.zeros((), abi.CURVE)
    for s in (0.2, 0.4, 0.6, 0.8):
        port.dso_observe(P(c), s, 1.0)
    f = np.zeros(1)

    def frac(t):
        assert port.dso_deferral_fraction(P(c), t, P(f)) == 0
        return f[0]

    assert frac(0.5) == pytest.approx(0.5)
    assert frac(0.0) == 0.0
    assert frac(1.0) == pytest.approx(1.0)
    assert frac(0.2) == pytest.approx(0.0)
    assert frac(0.21) == pytest.approx(0.25)
    assert port.dso_deferral_fraction(P(c), -0.1, P(f)) == abi.ERR_DOMAIN
    d = np.zeros((), abi.CURVE)
    for _ in range(4):
        port.dso_observe(P(d), 0.25, 1.0)
    port.dso_observe(P(d), 0.25, 0.5)
    assert d["total_mass"] == pytest.approx(3.0)
    assert port.dso_observe(P(d), 1.5, 1.0) == abi.ERR_DOMAIN
    prior = workloads.uniform_prior()
    for k in range(0, 101, 10):
        assert port.dso_deferral_fraction(P(prior), k / 100.0, P(f)) == 0
        assert f[0] == pytest.approx(k / 100.0)


needs_ref = pytest.mark.skipif(not lib.ref_available(), reason="oracle/_ref not built")


@needs_ref
def test_port_vs_reference_fresh_latent():
    rng = np.random.default_rng(1234)
    for _ in range(20):
        m = workloads.query_model(easy_fraction=float(rng.random()),
                                  quality_gap_scale=float(rng.uniform(0, 3)),
                                  confidence_fidelity=float(rng.uniform(0, 3)),
                                  noise_sigma=float(rng.uniform(0, 0.5)),
                                  seed=int(rng.integers(0, 2**63)))
        id0 = int(rng.integers(0, 2**62))
        n = 500
        a = np.zeros(n)
        qa = np.zeros(n)
        b = np.zeros(n)
        qb = np.zeros(n)
        assert lib.ref().dsref_sample_queries(P(m), id0, n, 5.0, P(a), P(qa), 1) == 0
        assert lib.port().dso_sample_queries(P(m), id0, n, P(b), P(qb), 1) == 0
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
        assert np.array_equal(qa.view(np.uint64), qb.view(np.uint64))


@needs_ref
def test_reference_unit_suites_pass_under_oracle_build():
    """The reference's own 89 doctest cases, built by oracle/Makefile against
    oracle/doctest_stub, pass (proj/test_output.txt:3-19)."""
    import os
    import subprocess
    exe = os.path.join(lib.HERE, "_ref", "ref_unit_tests")
    src = "/root/reference/proj"
    if not (os.path.exists(exe) and os.path.isdir(src)):
        pytest.skip("reference sources not present")
    r = subprocess.run([exe], cwd=src, capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "0 failed" in r.stdout


def test_disc_weight_restatement_matches_committed_export():
    """oracle/disc_oracle.gen_weights vs the GPU export committed in profiles/."""
    import os
    from oracle import disc_oracle
    path = os.path.join(os.path.dirname(lib.HERE), "profiles", "disc_weights_seed2024.npz")
    if not os.path.exists(path):
        pytest.skip("no committed export")
    c = dict(np.load(path))
    if "q1" not in c:
        pytest.skip("committed export predates the int8 layer 1")
    w = disc_oracle.gen_weights(2024, calibrate=False)
    for k in ("q1", "w2", "w3", "b1"):
        assert np.array_equal(w[k], c[k]), k
    assert np.float32(w["s1"]) == np.float32(c["s1"])


def test_synth_images_host_restatement_is_deterministic():
    from oracle import disc_oracle
    a = disc_oracle.synth_images(1, 0, 2, 32, 32)
    b = disc_oracle.synth_images(1, 0, 2, 32, 32)
    assert np.array_equal(a, b) and a.dtype == np.uint8 and a.shape == (2, 32, 32, 3)
    assert not np.array_equal(a[0], a[1])


def test_port_arrivals_match_reference_goldens(golden):
    """dso_generate_arrivals (the C restatement of workload.cpp:82-106)
    reproduces the reference's timestamps on every golden trace."""
    from tests.helpers import arrival_case, assert_arrivals_match
    g = golden("arrivals")
    for name in g["names"]:
        rates, dt, seed, mode = arrival_case(g, str(name))
        n = lib.port().dso_generate_arrivals(P(rates), len(rates), dt, seed, mode, None, 0)
        a = np.zeros(max(n, 1))
        assert lib.port().dso_generate_arrivals(P(rates), len(rates), dt, seed, mode, P(a),
                                                len(a)) == n
        assert_arrivals_match(g, str(name), a[:n])


def test_arrival_goldens_hold_reference_known_answers(golden):
    """test_workload.cpp:71-103 known answers, and the SURVEY A.1 arrival
    counts of the shipped configs (cascade1 11,559; cascade3 1,986)."""
    g = golden("arrivals")
    assert list(g["unit_uniform_2__arrivals"]) == [0.0, 0.5]
    np.testing.assert_allclose(g["unit_uniform_13__arrivals"], [0, 1, 1 + 1 / 3, 1 + 2 / 3])
    assert int(g["unit_zero__count"]) == 0
    a = g["unit_poisson_42__arrivals"]
    assert 5700 < len(a) < 6300 and np.all(np.diff(a) > 0) and a[0] >= 0 and a[-1] < 600
    assert int(g["trace_4to32qps_s1__count"]) == 11559
    assert int(g["trace_1to8qps_s1__count"]) == 1986


def test_log1p_restatement_matches_host_libm(tmp_path):
    """paper_2411_15381_b200/csrc/fdlibm_log1p.h (the device's log1p, used for
    every Exp(1) arrival draw) compiled for the host equals the host libm's
    log1p bit for bit on 2^24 inputs: the reference's own U in [0, 1) draws,
    tiny and near -1 arguments, and random doubles."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    src = tmp_path / "t.c"
    src.write_text(r'''
#include <math.h>
#include <stdio.h>
#include "fdlibm_log1p.h"
static uint64_t rs = 88172645463325252ull;
static uint64_t xr(void) { rs ^= rs << 13; rs ^= rs >> 7; rs ^= rs << 17; return rs; }
int main(void) {
    long bad = 0, n = 1L << 24;
    for (long i = 0; i < n; i++) {
        double x;
        switch (i & 3) {
        case 0: x = -(double)(xr() >> 11) * 0x1.0p-53; break;          /* -U */
        case 1: x = -ldexp((double)(xr() >> 11), -(int)(53 + xr() % 60)); break; /* tiny */
        case 2: x = -1.0 + ldexp((double)(xr() >> 11), -(int)(53 + xr() % 8)); break;
        default: x = ds_bitsd(xr()); if (isnan(x)) continue;
        }
        double a = log1p(x), b = ds_log1p(x);
        if (ds_dbits(a) != ds_dbits(b) && !(isnan(a) && isnan(b))) {
            if (bad < 5) printf("x=%a libm=%a restated=%a\n", x, a, b);
            bad++;
        }
    }
    printf("bad=%ld\n", bad);
    return bad != 0;
}
''')
    exe = tmp_path / "t"
    subprocess.run(["gcc", "-O2", "-ffp-contract=off",
                    f"-I{root}/paper_2411_15381_b200/csrc", str(src), "-o", str(exe), "-lm"],
                   check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout


def _compile_and_run(tmp_path, name, source, defines=()):
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    src = tmp_path / f"{name}.c"
    src.write_text(source)
    exe = tmp_path / name
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", *[f"-D{d}" for d in defines],
                    f"-I{root}/paper_2411_15381_b200/csrc", str(src), "-o", str(exe), "-lm"],
                   check=True)
    return subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)


FMT6_PROGRAM = r'''
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>
#include "fmt6.h"
static uint64_t rs = 88172645463325252ull;
static uint64_t xr(void) { rs ^= rs << 13; rs ^= rs >> 7; rs ^= rs << 17; return rs; }
static double pick(long i) {
    double x; uint64_t b;
    switch (i % 8) {
    case 0: b = xr(); memcpy(&x, &b, 8); return x;
    case 1: return ldexp((double)(xr() >> 11), -53) * pow(10.0, (double)(xr() % 16) - 8);
    case 2: return (double)(xr() % 100000000) / (double)ds_pow10_u64(xr() % 12);
    case 3: return (double)(xr() % 20000000);
    case 4: { double p = pow(10.0, (double)((int)(xr() % 40) - 20)); memcpy(&b, &p, 8);
              b += (int)(xr() % 7) - 3; memcpy(&x, &b, 8); return x; }
    case 5: return ldexp((double)(xr() >> 11), (int)(xr() % 2200) - 1127);
    case 6: return -((double)(xr() % 1000000) + 0.5) * pow(10.0, (double)((int)(xr() % 14) - 10));
    default: return (double)(xr() >> 11) * 0x1.0p-53 * 3600.0;
    }
}
int main(void) {
    long n = N, bad = 0;
    char a[64], b[64];
    for (long i = 0; i < n; i++) {
        double x = pick(i);
        snprintf(a, sizeof a, "%.6g", x);
        int k = ds_fmt_g6(x, b);
        b[k] = 0;
        if (strcmp(a, b)) { if (bad < 5) printf("%a: libc=%s restated=%s\n", x, a, b); bad++; }
    }
    for (long i = 0; i < n / 4; i++) {   /* the integer columns (operator<<) */
        uint64_t u = xr() >> (xr() % 64);
        if (i % 16 == 0) u = (i % 32 == 0) ? 0xffffffffffffffffull : (uint64_t)(i / 16);
        snprintf(a, sizeof a, "%llu", (unsigned long long)u);
        int k = ds_fmt_u64(u, b);
        b[k] = 0;
        if (strcmp(a, b)) { if (bad < 5) printf("u64 %s restated=%s\n", a, b); bad++; }
        int64_t s = (int64_t)u;
        if (i % 64 == 1) s = INT64_MIN;
        snprintf(a, sizeof a, "%lld", (long long)s);
        k = ds_fmt_i64(s, b);
        b[k] = 0;
        if (strcmp(a, b)) { if (bad < 5) printf("i64 %s restated=%s\n", a, b); bad++; }
    }
    printf("bad=%ld\n", bad);
    return bad != 0;
}
'''


@pytest.mark.parametrize("path", ["fast", "big"])
def test_fmt6_restatement_matches_host_printf(tmp_path, path):
    """paper_2411_15381_b200/csrc/fmt6.h (the device's "%.6g", metrics.cpp:67-71)
    compiled for the host equals the host snprintf byte for byte: 4M doubles
    through the 128-bit fast path, 1M with the 1280-bit path forced, and the
    integer columns (ds_fmt_u64 / ds_fmt_i64 against %llu / %lld)."""
    defines = ["N=4000000"] if path == "fast" else ["N=1000000", "DS_FMT_FORCE_BIG"]
    r = _compile_and_run(tmp_path, "fmt6", FMT6_PROGRAM, defines)
    assert r.returncode == 0, r.stdout


def test_port_csv_matches_reference_goldens(golden):
    """dso_format_*_csv (C restatement of write_csv, metrics.cpp:91-127) and
    dso_fmt6 reproduce the bytes the reference wrote."""
    g = golden("csv")
    port = lib.port()
    for name, key in (("queries", "records"), ("intervals", "intervals"), ("plans", "plans")):
        rows = np.ascontiguousarray(g[key])
        fn = getattr(port, f"dso_format_{name}_csv")
        n = fn(P(rows), len(rows), None, 0)
        out = np.zeros(n, np.uint8)
        assert fn(P(rows), len(rows), P(out), n) == n
        assert out.tobytes() == g[f"{name}_csv"].tobytes(), name
    vals = np.ascontiguousarray(g["g6_values"])
    txt = np.zeros(len(vals), "S16")
    port.dso_fmt6(P(vals), len(vals), P(txt))
    assert np.array_equal(txt, g["g6_text"])


@needs_ref
def test_port_csv_vs_reference_fresh(tmp_path):
    from tests import helpers
    rng = np.random.default_rng(77)
    q = helpers.random_query_records(rng, 20000)
    iv = helpers.random_intervals(rng, 500)
    pl = helpers.random_plan_log(rng, 500)
    assert lib.ref().dsref_write_csv(str(tmp_path).encode(), P(iv), len(iv), P(q), len(q), P(pl),
                                     len(pl)) == 0
    for name, rows in (("queries", q), ("intervals", iv), ("plans", pl)):
        fn = getattr(lib.port(), f"dso_format_{name}_csv")
        n = fn(P(rows), len(rows), None, 0)
        out = np.zeros(n, np.uint8)
        fn(P(rows), len(rows), P(out), n)
        assert out.tobytes() == (tmp_path / f"{name}.csv").read_bytes(), name


def test_disc_numpy_oracle_agrees_with_torch_reference():
    """Two independent CPU restatements of the discriminator (numpy oracle,
    PyTorch fp32) agree within the north_star tolerance on the host weights."""
    from oracle import disc_oracle
    from tests.torch_ref import disc_forward_torch
    w = disc_oracle.gen_weights(2024, calibrate=True)
    imgs = disc_oracle.synth_images(5, 0, 3, 256, 512)
    a = disc_oracle.disc_forward(imgs, w).astype(np.float64)
    b = disc_forward_torch(imgs, w)
    assert np.all(np.abs(a - b) <= 1e-3 * np.maximum(np.abs(a), 1e-2)), np.abs(a - b).max()


def test_disc_fast_cpu_port_equals_oracle():
    """The bench's CPU baseline (disc_forward_fast: centred fp32 layer 1,
    threads over images) computes the oracle's values: layer 1's integers are
    exact either way; layers 2-3 may differ only by fp32 summation order."""
    from oracle import disc_oracle
    w = disc_oracle.gen_weights(2024, calibrate=True)
    imgs = disc_oracle.synth_images(6, 0, 5, 256, 512)
    a = disc_oracle.disc_forward(imgs, w).astype(np.float64)
    b = disc_oracle.disc_forward_fast(imgs, w, threads=3).astype(np.float64)
    assert np.all(np.abs(a - b) <= 1e-6 * np.maximum(np.abs(a), 1e-2)), np.abs(a - b).max()
