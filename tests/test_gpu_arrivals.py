"""GPU parity: K8 generate_arrivals and K4 Query records.

Timestamps must be bit-identical to the reference's (tests/golden/arrivals.npz,
from the reference's own generate_arrivals via oracle/make_golden.py) and to
the C restatement (oracle/ds_oracle.c, itself pinned to those goldens) on
fresh traces."""
import ctypes
import os

import numpy as np
import pytest

from oracle import lib
from paper_2411_15381_b200 import abi, native
from paper_2411_15381_b200.api import (POISSON, UNIFORM, CapacityError, DomainError,
                                       InvalidArgument, QueryOutcomeModel, Trace,
                                       default_context, generate_arrivals,
                                       sample_query_records)
from tests.helpers import arrival_case, assert_arrivals_match

pytestmark = pytest.mark.gpu

P = abi.ptr
# Query.confidence / quality_light go through CUDA's log/cos (<= 2 ulp), the


@pytest.fixture(scope="module")
def ctx():
    return default_context()


def port_arrivals(rates, dt, seed, mode):
    rates = np.ascontiguousarray(rates, np.float64)
    n = lib.port().dso_generate_arrivals(P(rates), len(rates), dt, seed, mode, None, 0)
    a = np.zeros(max(n, 1))
    lib.port().dso_generate_arrivals(P(rates), len(rates), dt, seed, mode, P(a), len(a))
    return a[:n]


def test_arrivals_match_reference_goldens(ctx, golden):
    g = golden("arrivals")
    for name in g["names"]:
        rates, dt, seed, mode = arrival_case(g, str(name))
        got = ctx.generate_arrivals(rates, dt, seed, mode)
        assert_arrivals_match(g, str(name), got)


def test_reference_api_mirror(golden):
    """api.generate_arrivals reads like the reference call
    (generate_arrivals(trace, seed, ArrivalMode), workload.hpp:35)."""
    g = golden("arrivals")
    a = generate_arrivals(Trace(1.0, [2.0]), 0, UNIFORM)
    assert list(a) == [0.0, 0.5]
    rates, dt, seed, _ = arrival_case(g, "trace_4to32qps_s1")
    a = generate_arrivals(Trace(dt, list(rates)), seed, POISSON)
    assert_arrivals_match(g, "trace_4to32qps_s1", a)
    assert len(generate_arrivals(Trace(1.0, []), 0)) == 0
    with pytest.raises(ValueError):
        generate_arrivals(Trace(1.0, [1.0]), 0, "bursty")


def random_trace(rng):
    n = int(rng.integers(1, 3000))
    rates = rng.uniform(0.0, rng.choice([0.5, 20.0, 400.0, 5000.0]), n)
    gaps = rng.random(n) < rng.choice([0.0, 0.1, 0.6])
    rates[gaps] = 0.0
    if rng.random() < 0.3:
        rates[rng.random(n) < 0.2] = rng.uniform(1e-9, 1e-3)
    dt = float(rng.choice([1.0, 0.37, 0.01, 10.0, 1e-3]))
    return rates, dt


@pytest.mark.parametrize("mode", [0, 1])
def test_arrivals_match_port_on_random_traces(ctx, mode):
    rng = np.random.default_rng(20261017 + mode)
    total = 0
    for k in range(40):
        rates, dt = random_trace(rng)
        seed = int(rng.integers(0, 2**63))
        got = ctx.generate_arrivals(rates, dt, seed, mode)
        want = port_arrivals(rates, dt, seed, mode)
        assert len(got) == len(want), (k, len(got), len(want))
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), k
        assert np.all(np.diff(got) > 0)
        total += len(got)
    assert total > 10000


def test_draw_buffer_extension_is_transparent(ctx, golden, monkeypatch):
    """When the initial Exp(1) draw buffer is too short the call reruns with
    a longer one; results do not depend on the starting size."""
    g = golden("arrivals")
    rates, dt, seed, mode = arrival_case(g, "trace_4to32qps_s1")
    for start in ("2", "100", "5000"):
        monkeypatch.setenv("DS_ARRIVALS_INITIAL_DRAWS", start)
        assert_arrivals_match(g, "trace_4to32qps_s1", ctx.generate_arrivals(rates, dt, seed, mode))


def test_large_traces_match_port(ctx):
    """~1M and ~4M arrivals: many binade changes of the running target sum and
    thousands of interval boundaries."""
    for rates, dt, seed in (([2500.0] * 400, 1.0, 3), (list(np.linspace(0, 8000, 1000)), 1.0, 5)):
        got = ctx.generate_arrivals(rates, dt, seed, 0)
        want = port_arrivals(rates, dt, seed, 0)
        assert len(got) == len(want) > 900_000
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


def test_device_entry_point(ctx, golden):
    torch = pytest.importorskip("torch")
    g = golden("arrivals")
    rates, dt, seed, mode = arrival_case(g, "trace_1to8qps_s1")
    n = native.i64(0)
    L = native.lib()
    out = torch.full((4000,), -1.0, dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    native.check(L.ds_generate_arrivals_device(ctx.handle, P(rates), len(rates), dt, seed, mode,
                                               ctypes.c_void_p(out.data_ptr()), 4000,
                                               ctypes.byref(n), ctypes.c_void_p(stream)))
    torch.cuda.synchronize()
    c = n.value
    assert_arrivals_match(g, "trace_1to8qps_s1", out[:c].cpu().numpy())
    assert bool((out[c:] == -1.0).all())   # nothing written past the count
    small = torch.zeros(10, dtype=torch.float64, device="cuda")
    with pytest.raises(CapacityError):
        native.check(L.ds_generate_arrivals_device(ctx.handle, P(rates), len(rates), dt, seed,
                                                   mode, ctypes.c_void_p(small.data_ptr()), 10,
                                                   ctypes.byref(n), ctypes.c_void_p(stream)))
    assert n.value == c


def test_arrivals_errors(ctx):
    L = native.lib()
    n = native.i64(0)
    r = np.array([1.0, -2.0])
    with pytest.raises(DomainError):
        native.check(L.ds_generate_arrivals(ctx.handle, P(r), 2, 1.0, 0, 0, None, 0,
                                            ctypes.byref(n)))
    r = np.array([1.0, np.nan])
    with pytest.raises(DomainError):
        native.check(L.ds_generate_arrivals(ctx.handle, P(r), 2, 1.0, 0, 0, None, 0,
                                            ctypes.byref(n)))
    r = np.array([1.0])
    for dt in (0.0, -1.0, np.inf):
        with pytest.raises(DomainError):
            native.check(L.ds_generate_arrivals(ctx.handle, P(r), 1, dt, 0, 0, None, 0,
                                                ctypes.byref(n)))
    with pytest.raises(InvalidArgument):
        native.check(L.ds_generate_arrivals(ctx.handle, P(r), 1, 1.0, 0, 7, None, 0,
                                            ctypes.byref(n)))
    r = np.array([50.0])
    out = np.zeros(3)
    with pytest.raises(CapacityError):
        native.check(L.ds_generate_arrivals(ctx.handle, P(r), 1, 1.0, 0, 1, P(out), 3,
                                            ctypes.byref(n)))
    assert n.value == 50


def test_query_records_match_reference(ctx, golden):
    """Query records of the cascade-3 run (experiment.cpp:76-79): every field
    bit-exact (the latent scorer restates glibc's log/cos)."""
    g = golden("arrivals")
    want = g["records_cascade3"]
    m = QueryOutcomeModel(easy_fraction=0.3, quality_gap_scale=1.0, confidence_fidelity=0.35,
                          noise_sigma=0.12, seed=1)
    arr = g["trace_1to8qps_s1__arrivals"]
    got = sample_query_records(m, arr, float(g["records_cascade3_slo"]))
    for f in ("id", "arrival", "deadline", "quality_heavy", "confidence", "quality_light"):
        assert np.array_equal(got[f].view(np.uint64), want[f].view(np.uint64)), f


def test_query_records_match_latent_columns(ctx):
    """The record kernel and the column kernel are the same stream."""
    m = QueryOutcomeModel(seed=77)
    arr = np.linspace(0.0, 1000.0, 200_000)
    rec = ctx.sample_query_records(m.pod(), arr, 5.0, id0=123)
    conf, ql = ctx.score_latent(m.pod(), 123, len(arr), with_quality=True)
    assert np.array_equal(rec["confidence"], conf)
    assert np.array_equal(rec["quality_light"], ql)
    assert np.array_equal(rec["id"], np.arange(123, 123 + len(arr), dtype=np.uint64))
    assert np.array_equal(rec["deadline"], arr + 5.0)
    assert np.all(rec["quality_heavy"] == 1.0)
    with pytest.raises(DomainError):
        ctx.sample_query_records(m.pod(), arr[:10], 0.0)
    with pytest.raises(DomainError):
        ctx.sample_query_records(QueryOutcomeModel(easy_fraction=1.5).pod(), arr[:10], 1.0)


def test_grid_wide_target_sum_equals_single_cta_scan(ctx, monkeypatch):
    """K8c runs grid-wide (approximate prefix -> binades, exact integer scan,
    fp64 adds only at the special steps); DS_TARGET_SUM_SEQUENTIAL forces the
    single-CTA exact scan it falls back to. Both must give the same bits, and
    the C restatement's, on a 1M-arrival trace and on bursty rates."""
    for rates, seed in (([2500.0] * 400, 3), ([0.0, 9000.0, 1.0, 0.0, 52000.0, 3.0] * 5, 11)):
        rates = np.asarray(rates, np.float64)
        grid = ctx.generate_arrivals(rates, 1.0, seed, abi.ARRIVALS_POISSON)
        monkeypatch.setenv("DS_TARGET_SUM_SEQUENTIAL", "1")
        seq = ctx.generate_arrivals(rates, 1.0, seed, abi.ARRIVALS_POISSON)
        monkeypatch.delenv("DS_TARGET_SUM_SEQUENTIAL")
        assert grid.tobytes() == seq.tobytes()
        assert grid.tobytes() == port_arrivals(rates, 1.0, seed, abi.ARRIVALS_POISSON).tobytes()
