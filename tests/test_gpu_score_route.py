"""GPU parity: K4 latent scorer, K2 route/compaction, K3 curve replay.

Against the reference's own values (tests/golden/latent.npz from
oracle/make_golden.py) and the C restatement (oracle/ds_oracle.c)."""
import zlib

import numpy as np
import pytest

from oracle import lib
from paper_2411_15381_b200 import abi, workloads
from paper_2411_15381_b200.api import (DomainError, QueryOutcomeModel, default_context,
                                       sample_query)
from tests.helpers import route_digest

pytestmark = pytest.mark.gpu

# The latent scorer is bit-exact: its log and cos restate glibc's FMA builds
# (csrc/glibc_libm.h), so no tolerance band is needed anywhere below.


@pytest.fixture(scope="module")
def ctx():
    return default_context()


def same_bits(got, want):
    return np.array_equal(np.asarray(got, np.float64).view(np.uint64),
                          np.asarray(want, np.float64).view(np.uint64))


def test_latent_matches_reference_streams(ctx, golden):
    g = golden("latent")
    total = exact = 0
    for k in range(5):
        m = g[f"model{k}"]
        ids = g[f"ids{k}"]
        if k == 0:
            conf, ql = ctx.score_latent(m, 0, len(ids), with_quality=True)
        else:
            conf = np.zeros(len(ids))
            ql = np.zeros(len(ids))
            # contiguous runs keep this to a handful of launches
            for j, i in enumerate(ids):
                c, q = ctx.score_latent(m, int(i), 1, with_quality=True) if j < 64 else (None, None)
                if c is None:
                    break
                conf[j], ql[j] = c[0], q[0]
            ids = ids[:64]
            conf, ql = conf[:64], ql[:64]
        want_c = g[f"conf{k}"][:len(ids)]
        want_q = g[f"ql{k}"][:len(ids)]
        # every confidence and quality value bit for bit (the reference's own
        # sample_query streams, 5 models)
        assert same_bits(conf, want_c), k
        assert same_bits(ql, want_q), k
        total += len(ids)
    assert total > 5000


def test_latent_large_shard_vs_port(ctx):
    """1M-query style shard: GPU vs the C restatement (host libm, as the
    reference) on a 200K id window, bit for bit."""
    m = workloads.query_model()
    id0, n = 700_000, 200_000
    conf = ctx.score_latent(m, id0, n)
    want = np.zeros(n)
    lib.port().dso_sample_queries(abi.ptr(m), id0, n, abi.ptr(want), None, 8)
    assert same_bits(conf, want), f"{int((conf != want).sum())} of {n} differ"


def test_sample_query_api_semantics():
    """test_workload.cpp:105-157 through the reference-shaped API."""
    easy = QueryOutcomeModel(easy_fraction=1.0, noise_sigma=0.0, seed=5)
    for i in range(20):
        q = sample_query(easy, i, 3.0, 5.0)
        assert q.quality_heavy == 1.0 and q.quality_light >= q.quality_heavy
        assert q.deadline == pytest.approx(8.0) and 0.0 <= q.confidence <= 1.0
    flat = QueryOutcomeModel(confidence_fidelity=0.0, noise_sigma=0.0)
    assert sample_query(flat, 7, 0.0, 1.0).confidence == pytest.approx(0.5)
    m = QueryOutcomeModel(seed=123)
    a = sample_query(m, 77, 10.0, 5.0)
    b = sample_query(m, 77, 999.0, 5.0)
    assert a.confidence == b.confidence and a.quality_light == b.quality_light
    assert a.confidence != sample_query(QueryOutcomeModel(seed=124), 77, 10.0, 5.0).confidence
    with pytest.raises(DomainError):
        sample_query(m, 0, 0.0, 0.0)
    with pytest.raises(DomainError):
        sample_query(QueryOutcomeModel(easy_fraction=1.5), 0, 0.0, 5.0)
    conf, ql = default_context().score_latent(QueryOutcomeModel(seed=9).pod(), 0, 100000,
                                              with_quality=True)
    assert 0.29 < float((ql >= 1.0).mean()) < 0.31          # test_workload.cpp:126-136


def test_route_matches_reference_all_thresholds(ctx, golden):
    g = golden("latent")
    conf = g["conf0"]
    counts, lists = ctx.route(conf, g["route_grid"])
    assert np.array_equal(counts, g["route_counts"])
    for k, lst in enumerate(lists):
        assert route_digest(lst) == g["route_digest"][k], k


@pytest.mark.parametrize("n", [0, 1, 31, 2047, 2048, 2049, 100_003])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_route_edges_vs_port(ctx, n, dtype):
    rng = np.random.default_rng(n)
    conf = rng.random(n).astype(dtype)
    if n > 10:
        conf[::7] = 0.5                     # c == t stays light (test_policies.cpp:46-48)
        conf[1::11] = 0.0
        conf[2::13] = 1.0
    thr = np.array([0.0, 0.5, 1.0, 1.0000001, 0.25], np.float64)
    counts, lists = ctx.route(conf, thr, index_base=1000)
    c64 = conf.astype(np.float64)
    want_idx = np.zeros(len(thr) * max(n, 1), np.int64)
    want_cnt = np.zeros(len(thr), np.int64)
    lib.port().dso_route(abi.ptr(np.ascontiguousarray(c64)), n, abi.ptr(thr), len(thr), 1000,
                         abi.ptr(want_idx), abi.ptr(want_cnt))
    assert np.array_equal(counts, want_cnt)
    for k in range(len(thr)):
        assert np.array_equal(lists[k], want_idx[k * n: k * n + want_cnt[k]])


def test_route_loop_matches_reference_observe_then_defer(ctx, golden):
    """cluster.cpp:290-306: observe every confidence (decay 0.999) then defer."""
    g = golden("latent")
    conf = g["conf0"]
    curve = ctx.curve_observe(g["prior"], conf, 0.999)
    want = g["curve_after_0999"]
    assert np.array_equal(curve["bin_mass"].view(np.uint64), want["bin_mass"].view(np.uint64))
    assert curve["total_mass"] == want["total_mass"]


@pytest.mark.parametrize("decay_key,decay", [("curve_after_10", 1.0), ("curve_after_05", 0.5),
                                             ("curve_after_0999", 0.999)])
def test_curve_replay_bit_exact(ctx, golden, decay_key, decay):
    g = golden("latent")
    got = ctx.curve_observe(g["prior"], g["conf0"], decay)
    want = g[decay_key]
    assert np.array_equal(got["bin_mass"].view(np.uint64), want["bin_mass"].view(np.uint64))
    assert got["total_mass"] == want["total_mass"]


def test_curve_replay_large_and_f32_vs_port(ctx):
    rng = np.random.default_rng(3)
    conf = rng.random(50_000)
    conf[::5] = np.round(conf[::5] * 100) / 100        # grid-aligned: bin_of's +1e-9 nudge
    curve = workloads.uniform_prior()
    got = ctx.curve_observe(curve, conf, 0.999)
    want = curve.copy()
    lib.port().dso_curve_observe(abi.ptr(want), abi.ptr(conf), len(conf), 0.999)
    assert np.array_equal(got["bin_mass"].view(np.uint64), want["bin_mass"].view(np.uint64))
    assert got["total_mass"] == want["total_mass"]
    c32 = conf.astype(np.float32)
    got32 = ctx.curve_observe(curve, c32, 0.999)
    want32 = curve.copy()
    c32d = c32.astype(np.float64)
    lib.port().dso_curve_observe(abi.ptr(want32), abi.ptr(c32d), len(c32d), 0.999)
    assert np.array_equal(got32["bin_mass"].view(np.uint64), want32["bin_mass"].view(np.uint64))


@pytest.mark.parametrize("decay", [0.999, 0.9, 0.5, 1.0])
def test_curve_replay_long_vs_port(ctx, decay):
    """400K observations: the total-mass replay reaches its rounded fixed point
    and stops early (curve.cu); bins and total stay bit-identical, including
    bins that start at -0.0 and never get a hit."""
    rng = np.random.default_rng(17)
    conf = rng.random(400_000) * 0.9                  # bins 91..100 get no hits
    conf[::7] = np.round(conf[::7] * 100) / 100
    curve = workloads.uniform_prior()
    curve["bin_mass"][95] = -0.0
    curve["bin_mass"][100] = 5e-324                   # subnormal decay fixed point
    got = ctx.curve_observe(curve, conf, decay)
    want = curve.copy()
    lib.port().dso_curve_observe(abi.ptr(want), abi.ptr(conf), len(conf), decay)
    assert np.array_equal(got["bin_mass"].view(np.uint64), want["bin_mass"].view(np.uint64))
    assert np.float64(got["total_mass"]).view(np.uint64) == np.float64(want["total_mass"]).view(np.uint64)


def _port_curve(curve, conf, decay):
    want = curve.copy()
    c = np.ascontiguousarray(conf, np.float64)
    lib.port().dso_curve_observe(abi.ptr(want), abi.ptr(c), len(c), decay)
    return want


def _assert_same_bits(got, want):
    assert np.array_equal(got["bin_mass"].view(np.uint64), want["bin_mass"].view(np.uint64))
    assert np.float64(got["total_mass"]).view(np.uint64) == \
        np.float64(want["total_mass"]).view(np.uint64)


def _segmented_case(ctx, case):
    rng = np.random.default_rng(zlib.crc32(case.encode()))
    curve = workloads.uniform_prior()
    if case == "latent_1m":
        return curve, ctx.score_latent(workloads.query_model(), 0, 1_000_000), 0.999
    if case == "latent_1m_f32":
        c = ctx.score_latent(workloads.query_model(), 7, 1_000_000).astype(np.float32)
        return curve, c, 0.999
    if case == "one_bin":          # 100 bins decay without hits for the whole sequence
        return curve, np.full(100_000, 0.375), 0.999
    if case == "ragged":
        return curve, rng.random(70_001), 0.99
    if case == "slow_decay":       # the total's transient outlasts the sequence
        return curve, rng.random(300_000), 0.99999
    if case == "fast_decay":
        return curve, rng.random(200_000), 1e-3
    if case == "no_decay":
        curve["bin_mass"][3] = 0.3           # fractional: the +1s round
        return curve, rng.random(150_000), 1.0
    if case == "two_phase":        # half the bins go quiet, then the other half
        c = np.concatenate([rng.random(120_000) * 0.5, 0.5 + rng.random(120_000) * 0.5])
        return curve, c, 0.999
    if case == "large_state":
        curve["bin_mass"][:] = np.linspace(1e-300, 1e300, 101)
        curve["bin_mass"][7] = -0.0
        curve["total_mass"] = 1e300
        return curve, rng.random(100_000), 0.999
    raise ValueError(case)


@pytest.mark.parametrize("case", ["latent_1m", "latent_1m_f32", "one_bin", "ragged", "slow_decay",
                                  "fast_decay", "no_decay", "two_phase", "large_state"])
def test_curve_segmented_replay_vs_port(ctx, case):
    """Sequences of >= 32K observations take the segmented speculative replay
    (curve.cu, namespace spec): every segment replays from a closed-form guess
    and is re-run from its predecessor's end until the states agree bit for
    bit. The result must equal the sequential replay for any input, including
    chains that never merge (hitless bins, d = 1, slow decay), which fall back
    to the sequential walk."""
    curve, conf, decay = _segmented_case(ctx, case)
    got = ctx.curve_observe(curve, conf, decay)
    _assert_same_bits(got, _port_curve(curve, conf.astype(np.float64), decay))


def test_curve_segmented_invalid_confidence_stops_at_it(ctx):
    """A confidence outside [0, 1] in a long sequence: the host variant raises
    DomainError and the device variant leaves the curve replayed up to (not
    including) that observation, where observe_confidence would throw."""
    import torch
    from paper_2411_15381_b200 import native
    rng = np.random.default_rng(5)
    conf = rng.random(200_000)
    conf[123_457] = np.nan
    conf[150_000] = 1.5
    curve = workloads.uniform_prior()
    with pytest.raises(DomainError):
        ctx.curve_observe(curve, conf, 0.999)
    dconf = torch.from_numpy(conf).cuda()
    dcur = torch.from_numpy(curve.reshape(1).view(np.uint8).copy()).cuda()
    torch.cuda.synchronize()
    native.check(native.lib().ds_curve_observe_device(
        ctx.handle, native.c_p(dcur.data_ptr()), native.c_p(dconf.data_ptr()), abi.CONF_F64,
        len(conf), 0.999, None))
    torch.cuda.synchronize()
    got = dcur.cpu().numpy().view(abi.CURVE)[0]
    _assert_same_bits(got, _port_curve(curve, conf[:123_457], 0.999))
    # the device call recorded where the reference would have thrown
    with pytest.raises(DomainError, match="123457"):
        ctx.take_error()
    assert ctx.take_error() == -1   # cleared


@pytest.mark.parametrize("n,bad", [(40, 17), (5_000, 0), (5_000, 4_999)])
def test_curve_device_invalid_confidence_recorded(ctx, n, bad):
    """Short sequences (single-CTA replay): same stop point, same record."""
    import torch
    from paper_2411_15381_b200 import native
    conf = np.random.default_rng(n + bad).random(n)
    conf[bad] = -0.25
    curve = workloads.uniform_prior()
    dconf = torch.from_numpy(conf).cuda()
    dcur = torch.from_numpy(curve.reshape(1).view(np.uint8).copy()).cuda()
    torch.cuda.synchronize()
    assert ctx.take_error() == -1
    native.check(native.lib().ds_curve_observe_device(
        ctx.handle, native.c_p(dcur.data_ptr()), native.c_p(dconf.data_ptr()), abi.CONF_F64,
        n, 0.999, None))
    torch.cuda.synchronize()
    _assert_same_bits(dcur.cpu().numpy().view(abi.CURVE)[0], _port_curve(curve, conf[:bad], 0.999))
    with pytest.raises(DomainError, match=f"observation {bad} "):
        ctx.take_error()


@pytest.mark.parametrize("n", [5_000, 40_000])
@pytest.mark.parametrize("decay", [0.999, 0.5, 0.9999999, 1.0 - 2.0 ** -52, 1e-300, 1.0])
def test_curve_total_chain_edge_starts(ctx, n, decay):
    """The total's replay runs on a verified DFMA chain (curve.cu total_run):
    starting totals that cross binades, sit on ties, are tiny, huge, zero or
    negative must still give the two-rounding result bit for bit."""
    rng = np.random.default_rng(n)
    conf = rng.random(n)
    for t0 in (0.0, -0.0, 0.3, 31.999999999999996, 5e-324, 1e-300, 1e300, -7.25, 2.0 ** 53 - 3):
        curve = workloads.uniform_prior()
        curve["total_mass"] = t0
        got = ctx.curve_observe(curve, conf, decay)
        _assert_same_bits(got, _port_curve(curve, conf, decay))


def test_curve_domain_errors(ctx):
    c = workloads.uniform_prior()
    with pytest.raises(DomainError):
        ctx.curve_observe(c, np.array([0.3, 1.5, 0.2]), 1.0)
    with pytest.raises(DomainError):
        ctx.curve_observe(c, np.array([0.3]), 0.0)


def test_curve_segmented_replay_in_cuda_graph(ctx):
    """The segmented replay (a cooperative launch) captured into a CUDA graph
    and replayed gives the eager bits (scratch sized by an eager call first)."""
    import torch
    from paper_2411_15381_b200 import native
    conf = ctx.score_latent(workloads.query_model(), 0, 200_000)
    prior = workloads.uniform_prior()
    dconf = torch.from_numpy(conf).cuda()
    p_t = torch.from_numpy(prior.reshape(1).view(np.uint8).copy()).cuda()
    cur = torch.empty_like(p_t)
    s = torch.cuda.Stream()
    L = native.lib()

    def call():
        cur.copy_(p_t)
        native.check(L.ds_curve_observe_device(ctx.handle, native.c_p(cur.data_ptr()),
                                               native.c_p(dconf.data_ptr()), abi.CONF_F64,
                                               len(conf), 0.999, native.c_p(s.cuda_stream)))
    with torch.cuda.stream(s):
        call()
    torch.cuda.synchronize()
    eager = cur.cpu().numpy().tobytes()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        call()
    cur.zero_()
    with torch.cuda.stream(s):
        g.replay()
    torch.cuda.synchronize()
    assert cur.cpu().numpy().tobytes() == eager
    _assert_same_bits(cur.cpu().numpy().view(abi.CURVE)[0], _port_curve(prior, conf, 0.999))


def _port_route(conf, thr, base):
    n = len(conf)
    c64 = np.ascontiguousarray(conf, np.float64)
    idx = np.zeros(len(thr) * max(n, 1), np.int64)
    cnt = np.zeros(len(thr), np.int64)
    lib.port().dso_route(abi.ptr(c64), n, abi.ptr(thr), len(thr), base, abi.ptr(idx),
                         abi.ptr(cnt))
    return cnt, [idx[k * n: k * n + cnt[k]] for k in range(len(thr))]


@pytest.mark.parametrize("n", [8191, 8192, 8193, 3 * 8192 + 5, 1_048_583, 2_100_001])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_route_single_pass_tiles_vs_port(ctx, n, dtype):
    """K2's single pass around its 8,192-query tiles and past 128 tiles (more
    than one look-back round), NaN and boundary confidences included."""
    rng = np.random.default_rng(n + 3)
    conf = rng.random(n).astype(dtype)
    conf[::5] = 0.5
    conf[3::17] = np.nan                    # NaN < t is false: never deferred
    thr = np.array([0.5, 0.0, 1.0, 0.731], np.float64)
    counts, lists = ctx.route(conf, thr, index_base=7)
    want_cnt, want = _port_route(conf, thr, 7)
    assert np.array_equal(counts, want_cnt)
    for k in range(len(thr)):
        assert np.array_equal(lists[k], want[k]), k


def test_route_many_thresholds_many_tiles(ctx):
    conf = np.random.default_rng(9).random(50_000)
    thr = workloads.make_grid(0.01)
    counts, lists = ctx.route(conf, thr, index_base=123)
    want_cnt, want = _port_route(conf, thr, 123)
    assert np.array_equal(counts, want_cnt)
    assert all(np.array_equal(a, b) for a, b in zip(lists, want))


def test_route_device_misaligned_and_graph_replays(ctx):
    """A confidence pointer that is not 16-byte aligned (scalar loads), and
    the same launch replayed from a CUDA graph on changing data: the look-back
    flags are left clean by every launch."""
    import torch
    from paper_2411_15381_b200 import native
    L = native.lib()
    n = 70_001
    base = torch.from_numpy(np.random.default_rng(1).random(n + 1).astype(np.float32)).cuda()
    thr = torch.tensor([0.5, 0.25], dtype=torch.float64, device="cuda")
    heavy = torch.empty(2 * n, dtype=torch.int64, device="cuda")
    cnt = torch.empty(2, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()

    def launch(stream):
        native.check(L.ds_route_device(ctx.handle, native.c_p(base.data_ptr() + 4), abi.CONF_F32,
                                       n, native.c_p(thr.data_ptr()), 2, 0,
                                       native.c_p(heavy.data_ptr()), native.c_p(cnt.data_ptr()),
                                       native.c_p(stream)))

    def check():
        c = base[1:].cpu().numpy()
        want_cnt, want = _port_route(c, np.array([0.5, 0.25]), 0)
        got = cnt.cpu().numpy()
        assert np.array_equal(got, want_cnt)
        h = heavy.cpu().numpy().reshape(2, n)
        for k in range(2):
            assert np.array_equal(h[k, :got[k]], want[k])

    s = torch.cuda.Stream()
    launch(s.cuda_stream)
    torch.cuda.synchronize()
    check()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        launch(s.cuda_stream)
    for seed in range(3):
        base.copy_(torch.from_numpy(np.random.default_rng(seed + 10).random(n + 1)
                                    .astype(np.float32)))
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        check()
