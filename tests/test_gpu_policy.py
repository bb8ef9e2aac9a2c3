"""GPU: the Policy plugin API (policies.hpp:30-77) of api.Policy for every
PolicyKind, against the reference's own make_policy (policies.cpp:63-219) run
through oracle/_ref: per control tick, plan() (the GPU planner under the
reference's per-kind logic: Clipper's single frozen solve, Proteus' fix-ups,
AIMD's batch state fed by observe_batch), live_batch() after the feedback, and
entry_stage() on the reference's own RandomStream draws."""
import numpy as np
import pytest

from oracle import lib
from paper_2411_15381_b200 import abi, api, workloads

pytestmark = pytest.mark.gpu

KINDS = list(api.POLICY_KINDS)   # PolicyKind order (policies.hpp:11-20)


class RefStream:
    """bernoulli(p) on the reference's RandomStream(seed, "entry") outputs
    (rng.hpp:26-33: uniform = (u64 >> 11) * 2^-53, bernoulli = uniform < p)."""

    def __init__(self, seed, n):
        self.raw = np.zeros(n, np.uint64)
        lib.ref().dsref_stream_raw(seed, b"entry", n, abi.ptr(self.raw))
        self.i = 0

    def bernoulli(self, p):
        r = int(self.raw[self.i])
        self.i += 1
        return (r >> 11) * 2.0 ** -53 < p


def _cascade():
    light, heavy, slo = workloads.SHIPPED["cascade1"]["light"], \
        workloads.SHIPPED["cascade1"]["heavy"], workloads.SHIPPED["cascade1"]["slo"]
    c = api.CascadeProfile("cascade1", api.ModelProfile("light", dict(light)),
                           api.ModelProfile("heavy", dict(heavy)),
                           api.DeferralCurve.uniform_prior(), slo)
    return c


@pytest.mark.parametrize("kind", KINDS)
def test_policy_kind_matches_reference(kind):
    if not lib.ref_available():
        pytest.skip("reference library not built")
    rng = np.random.default_rng(KINDS.index(kind) + 7)
    n = 14
    cas = _cascade()
    grid = list(workloads.make_grid(0.01))
    demands = rng.uniform(1.0, 60.0, n)
    problems = [api.AllocationProblem(float(d), 16, cas, 1.05, grid,
                                      api.QueueState(int(rng.integers(0, 12)), float(d) + 0.1),
                                      api.QueueState(int(rng.integers(0, 5)), 0.3 * float(d)))
                for d in demands]
    ev_model = rng.integers(0, 2, n).astype(np.int32)
    ev_timeout = (rng.random(n) < 0.3).astype(np.int32)
    params = api.PolicyParams(kind=kind, peak_demand_qps=55.0, fixed_threshold=0.37,
                              aimd_add_step=2, aimd_mult_factor=0.5)
    # the reference
    pods = np.concatenate([api._problem_pod(p, abi.SOLVE).reshape(1) for p in problems])
    cpod = cas.pod().reshape(1)
    g = np.asarray(grid, np.float64)
    want = np.zeros(n, abi.PLAN)
    live = np.zeros(2 * n, np.int32)
    entry = np.zeros(n, np.int32)
    rc = lib.ref().dsref_policy_run(KINDS.index(kind), params.peak_demand_qps,
                                    params.fixed_threshold, params.aimd_add_step,
                                    params.aimd_mult_factor, abi.ptr(pods), n, abi.ptr(cpod),
                                    abi.ptr(g), len(g), abi.ptr(ev_model), abi.ptr(ev_timeout),
                                    11, abi.ptr(want), abi.ptr(live), abi.ptr(entry))
    assert rc == 0, lib.ref().dsref_last_error()
    # the GPU-planned mirror
    pol = api.make_policy(params)
    stream = RefStream(11, 4 * n)
    assert pol.kind() == kind
    assert pol.uses_discriminator() == (kind not in ("clipper_light", "clipper_heavy",
                                                     "proteus_like"))
    for i, p in enumerate(problems):
        got = pol.plan(p)
        w = want[i]
        assert (got.x1, got.x2, got.b1, got.b2, got.threshold, got.feasible) == (
            w["x1"], w["x2"], w["b1"], w["b2"], w["threshold"], bool(w["feasible"])), (kind, i)
        pol.observe_batch(api.HEAVY if ev_model[i] else api.LIGHT, bool(ev_timeout[i]))
        assert (pol.live_batch(api.LIGHT), pol.live_batch(api.HEAVY)) == (
            live[2 * i], live[2 * i + 1]), (kind, i)
        stage = pol.entry_stage(got, stream)
        assert stage == (api.HEAVY if entry[i] else api.LIGHT), (kind, i)
    # defers: strict < for the discriminator kinds, never for the others
    assert pol.defers(0.49, 0.5) == pol.uses_discriminator()
    assert not pol.defers(0.5, 0.5)
