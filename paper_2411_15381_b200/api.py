"""Reference-shaped operator API over the C ABI.

Mirrors the reference's free functions and types for the hot path
(proj/include/diffserve/allocator.hpp:12-91, profiles.hpp:11-68,
workload.hpp:39-63, policies.hpp:30-77) with the same names, argument meaning
and exception behaviour, so parity tests read like the reference's own
(tests/test_api_*.py vs proj/tests/test_allocator.cpp). Every call runs on the
GPU through libds_b200.so; there is no CPU fallback.
"""
from __future__ import annotations

import dataclasses
from dataclasses import dataclass, field

import numpy as np

from . import abi, workloads
from .native import (CapacityError, Context, DomainError, InvalidArgument, InvariantError,
                     OutOfRange)

__all__ = ["ModelProfile", "DeferralCurve", "CascadeProfile", "QueueState", "AllocationProblem",
           "AllocationPlan", "QueryOutcomeModel", "Query", "solve", "solve_static_peak",
           "solve_pinned_threshold", "solve_fixed_batches", "solve_single_model",
           "solve_even_split", "solve_batch", "sample_query", "sample_queries",
           "observe_confidences", "route", "InvalidArgument", "DomainError", "InvariantError",
           "OutOfRange", "CapacityError", "default_context", "Policy", "make_policy",
           "PolicyParams", "POLICY_KINDS", "LIGHT", "HEAVY", "aimd_update", "Trace",
           "POISSON", "UNIFORM", "generate_arrivals",
           "sample_query_records", "fmt6", "write_csv"]

_ctx: Context | None = None


def default_context() -> Context:
    global _ctx
    if _ctx is None:
        _ctx = Context(0)
    return _ctx


@dataclass
class ModelProfile:                       # profiles.hpp:11-19
    name: str
    latency_table: dict

    def batch_sizes(self):
        return sorted(self.latency_table)

    def min_batch(self):
        return min(self.latency_table)

    def max_batch(self):
        return max(self.latency_table)


@dataclass
class DeferralCurve:                      # profiles.hpp:35-48
    bin_mass: np.ndarray = field(default_factory=lambda: np.zeros(abi.CURVE_BINS))
    total_mass: float = 0.0

    @staticmethod
    def empty() -> "DeferralCurve":
        return DeferralCurve()

    @staticmethod
    def uniform_prior() -> "DeferralCurve":
        c = workloads.uniform_prior()
        return DeferralCurve(np.array(c["bin_mass"]), float(c["total_mass"]))

    @staticmethod
    def from_samples(samples) -> "DeferralCurve":
        return observe_confidences(DeferralCurve(), np.asarray(samples, np.float64), 1.0)

    def pod(self) -> np.ndarray:
        c = np.zeros((), abi.CURVE)
        c["bin_mass"] = self.bin_mass
        c["total_mass"] = self.total_mass
        return c


@dataclass
class CascadeProfile:                     # profiles.hpp:62-68
    name: str
    light: ModelProfile
    heavy: ModelProfile
    deferral: DeferralCurve = field(default_factory=DeferralCurve)
    slo_seconds: float = 0.0

    def pod(self) -> np.ndarray:
        return workloads.make_cascade(self.light.latency_table, self.heavy.latency_table,
                                      self.slo_seconds, self.deferral.pod())


@dataclass
class QueueState:                         # allocator.hpp:12-15
    queue_length: int = 0
    arrival_rate: float = 0.0


@dataclass
class AllocationProblem:                  # allocator.hpp:27-37
    demand_qps: float = 0.0
    total_servers: int = 0
    cascade: CascadeProfile | None = None
    overprovision_lambda: float = 1.05
    threshold_grid: list = field(default_factory=list)
    light_queue: QueueState = field(default_factory=QueueState)
    heavy_queue: QueueState = field(default_factory=QueueState)
    queuing: str = "littles_law"          # or "twice_exec"
    queue_sentinel_seconds: float = 1e6


@dataclass
class AllocationPlan:                     # allocator.hpp:39-46
    x1: int = 0
    x2: int = 0
    b1: int = 0
    b2: int = 0
    threshold: float = 0.0
    feasible: bool = False


def _problem_pod(p: AllocationProblem, mode: int, **extra) -> np.ndarray:
    if p.cascade is None:
        raise InvalidArgument("allocation problem has no cascade")
    r = np.zeros((), abi.PROBLEM)
    r["demand_qps"] = p.demand_qps
    r["overprovision_lambda"] = p.overprovision_lambda
    r["queue_sentinel_seconds"] = p.queue_sentinel_seconds
    r["light_len"] = p.light_queue.queue_length
    r["light_rate"] = p.light_queue.arrival_rate
    r["heavy_len"] = p.heavy_queue.queue_length
    r["heavy_rate"] = p.heavy_queue.arrival_rate
    r["total_servers"] = p.total_servers
    r["queuing"] = abi.QUEUING_TWICE_EXEC if p.queuing == "twice_exec" else abi.QUEUING_LITTLES_LAW
    r["mode"] = mode
    for k, v in extra.items():
        r[k] = v
    return r


def _run(p: AllocationProblem, mode: int, **extra) -> AllocationPlan:
    prob = _problem_pod(p, mode, **extra).reshape(1)
    cas = p.cascade.pod().reshape(1)
    grid = np.asarray(p.threshold_grid, np.float64)
    out = default_context().plan_batch(prob, cas, grid if len(grid) else np.zeros(0),
                                       np.array([0, len(grid)], np.int32))[0]
    return AllocationPlan(int(out["x1"]), int(out["x2"]), int(out["b1"]), int(out["b2"]),
                          float(out["threshold"]), bool(out["feasible"]))


def solve(p: AllocationProblem) -> AllocationPlan:                    # allocator.cpp:153
    return _run(p, abi.SOLVE)


def solve_static_peak(p: AllocationProblem, peak_demand_qps: float) -> AllocationPlan:
    return solve(dataclasses.replace(p, demand_qps=peak_demand_qps))   # allocator.cpp:171


def solve_pinned_threshold(p: AllocationProblem, fixed_t: float) -> AllocationPlan:
    return _run(p, abi.SOLVE_PINNED, fixed_threshold=fixed_t)          # allocator.cpp:176


def solve_fixed_batches(p: AllocationProblem, b1: int, b2: int) -> AllocationPlan:
    return _run(p, abi.SOLVE_FIXED_BATCHES, fixed_b1=b1, fixed_b2=b2)  # allocator.cpp:213


def solve_even_split(p: AllocationProblem) -> AllocationPlan:          # allocator.cpp:270
    return _run(p, abi.SOLVE_EVEN_SPLIT)


def solve_single_model(m: ModelProfile, is_light: bool, total_servers: int, demand_qps: float,
                       overprovision_lambda: float, slo_seconds: float) -> AllocationPlan:
    """allocator.cpp:232-268: all servers host `m` (the other side is unused)."""
    other = ModelProfile("unused", {1: 1.0})
    c = CascadeProfile("single", m if is_light else other, other if is_light else m,
                       DeferralCurve(), slo_seconds)
    p = AllocationProblem(demand_qps, total_servers, c, overprovision_lambda)
    return _run(p, abi.SOLVE_SINGLE_LIGHT if is_light else abi.SOLVE_SINGLE_HEAVY)


def solve_batch(problems: np.ndarray, cascades: np.ndarray, grid_values: np.ndarray,
                grid_offsets: np.ndarray, ctx: Context | None = None) -> np.ndarray:
    """Bulk planner: one launch for many problems (the K1 hot path)."""
    return (ctx or default_context()).plan_batch(problems, cascades, grid_values, grid_offsets)


@dataclass
class QueryOutcomeModel:                  # workload.hpp:52-58
    easy_fraction: float = 0.3
    quality_gap_scale: float = 1.0
    confidence_fidelity: float = 1.5
    noise_sigma: float = 0.15
    seed: int = 0

    def pod(self) -> np.ndarray:
        m = np.zeros((), abi.QUERY_MODEL)
        for k in ("easy_fraction", "quality_gap_scale", "confidence_fidelity", "noise_sigma",
                  "seed"):
            m[k] = getattr(self, k)
        return m


@dataclass
class Query:                              # workload.hpp:39-46
    id: int
    arrival: float
    deadline: float
    quality_light: float
    quality_heavy: float
    confidence: float


def sample_queries(model: QueryOutcomeModel, n: int, id0: int = 0, ctx: Context | None = None):
    """(confidence, quality_light) of ids id0..id0+n-1 on the GPU (K4)."""
    return (ctx or default_context()).score_latent(model.pod(), id0, n, with_quality=True)


def sample_query(model: QueryOutcomeModel, id: int, arrival_time: float,
                 slo_seconds: float) -> Query:                          # workload.cpp:108
    if not (0.0 <= model.easy_fraction <= 1.0):
        raise DomainError("easy_fraction must lie in [0, 1]")
    if not (slo_seconds > 0.0):
        raise DomainError("slo_seconds must be positive")
    conf, ql = sample_queries(model, 1, id)
    return Query(id, arrival_time, arrival_time + slo_seconds, float(ql[0]), 1.0, float(conf[0]))


@dataclass
class Trace:                              # workload.hpp:10-16
    interval_seconds: float = 1.0
    rates: list = None

    def duration(self) -> float:
        return self.interval_seconds * float(len(self.rates or []))

    def peak(self) -> float:
        return max(self.rates) if self.rates else 0.0


POISSON = "poisson"                       # ArrivalMode, workload.hpp:26
UNIFORM = "uniform"


def generate_arrivals(trace: Trace, seed: int, mode: str = POISSON,
                      ctx: Context | None = None) -> np.ndarray:
    """generate_arrivals (workload.cpp:82-106) on the GPU (K8), bit-identical."""
    if mode not in (POISSON, UNIFORM):
        raise ValueError(f"unknown arrival mode '{mode}'")
    m = abi.ARRIVALS_UNIFORM if mode == UNIFORM else abi.ARRIVALS_POISSON
    return (ctx or default_context()).generate_arrivals(trace.rates or [], trace.interval_seconds,
                                                        seed, m)


def sample_query_records(model: QueryOutcomeModel, arrivals, slo_seconds: float, id0: int = 0,
                         ctx: Context | None = None) -> np.ndarray:
    """The run_experiment query loop (experiment.cpp:76-79): Query records
    (abi.QUERY) for ids id0.. at the given arrivals, on the GPU (K4)."""
    return (ctx or default_context()).sample_query_records(model.pod(), arrivals, slo_seconds,
                                                           id0)


def fmt6(v: float) -> str:
    """metrics.cpp:67-71 ("%.6g"), computed on the GPU (K9)."""
    return default_context().format_g6([v])[0].decode()


def write_csv(out_dir: str, intervals: np.ndarray, records: np.ndarray, plans: np.ndarray,
              ctx: Context | None = None) -> None:
    """write_csv (metrics.cpp:91-127): intervals.csv, queries.csv, plans.csv in
    out_dir, rows formatted on the GPU (K9) from abi.INTERVAL_SNAPSHOT /
    abi.QUERY_RECORD / abi.PLAN_LOG_ENTRY arrays; byte-identical files."""
    import os
    c = ctx or default_context()
    os.makedirs(out_dir, exist_ok=True)
    for name, data in (("intervals.csv", c.format_intervals_csv(intervals)),
                       ("queries.csv", c.format_queries_csv(records)),
                       ("plans.csv", c.format_plans_csv(plans))):
        with open(os.path.join(out_dir, name), "wb") as f:
            f.write(data)


def observe_confidences(curve: DeferralCurve, conf, decay: float) -> DeferralCurve:
    """observe_confidence (profiles.cpp:108-120) applied in order (K3)."""
    out = default_context().curve_observe(curve.pod(), np.ascontiguousarray(conf), decay)
    return DeferralCurve(np.array(out["bin_mass"]), float(out["total_mass"]))


def route(conf, thresholds, index_base: int = 0):
    """Policy::defers (policies.cpp:37-39) over a batch, order-preserving (K2)."""
    return default_context().route(np.ascontiguousarray(conf), thresholds, index_base)


# ---- Policy plugin boundary (policies.hpp:30-77) ------------------------------------

@dataclass
class PolicyParams:                        # policies.hpp:62-68
    kind: str = "diffserve"
    peak_demand_qps: float = 0.0
    fixed_threshold: float = 0.5
    aimd_add_step: int = 1
    aimd_mult_factor: float = 0.5


LIGHT, HEAVY = "light", "heavy"            # ModelKind, policies.hpp:25
POLICY_KINDS = ("diffserve", "diffserve_static", "clipper_light", "clipper_heavy",
                "proteus_like", "abl_static_threshold", "abl_aimd_batching",
                "abl_no_queuing_model")     # PolicyKind, policies.hpp:11-20


def aimd_update(m: ModelProfile, current_batch: int, slo_timeout: bool, add_step: int,
                mult_factor: float) -> int:
    """aimd_update (policies.cpp:45-59): multiplicative decrease to the largest
    profiled batch <= b * mult on an SLO timeout, else additive increase to the
    smallest profiled batch >= b + add (capped at the largest)."""
    sizes = m.batch_sizes()
    if slo_timeout:
        target = current_batch * mult_factor
        nxt = sizes[0]
        for b in sizes:
            if b <= target:
                nxt = b
        return nxt
    want = current_batch + add_step
    for b in sizes:
        if b >= want:
            return b
    return sizes[-1]


class Policy:
    """The reference's plugin API (policies.hpp:30-60) for every PolicyKind
    make_policy knows (policies.cpp:63-219); plan() runs on the GPU planner
    (K1), the per-kind control logic -- Clipper's one frozen solve, Proteus'
    fix-ups and random entry stage, AIMD's batch state -- is the reference's."""

    def __init__(self, params: PolicyParams):
        if params.kind not in POLICY_KINDS:
            raise InvalidArgument(f"unknown policy kind '{params.kind}'")
        self.params = params
        self._frozen = None            # Clipper: the one solve, frozen (policies.cpp:98-110)
        self._cascade = None           # AIMD state (policies.cpp:157-183)
        self._b1 = self._b2 = 0

    def kind(self) -> str:
        return self.params.kind

    def entry_stage(self, plan: AllocationPlan, rng=None) -> str:
        """policies.cpp:31-35 (light), 92-94 (Clipper), 123-128 (Proteus:
        uniform over hosted variants via rng.bernoulli(0.5))."""
        k = self.params.kind
        if k == "clipper_light":
            return LIGHT
        if k == "clipper_heavy":
            return HEAVY
        if k == "proteus_like":
            if plan.x1 > 0 and plan.x2 > 0:
                if rng is None:
                    raise InvalidArgument("proteus_like entry_stage needs a random stream")
                return HEAVY if rng.bernoulli(0.5) else LIGHT
            return HEAVY if plan.x2 > 0 else LIGHT
        return LIGHT

    def defers(self, confidence: float, threshold: float) -> bool:     # policies.cpp:37-39
        if not self.uses_discriminator():
            return False
        return confidence < threshold

    def uses_discriminator(self) -> bool:
        return self.params.kind not in ("clipper_light", "clipper_heavy", "proteus_like")

    def plan(self, p: AllocationProblem) -> AllocationPlan:
        k = self.params.kind
        if k == "diffserve":
            return solve(p)
        if k == "diffserve_static":
            return solve_static_peak(p, self.params.peak_demand_qps)
        if k in ("clipper_light", "clipper_heavy"):
            if self._frozen is None:
                light = k == "clipper_light"
                m = p.cascade.light if light else p.cascade.heavy
                out = solve_single_model(m, light, p.total_servers, self.params.peak_demand_qps,
                                         p.overprovision_lambda, p.cascade.slo_seconds)
                if light:
                    out.b2 = p.cascade.heavy.min_batch()
                else:
                    out.b1 = p.cascade.light.min_batch()
                self._frozen = out
            return dataclasses.replace(self._frozen)
        if k == "proteus_like":
            out = solve_even_split(p)
            if out.b1 == 0:
                out.b1 = p.cascade.light.min_batch()
            if out.b2 == 0:
                out.b2 = p.cascade.heavy.min_batch()
            return out
        if k == "abl_static_threshold":
            return solve_pinned_threshold(p, self.params.fixed_threshold)
        if k == "abl_aimd_batching":
            self._cascade = p.cascade
            if self._b1 == 0:          # slow start at the smallest profiled batches
                self._b1 = p.cascade.light.min_batch()
                self._b2 = p.cascade.heavy.min_batch()
            return solve_fixed_batches(p, self._b1, self._b2)
        # abl_no_queuing_model (policies.cpp:188-192)
        return solve(dataclasses.replace(p, queuing="twice_exec"))

    def observe_batch(self, model: str, slo_timeout: bool) -> None:    # policies.cpp:166-172
        if self.params.kind != "abl_aimd_batching" or self._cascade is None or self._b1 == 0:
            return
        if model == LIGHT:
            self._b1 = aimd_update(self._cascade.light, self._b1, slo_timeout,
                                   self.params.aimd_add_step, self.params.aimd_mult_factor)
        else:
            self._b2 = aimd_update(self._cascade.heavy, self._b2, slo_timeout,
                                   self.params.aimd_add_step, self.params.aimd_mult_factor)

    def live_batch(self, model: str) -> int:                           # policies.cpp:175-177
        if self.params.kind != "abl_aimd_batching":
            return 0
        return self._b1 if model == LIGHT else self._b2


def make_policy(params: PolicyParams) -> Policy:                       # policies.cpp:198
    return Policy(params)
