"""Named input shapes of the hot path.

* SHIPPED: the three cascades of the reference profile file
  (reference proj/configs/cascades.profiles:13-41) and their experiment
  configs (proj/configs/cascade{1,2,3}.cfg).
* fitted_cascade(): config 4's 32-batch tables e(b) = e1*(1 + s*(b-1)),
  b = 1..32, fitted to the shipped tables.
* c2_problems(): the acceptance-C2 problem recipe (acceptance_main.cpp:177-190)
  re-expressed with a numpy generator for benchmark batches of any size (the
  parity fixtures use the reference's own generator, see oracle/make_golden.py).
"""
from __future__ import annotations

import math

import numpy as np

from . import abi

# cascades.profiles:13-41 (shipped prior: 32 samples 0.2125 .. 0.9875).
_PRIOR = [0.2125 + 0.025 * i for i in range(32)]
SHIPPED = {
    "cascade1": dict(slo=5.0, light={1: 0.10, 2: 0.13, 4: 0.18, 8: 0.30, 16: 0.52},
                     heavy={1: 1.78, 2: 1.90}),
    "cascade2": dict(slo=5.0, light={1: 0.05, 2: 0.07, 4: 0.10, 8: 0.17, 16: 0.30},
                     heavy={1: 1.78, 2: 1.90}),
    "cascade3": dict(slo=15.0, light={1: 0.50, 2: 0.65, 4: 0.95, 8: 1.60, 16: 2.90},
                     heavy={1: 6.0, 2: 6.4}),
}
SHIPPED_PRIOR_SAMPLES = [float(f"{x:.4f}") for x in _PRIOR]

# cascade{1,2,3}.cfg:15-21 + config.hpp:40-43 defaults (easy 0.3, gap 1.0).
QUERY_MODEL = dict(easy_fraction=0.3, quality_gap_scale=1.0, confidence_fidelity=0.35,
                   noise_sigma=0.12, seed=1)

# (e1, s) per cascade, light then heavy.
FITTED = {
    "cascade1": dict(light=(0.10, 0.28), heavy=(1.78, 0.0674), slo=5.0),
    "cascade2": dict(light=(0.05, 1.0 / 3.0), heavy=(1.78, 0.0674), slo=5.0),
    "cascade3": dict(light=(0.50, 0.32), heavy=(6.0, 0.0667), slo=15.0),
}


def query_model(**over) -> np.ndarray:
    m = np.zeros((), abi.QUERY_MODEL)
    for k, v in {**QUERY_MODEL, **over}.items():
        m[k] = v
    return m


def make_cascade(light: dict, heavy: dict, slo: float, curve: np.ndarray | None = None
                 ) -> np.ndarray:
    """A ds_cascade record; curve defaults to uniform_prior (profiles.cpp:84-90)."""
    c = np.zeros((), abi.CASCADE)
    c["light"] = abi.model_profile(light)
    c["heavy"] = abi.model_profile(heavy)
    c["slo_seconds"] = slo
    if curve is None:
        curve = uniform_prior()
    c["deferral"] = curve
    return c


def empty_curve() -> np.ndarray:
    return np.zeros((), abi.CURVE)


def uniform_prior() -> np.ndarray:
    """DeferralCurve::uniform_prior (profiles.cpp:84-90): exact f(k/100) = k/100."""
    c = np.zeros((), abi.CURVE)
    c["bin_mass"][:100] = 1.0
    c["total_mass"] = 100.0
    return c


def fitted_tables(name: str) -> tuple[dict, dict, float]:
    f = FITTED[name]
    e1, s = f["light"]
    h1, hs = f["heavy"]
    light = {b: e1 * (1.0 + s * (b - 1)) for b in range(1, 33)}
    heavy = {b: h1 * (1.0 + hs * (b - 1)) for b in range(1, 33)}
    return light, heavy, f["slo"]


def full_grid(step: float = 0.01) -> np.ndarray:
    """testutil::full_grid (helpers.hpp:74-82): k*step clamped to 1."""
    g = []
    k = 0
    while True:
        t = k * step
        if t > 1.0 + 1e-12:
            break
        g.append(min(t, 1.0))
        k += 1
    return np.asarray(g, np.float64)


def make_grid(step: float = 0.01) -> np.ndarray:
    """Simulation's grid (cluster.cpp:20-28): k/n with n = lround(1/step).

    std::lround rounds halves away from zero (np.round would round them to
    even: step 0.4 gives n = 3 here as in the reference, not 2); a step
    outside (0, 1] raises like the reference's std::invalid_argument."""
    if not (step > 0.0) or step > 1.0:
        raise ValueError("threshold grid step must be in (0, 1]")
    x = 1.0 / step
    n = math.floor(x)
    if x - n >= 0.5:     # exact for x >= 1
        n += 1
    n = int(n)
    return np.asarray([k / n for k in range(n + 1)], np.float64)


def c2_problems(cascade: np.ndarray, servers: int, n: int, seed: int = 7) -> np.ndarray:
    """acceptance_main.cpp:177-190 recipe with a numpy stream (bench batches)."""
    rng = np.random.default_rng(seed)
    light = cascade["light"]
    nb = int(light["n"])
    bmax = int(light["batch"][nb - 1])
    cap = servers * (bmax / float(light["latency"][nb - 1]))
    u = rng.random((n, 3))
    p = np.zeros(n, abi.PROBLEM)
    p["total_servers"] = servers
    p["demand_qps"] = 1.2 * u[:, 0] * cap
    p["overprovision_lambda"] = 1.05
    p["queue_sentinel_seconds"] = 1e6
    p["light_len"] = np.floor(20.0 * u[:, 1]).astype(np.int64)
    p["light_rate"] = p["demand_qps"] + 0.1
    p["heavy_len"] = np.floor(8.0 * u[:, 2]).astype(np.int64)
    p["heavy_rate"] = 0.3 * p["demand_qps"] + 0.1
    p["mode"] = abi.SOLVE
    return p
