"""Shared test helpers: golden-set unpacking and plan comparison."""
import numpy as np

from paper_2411_15381_b200 import abi


def plan_fields(p):
    return (int(p["x1"]), int(p["x2"]), int(p["b1"]), int(p["b2"]), float(p["threshold"]),
            int(p["feasible"]))


def assert_plans_equal(got, want, label=""):
    """Exact AllocationPlan equality (check_plans_equal, test_allocator.cpp:90-97)."""
    assert got.shape == want.shape
    bad = []
    for i in range(len(want)):
        if plan_fields(got[i]) != plan_fields(want[i]):
            bad.append(i)
    assert not bad, (f"{label}: {len(bad)} of {len(want)} plans differ; first {bad[0]}: "
                     f"got {plan_fields(got[bad[0]])} want {plan_fields(want[bad[0]])}")


def planner_set(g):
    return (np.ascontiguousarray(g["problems"]), np.ascontiguousarray(g["cascades"]),
            np.ascontiguousarray(g["grid_values"]), np.ascontiguousarray(g["grid_offsets"]))


def route_digest(idx):
    """Order-sensitive digest of a heavy list (same formula as make_golden.py)."""
    idx = np.asarray(idx, np.uint64)
    if len(idx) == 0:
        return np.uint64(0)
    return np.uint64(int(np.bitwise_xor.reduce(
        (idx * np.uint64(0x9E3779B97F4A7C15)) ^ np.arange(len(idx), dtype=np.uint64))))


def arrival_case(g, name):
    """(rates, interval_seconds, seed, mode) of a generate_arrivals golden."""
    dt, seed, mode = g[f"{name}__meta"]
    return np.ascontiguousarray(g[f"{name}__rates"]), float(dt), int(seed), int(mode)


def assert_arrivals_match(g, name, got):
    """Bit-exact equality with the reference's timestamps (count, sha256 of
    the bytes, and the stored values)."""
    import hashlib
    got = np.ascontiguousarray(got, np.float64)
    assert len(got) == int(g[f"{name}__count"]), (name, len(got), int(g[f"{name}__count"]))
    if f"{name}__arrivals" in g:
        want = g[f"{name}__arrivals"]
        bad = np.flatnonzero(got.view(np.uint64) != want.view(np.uint64))
        assert len(bad) == 0, (name, len(bad), bad[:5], got[bad[:5]], want[bad[:5]])
    else:
        idx = g[f"{name}__sample_idx"]
        assert np.array_equal(got[idx].view(np.uint64), g[f"{name}__sample"].view(np.uint64)), name
    assert hashlib.sha256(got.tobytes()).hexdigest() == str(g[f"{name}__sha256"]), name


def special_doubles():
    """Doubles that stress "%.6g": zeros, infinities, NaNs, subnormals,
    extreme exponents, exact decimal ties and powers of ten +- 1 ulp."""
    v = [0.0, -0.0, np.inf, -np.inf, np.nan, -np.nan, 5e-324, -5e-324, 2.2250738585072014e-308,
         1.7976931348623157e308, 1e-5, 1e-4, 9.999995e-5, 0.0001, 99999.95, 999999.5, 1e6,
         123456.5, 1234565.0, 1234575.0, 0.5, 2.5, 100000.0, 999999.0, 9999995.0, 1e15, 1e16,
         1e22, 1e23, 1e-17, 1e-18, 1e-300, 1e300, 3600.0, 0.1, 0.3, 1 / 3]
    out = []
    for x in v:
        out.append(x)
        if np.isfinite(x) and x != 0:
            if abs(x) < 1.7976931348623157e308:
                out.append(np.nextafter(x, np.inf))
            out.append(np.nextafter(x, -np.inf))
    return np.array(out, np.float64)


def random_doubles(rng, n):
    """Mixed distributions: raw bit patterns, log-uniform magnitudes, decimal
    grids (exact ties), times in seconds, qualities around 1."""
    k = n // 6
    raw = rng.integers(0, 2**63, k, dtype=np.int64).view(np.uint64)
    bits = (raw | (rng.integers(0, 2, k).astype(np.uint64) << np.uint64(63))).view(np.float64)
    logu = 10.0 ** rng.uniform(-30, 30, k) * rng.choice([-1, 1], k)
    grid = rng.integers(0, 10**8, k) / 10.0 ** rng.integers(0, 12, k)
    ints = rng.integers(0, 10**9, k).astype(np.float64)
    times = rng.uniform(0, 3600, k)
    qual = 1.0 + rng.normal(0, 0.5, n - 5 * k)
    return np.concatenate([bits, logu, grid, ints, times, qual])


def random_query_records(rng, n):
    """QueryRecord rows (abi.QUERY_RECORD) with random engaged optionals."""
    r = np.zeros(n, abi.QUERY_RECORD)
    r["id"] = rng.integers(0, 2**63, n, dtype=np.int64).astype(np.uint64)
    r["id"][: n // 2] = np.arange(n // 2, dtype=np.uint64)
    r["arrival"] = rng.uniform(0, 3600, n)
    r["deadline"] = r["arrival"] + rng.choice([5.0, 15.0, 0.3], n)
    r["confidence"] = np.clip(0.5 + rng.normal(0, 0.4, n), 0.0, 1.0)
    r["quality_light"] = 1.0 + rng.normal(0, 0.6, n)
    r["quality_heavy"] = 1.0
    fields = ("light_start", "light_end", "heavy_start", "heavy_end", "completion",
              "delivered_quality")
    for f in fields:
        r[f] = r["arrival"] + rng.exponential(1.0, n)
    r["delivered_quality"] = np.where(rng.random(n) < 0.5, r["quality_light"], 1.0)
    r["present"] = rng.integers(0, 128, n).astype(np.uint32)
    r["outcome"] = rng.integers(0, 4, n)
    sp = special_doubles()
    m = min(len(sp), n)
    for j, f in enumerate(("arrival", "confidence", "quality_light", "deadline", "completion")):
        r[f][j * m // 5: j * m // 5 + m] = np.roll(sp, j)[: len(r[f][j * m // 5: j * m // 5 + m])]
    return r


def random_intervals(rng, n):
    s = np.zeros(n, abi.INTERVAL_SNAPSHOT)
    s["interval_start"] = np.arange(n) * 10.0
    s["demand_observed"] = rng.uniform(0, 40, n)
    s["demand_estimated"] = rng.uniform(0, 40, n)
    for f in ("x1", "x2", "b1", "b2"):
        s["plan"][f] = rng.integers(-3, 200, n)
    s["plan"]["feasible"] = rng.integers(0, 2, n)
    s["threshold"] = rng.integers(0, 101, n) / 100.0
    for f in ("arrived", "served_light", "served_heavy", "dropped", "late"):
        s[f] = rng.integers(0, 2**40, n, dtype=np.int64).astype(np.uint64)
    s["arrived"][:3] = [0, 2**64 - 1, 10**19]
    s["mean_delivered_quality"] = rng.uniform(0.5, 1.5, n)
    s["has_mean_delivered_quality"] = rng.integers(0, 2, n)
    return s


def random_plan_log(rng, n):
    e = np.zeros(n, abi.PLAN_LOG_ENTRY)
    e["tick"] = np.arange(n) - 2
    e["time"] = np.arange(n) * 10.0
    e["demand_estimated"] = rng.uniform(0, 40, n)
    e["plan"]["threshold"] = rng.integers(0, 101, n) / 100.0
    for f in ("x1", "x2", "b1", "b2"):
        e["plan"][f] = rng.integers(0, 200, n)
    e["plan"]["feasible"] = rng.integers(0, 2, n)
    return e
