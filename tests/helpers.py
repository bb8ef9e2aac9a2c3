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
