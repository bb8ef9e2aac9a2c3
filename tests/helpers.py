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
