"""numpy/ctypes mirror of the POD types in include/ds_gpu.h.

Every struct here is laid out exactly as its C counterpart (numpy
``align=True`` reproduces the C ABI layout); ``_check_layout`` asserts the sizes
against the values the compiled library reports at load time.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

MAX_BATCHES = 64   # DS_MAX_BATCHES
CURVE_BINS = 101   # DS_CURVE_BINS, profiles.hpp:50

# ds_status
OK = 0
ERR_INVALID_ARGUMENT = 1
ERR_DOMAIN = 2
ERR_INVARIANT = 3
ERR_OUT_OF_RANGE = 4
ERR_CUDA = 5
ERR_NO_DEVICE = 6
ERR_CAPACITY = 7
ERR_COMM = 8

# ds_solve_mode
SOLVE = 0
SOLVE_PINNED = 1
SOLVE_FIXED_BATCHES = 2
SOLVE_EVEN_SPLIT = 3
SOLVE_SINGLE_LIGHT = 4
SOLVE_SINGLE_HEAVY = 5

QUEUING_LITTLES_LAW = 0
QUEUING_TWICE_EXEC = 1

CONF_F64 = 0
CONF_F32 = 1

# ds_arrival_mode (ArrivalMode, workload.hpp:26)
ARRIVALS_POISSON = 0
ARRIVALS_UNIFORM = 1

MODEL_PROFILE = np.dtype(
    [("n", "<i4"), ("_pad", "<i4"), ("batch", "<i4", (MAX_BATCHES,)),
     ("latency", "<f8", (MAX_BATCHES,))], align=True)
CURVE = np.dtype([("bin_mass", "<f8", (CURVE_BINS,)), ("total_mass", "<f8")], align=True)
CASCADE = np.dtype(
    [("light", MODEL_PROFILE), ("heavy", MODEL_PROFILE), ("deferral", CURVE),
     ("slo_seconds", "<f8")], align=True)
PROBLEM = np.dtype(
    [("demand_qps", "<f8"), ("overprovision_lambda", "<f8"),
     ("queue_sentinel_seconds", "<f8"), ("light_rate", "<f8"), ("heavy_rate", "<f8"),
     ("light_len", "<i8"), ("heavy_len", "<i8"), ("fixed_threshold", "<f8"),
     ("fixed_b1", "<i4"), ("fixed_b2", "<i4"), ("total_servers", "<i4"), ("queuing", "<i4"),
     ("cascade", "<i4"), ("grid", "<i4"), ("mode", "<i4"), ("_pad", "<i4")], align=True)
PLAN = np.dtype(
    [("x1", "<i4"), ("x2", "<i4"), ("b1", "<i4"), ("b2", "<i4"), ("threshold", "<f8"),
     ("feasible", "<i4"), ("_pad", "<i4")], align=True)
QUERY_MODEL = np.dtype(
    [("easy_fraction", "<f8"), ("quality_gap_scale", "<f8"), ("confidence_fidelity", "<f8"),
     ("noise_sigma", "<f8"), ("seed", "<u8")], align=True)

QUERY = np.dtype(
    [("id", "<u8"), ("arrival", "<f8"), ("deadline", "<f8"), ("quality_light", "<f8"),
     ("quality_heavy", "<f8"), ("confidence", "<f8")], align=True)

# ds_outcome / DS_REC_* (QueryRecord optionals, metrics.hpp:12-36)
OUTCOMES = ("served_light", "served_heavy", "dropped", "late")
REC_LIGHT_START, REC_LIGHT_END, REC_HEAVY_START, REC_HEAVY_END = 0x01, 0x02, 0x04, 0x08
REC_COMPLETION, REC_OUTCOME, REC_DELIVERED_QUALITY = 0x10, 0x20, 0x40
QUERY_RECORD = np.dtype(
    [("id", "<u8"), ("arrival", "<f8"), ("deadline", "<f8"), ("confidence", "<f8"),
     ("quality_light", "<f8"), ("quality_heavy", "<f8"), ("light_start", "<f8"),
     ("light_end", "<f8"), ("heavy_start", "<f8"), ("heavy_end", "<f8"), ("completion", "<f8"),
     ("delivered_quality", "<f8"), ("present", "<u4"), ("outcome", "<i4")], align=True)
INTERVAL_SNAPSHOT = np.dtype(
    [("interval_start", "<f8"), ("demand_observed", "<f8"), ("demand_estimated", "<f8"),
     ("plan", PLAN), ("arrived", "<u8"), ("served_light", "<u8"), ("served_heavy", "<u8"),
     ("dropped", "<u8"), ("late", "<u8"), ("threshold", "<f8"),
     ("mean_delivered_quality", "<f8"), ("has_mean_delivered_quality", "<i4"),
     ("_pad", "<i4")], align=True)
PLAN_LOG_ENTRY = np.dtype(
    [("tick", "<i4"), ("_pad", "<i4"), ("time", "<f8"), ("demand_estimated", "<f8"),
     ("plan", PLAN)], align=True)

assert MODEL_PROFILE.itemsize == 776
assert CURVE.itemsize == 816
assert CASCADE.itemsize == 2376
assert PROBLEM.itemsize == 96
assert PLAN.itemsize == 32
assert QUERY_MODEL.itemsize == 40
assert QUERY.itemsize == 48
assert QUERY_RECORD.itemsize == 104
assert INTERVAL_SNAPSHOT.itemsize == 120
assert PLAN_LOG_ENTRY.itemsize == 56


def ptr(a: np.ndarray | None) -> ctypes.c_void_p:
    """Host pointer of a contiguous numpy array (None -> NULL)."""
    if a is None:
        return ctypes.c_void_p(0)
    if not a.flags["C_CONTIGUOUS"]:
        raise ValueError("array must be C-contiguous")
    return ctypes.c_void_p(a.ctypes.data)


def model_profile(table: dict[int, float]) -> np.ndarray:
    """ModelProfile (profiles.hpp:11-19) from {batch: seconds}."""
    if len(table) > MAX_BATCHES:
        raise ValueError(f"at most {MAX_BATCHES} profiled batch sizes")
    m = np.zeros((), MODEL_PROFILE)
    items = sorted(table.items())
    m["n"] = len(items)
    for i, (b, e) in enumerate(items):
        m["batch"][i] = b
        m["latency"][i] = e
    return m


def plan_tuple(p) -> tuple:
    return (int(p["x1"]), int(p["x2"]), int(p["b1"]), int(p["b2"]), float(p["threshold"]),
            bool(p["feasible"]))


def repo_root() -> str:
    return os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
