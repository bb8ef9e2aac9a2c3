"""TEST INFRASTRUCTURE ONLY -- ctypes loaders for the CPU checkers.

* ``ref()``  -> oracle/_ref/libdsref.so: the UNMODIFIED reference library built
  from /root/reference/proj/src by oracle/Makefile, plus the extern "C" shim
  (oracle/ref_shim.cpp) and the reference test generators
  (oracle/ref_tests_*.cpp). Present only where the reference was compiled
  (here, and on a GPU box that received the built .so in the repo snapshot).
* ``port()`` -> oracle/_build/libds_oracle.so: this repo's plain-C restatement
  (oracle/ds_oracle.c), always buildable.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libdsref.so")
PORT_SO = os.path.join(HERE, "_build", "libds_oracle.so")

_ref = None
_port = None

c_p = ctypes.c_void_p
i32 = ctypes.c_int32
i64 = ctypes.c_int64
u64 = ctypes.c_uint64
f64 = ctypes.c_double


def build_port() -> str:
    if not os.path.exists(PORT_SO) or os.path.getmtime(PORT_SO) < os.path.getmtime(
            os.path.join(HERE, "ds_oracle.c")):
        subprocess.run(["make", "-s", "-C", HERE, "port"], check=True)
    return PORT_SO


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    """The reference library; raises FileNotFoundError if it was never built."""
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(REF_SO)
        lib = ctypes.CDLL(REF_SO)
        lib.dsref_last_error.restype = ctypes.c_char_p
        lib.dsref_plan_batch.argtypes = [c_p, i32, c_p, i32, c_p, c_p, i32, c_p, i32]
        lib.dsref_latency_feasible.argtypes = [c_p, c_p, c_p, ctypes.c_int, ctypes.c_int,
                                               ctypes.c_int, c_p]
        lib.dsref_throughput_feasible.argtypes = [c_p, c_p, c_p, ctypes.c_int, c_p, c_p]
        lib.dsref_deferral_fraction.argtypes = [c_p, f64, c_p]
        lib.dsref_deferral_fraction.restype = f64
        lib.dsref_curve_empty.argtypes = [c_p]
        lib.dsref_curve_uniform_prior.argtypes = [c_p]
        lib.dsref_curve_from_samples.argtypes = [c_p, i64, c_p]
        lib.dsref_curve_observe.argtypes = [c_p, c_p, i64, f64]
        lib.dsref_sample_queries.argtypes = [c_p, u64, i64, f64, c_p, c_p, i32]
        lib.dsref_route_loop.argtypes = [c_p, i64, f64, i32, f64, c_p, c_p, c_p]
        lib.dsref_defers.argtypes = [f64, f64]
        lib.dsref_load_cascade.argtypes = [ctypes.c_char_p, ctypes.c_char_p, c_p]
        lib.dsref_splitmix64.argtypes = [u64]
        lib.dsref_splitmix64.restype = u64
        lib.dsref_generate_arrivals.argtypes = [c_p, i32, f64, u64, i32, c_p, i64]
        lib.dsref_generate_arrivals.restype = i64
        lib.dsref_sample_query_records.argtypes = [c_p, u64, c_p, i64, f64, c_p]
        lib.dsref_write_csv.argtypes = [ctypes.c_char_p, c_p, i64, c_p, i64, c_p, i64]
        lib.dsref_hash_name.argtypes = [ctypes.c_char_p]
        lib.dsref_hash_name.restype = u64
        lib.dsref_stream_raw.argtypes = [u64, ctypes.c_char_p, ctypes.c_int, c_p]
        lib.dsref_stream_raw.restype = None
        lib.dsref_gen_alloc_random.argtypes = [u64, ctypes.c_int, c_p, c_p, c_p, c_p, c_p, c_p]
        lib.dsref_gen_accept_c1.argtypes = [u64, ctypes.c_int, c_p, c_p, c_p, c_p, c_p, c_p,
                                            c_p]
        lib.dsref_gen_c2_recipe.argtypes = [c_p, ctypes.c_int, u64, ctypes.c_int, c_p]
        lib.dsref_policy_run.argtypes = [i32, f64, f64, i32, f64, c_p, i32, c_p, c_p, i32, c_p,
                                         c_p, u64, c_p, c_p, c_p]
        _ref = lib
    return _ref


def port():
    """The plain-C restatement (built on demand)."""
    global _port
    if _port is None:
        lib = ctypes.CDLL(build_port())
        lib.dso_splitmix64.argtypes = [u64]
        lib.dso_splitmix64.restype = u64
        lib.dso_hash_name.argtypes = [ctypes.c_char_p]
        lib.dso_hash_name.restype = u64
        lib.dso_stream_raw.argtypes = [u64, ctypes.c_char_p, ctypes.c_int, c_p]
        lib.dso_sample_query.argtypes = [c_p, u64, c_p, c_p]
        lib.dso_generate_arrivals.argtypes = [c_p, i32, f64, u64, i32, c_p, i64]
        lib.dso_generate_arrivals.restype = i64
        lib.dso_fmt6.argtypes = [c_p, i64, c_p]
        lib.dso_fmt6.restype = None
        for name in ("dso_format_queries_csv", "dso_format_intervals_csv",
                     "dso_format_plans_csv"):
            getattr(lib, name).argtypes = [c_p, i64, c_p, i64]
            getattr(lib, name).restype = i64
        lib.dso_sample_queries.argtypes = [c_p, u64, i64, c_p, c_p, ctypes.c_int]
        lib.dso_bin_of.argtypes = [f64]
        lib.dso_bins_below.argtypes = [f64]
        lib.dso_deferral_fraction.argtypes = [c_p, f64, c_p]
        lib.dso_observe.argtypes = [c_p, f64, f64]
        lib.dso_curve_observe.argtypes = [c_p, c_p, i64, f64]
        lib.dso_route.argtypes = [c_p, i64, c_p, ctypes.c_int, i64, c_p, c_p]
        lib.dso_route.restype = None
        lib.dso_route_loop.argtypes = [c_p, i64, f64, ctypes.c_int, f64, c_p, c_p, c_p]
        lib.dso_solve_one.argtypes = [c_p, c_p, c_p, ctypes.c_int, c_p]
        lib.dso_plan_batch.argtypes = [c_p, i32, c_p, c_p, c_p, c_p, c_p, ctypes.c_int]
        lib.dso_plan_keys.argtypes = [c_p, i32, c_p, c_p, c_p, i32, i32, c_p]
        _port = lib
    return _port
