"""CPU suite: the C-ABI library builds, loads, and exports every symbol that
include/ds_gpu.h declares (no compute calls: there is no GPU here)."""
import ctypes
import os
import re

import numpy as np

from paper_2411_15381_b200 import abi, native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "ds_gpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ds_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = native.lib()
    names = declared_symbols()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    bound = {s[0] for s in native.SIGNATURES}
    assert set(names) == bound, set(names) ^ bound


def test_version_and_no_device_error():
    lib = native.lib()
    assert b"sm_100a" in lib.ds_version()
    h = ctypes.c_void_p()
    st = lib.ds_ctx_create(0, ctypes.byref(h))
    # no GPU in this container: must fail loudly with DS_ERR_NO_DEVICE, never fall back
    import torch
    if not torch.cuda.is_available():
        assert st == abi.ERR_NO_DEVICE
        assert b"no CUDA device" in lib.ds_last_error()


def test_struct_layouts_match_header():
    assert abi.PROBLEM.itemsize == 96 and abi.CASCADE.itemsize == 2376
    assert abi.PLAN.itemsize == 32 and abi.CURVE.itemsize == 816


def test_host_validation_runs_without_gpu(golden):
    """ds_plan_validate is host-only: the reference's checks, in its order."""
    lib = native.lib()
    g = golden("accept_c1")
    pro = np.ascontiguousarray(g["problems"])
    cas = np.ascontiguousarray(g["cascades"])
    gv = np.ascontiguousarray(g["grid_values"])
    go = np.ascontiguousarray(g["grid_offsets"])
    assert lib.ds_plan_validate(abi.ptr(pro), len(pro), abi.ptr(cas), len(cas), abi.ptr(gv),
                                abi.ptr(go), len(go) - 1) == abi.OK
    bad = pro[:1].copy()
    bad["total_servers"] = 0
    assert lib.ds_plan_validate(abi.ptr(bad), 1, abi.ptr(cas), len(cas), abi.ptr(gv),
                                abi.ptr(go), len(go) - 1) == abi.ERR_DOMAIN
    bad = pro[:1].copy()
    bad["cascade"] = 10_000
    assert lib.ds_plan_validate(abi.ptr(bad), 1, abi.ptr(cas), len(cas), abi.ptr(gv),
                                abi.ptr(go), len(go) - 1) == abi.ERR_INVALID_ARGUMENT
    g2 = np.array([0.5, 1.0])
    o2 = np.array([0, 2], np.int32)
    bad = pro[:1].copy()
    bad["grid"] = 0
    assert lib.ds_plan_validate(abi.ptr(bad), 1, abi.ptr(cas), len(cas), abi.ptr(g2),
                                abi.ptr(o2), 1) == abi.ERR_INVARIANT
    bad["mode"] = abi.SOLVE_FIXED_BATCHES
    bad["fixed_b1"] = 3
    g3 = np.array([0.0, 1.0])
    assert lib.ds_plan_validate(abi.ptr(bad), 1, abi.ptr(cas), len(cas), abi.ptr(g3),
                                abi.ptr(o2), 1) == abi.ERR_OUT_OF_RANGE
