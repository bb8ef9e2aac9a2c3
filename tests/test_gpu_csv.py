"""GPU parity: K9 CSV formatting, byte-identical to the
reference's write_csv (tests/golden/csv.npz holds the bytes the reference
wrote, oracle/make_golden.py) and to the C restatement (oracle/ds_oracle.c,
pinned to those bytes) on fresh rows."""
import ctypes

import numpy as np
import pytest

from oracle import lib
from paper_2411_15381_b200 import abi, native
from paper_2411_15381_b200.api import CapacityError, default_context, fmt6, write_csv
from tests import helpers

pytestmark = pytest.mark.gpu

P = abi.ptr


@pytest.fixture(scope="module")
def ctx():
    return default_context()


def port_csv(name, rows):
    fn = getattr(lib.port(), f"dso_format_{name}_csv")
    n = fn(P(rows), len(rows), None, 0)
    out = np.zeros(max(n, 1), np.uint8)
    fn(P(rows), len(rows), P(out), n)
    return out[:n].tobytes()


def port_g6(vals):
    vals = np.ascontiguousarray(vals, np.float64)
    out = np.zeros(len(vals), "S16")
    lib.port().dso_fmt6(P(vals), len(vals), P(out))
    return out


def test_csv_matches_reference_goldens(ctx, golden):
    g = golden("csv")
    assert ctx.format_queries_csv(g["records"]) == g["queries_csv"].tobytes()
    assert ctx.format_intervals_csv(g["intervals"]) == g["intervals_csv"].tobytes()
    assert ctx.format_plans_csv(g["plans"]) == g["plans_csv"].tobytes()
    assert np.array_equal(ctx.format_g6(g["g6_values"]), g["g6_text"])


def test_g6_matches_printf_on_many_doubles(ctx):
    rng = np.random.default_rng(11)
    vals = np.concatenate([helpers.special_doubles(), helpers.random_doubles(rng, 3_000_000)])
    got = ctx.format_g6(vals)
    want = port_g6(vals)
    bad = np.flatnonzero(got != want)
    assert len(bad) == 0, [(vals[i], got[i], want[i]) for i in bad[:5]]


def test_large_query_csv_matches_port(ctx):
    rng = np.random.default_rng(12)
    q = helpers.random_query_records(rng, 1_000_000)
    got = ctx.format_queries_csv(q)
    assert got == port_csv("queries", q)
    assert got.count(b"\n") == len(q) + 1


def test_empty_tables(ctx):
    assert ctx.format_queries_csv(np.zeros(0, abi.QUERY_RECORD)).count(b"\n") == 1
    assert ctx.format_plans_csv(np.zeros(0, abi.PLAN_LOG_ENTRY)) == port_csv(
        "plans", np.zeros(0, abi.PLAN_LOG_ENTRY))


def test_reference_api_mirror(tmp_path, golden):
    g = golden("csv")
    write_csv(str(tmp_path), g["intervals"], g["records"], g["plans"])
    for name in ("queries", "intervals", "plans"):
        assert (tmp_path / f"{name}.csv").read_bytes() == g[f"{name}_csv"].tobytes()
    assert fmt6(0.1) == "0.1" and fmt6(1234565.0) == "1.23456e+06" and fmt6(-0.0) == "-0"


def test_capacity_and_device_entry(ctx, golden):
    torch = pytest.importorskip("torch")
    g = golden("csv")
    rec = np.ascontiguousarray(g["records"])
    want = g["queries_csv"].tobytes()
    L = native.lib()
    n = native.i64(0)
    small = np.zeros(100, np.uint8)
    with pytest.raises(CapacityError):
        native.check(L.ds_format_queries_csv(ctx.handle, P(rec), len(rec), P(small), 100,
                                             ctypes.byref(n)))
    assert n.value == len(want)
    drec = torch.from_numpy(rec.view(np.uint8).copy()).cuda()
    dout = torch.zeros(len(want) + 64, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    native.check(L.ds_format_queries_csv_device(ctx.handle, ctypes.c_void_p(drec.data_ptr()),
                                                len(rec), ctypes.c_void_p(dout.data_ptr()),
                                                dout.numel(), ctypes.byref(n),
                                                ctypes.c_void_p(stream)))
    torch.cuda.synchronize()
    assert n.value == len(want)
    assert dout[:n.value].cpu().numpy().tobytes() == want
    assert int(dout[n.value:].sum()) == 0


@pytest.mark.parametrize("shift", [1, 2, 3, 5])
def test_device_entry_misaligned_out_and_short_capacity(ctx, shift):
    """Any output alignment gives the same bytes and touches nothing outside
    the file; a buffer shorter than the file gets DS_ERR_CAPACITY with the full
    size reported and is left untouched. Many blocks, rows of every length
    class (random records, NaN/inf/huge/tiny values)."""
    torch = pytest.importorskip("torch")
    rec = helpers.random_query_records(np.random.default_rng(40 + shift), 70_001)
    want = port_csv("queries", rec)
    L = native.lib()
    n = native.i64(0)
    drec = torch.from_numpy(rec.view(np.uint8).copy()).cuda()
    stream = torch.cuda.current_stream().cuda_stream
    dout = torch.zeros(len(want) + 64, dtype=torch.uint8, device="cuda")
    native.check(L.ds_format_queries_csv_device(
        ctx.handle, ctypes.c_void_p(drec.data_ptr()), len(rec),
        ctypes.c_void_p(dout.data_ptr() + shift), len(want), ctypes.byref(n),
        ctypes.c_void_p(stream)))
    torch.cuda.synchronize()
    got = dout.cpu().numpy()
    assert n.value == len(want)
    assert got[shift:shift + len(want)].tobytes() == want
    assert int(got[:shift].sum()) == 0 and int(got[shift + len(want):].sum()) == 0
    cap = len(want) // 2 + shift
    dout.zero_()
    with pytest.raises(CapacityError):
        native.check(L.ds_format_queries_csv_device(
            ctx.handle, ctypes.c_void_p(drec.data_ptr()), len(rec),
            ctypes.c_void_p(dout.data_ptr()), cap, ctypes.byref(n), ctypes.c_void_p(stream)))
    torch.cuda.synchronize()
    assert n.value == len(want)
    assert int(dout.sum()) == 0


def test_longest_rows(ctx):
    """Interval rows at their maximum length (every integer at its widest,
    every real at 13 characters): 225 bytes, inside the kernel's row buffer."""
    n = 3000
    s = np.zeros(n, abi.INTERVAL_SNAPSHOT)
    for f in ("interval_start", "demand_observed", "demand_estimated", "threshold",
              "mean_delivered_quality"):
        s[f] = -1.23456e-300
    for f in ("x1", "x2", "b1", "b2"):
        s["plan"][f] = np.iinfo(np.int32).min
    for f in ("arrived", "served_light", "served_heavy", "dropped", "late"):
        s[f] = np.iinfo(np.uint64).max
    s["has_mean_delivered_quality"] = 1
    want = port_csv("intervals", s)
    assert max(len(r) for r in want.split(b"\n")) + 1 == 225
    assert ctx.format_intervals_csv(s) == want
