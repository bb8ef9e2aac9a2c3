"""CPU suite: the multi-GPU host logic over world_size-2 gloo process groups.

Each rank routes its contiguous id shard (here with the C oracle, as test
infrastructure standing in for K2 on a GPU), all-gathers its routed counts,
and places its ordered ids at the exclusive-scan offset; the assembled global
heavy queues must equal single-rank routing of all queries (the reference's
id order, cluster.cpp:290-306). Planner sharding likewise reproduces the
single-rank plans."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import lib
from paper_2411_15381_b200 import abi, dist as ddist, workloads


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _route_worker(rank, world, port, conf, thr, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = len(conf)
        lo, hi = ddist.shard_range(n, world, rank)
        mine = np.ascontiguousarray(conf[lo:hi])
        nt = len(thr)
        idx = np.zeros(nt * max(hi - lo, 1), np.int64)
        cnt = np.zeros(nt, np.int64)
        lib.port().dso_route(abi.ptr(mine), hi - lo, abi.ptr(thr), nt, lo, abi.ptr(idx),
                             abi.ptr(cnt))
        g = ddist.gather_counts(torch.from_numpy(cnt)).numpy()
        offs = ddist.exclusive_offsets(g)[rank]
        total = g.sum(0)
        # every rank writes its block into its own copy of the global queues;
        # a sum-reduce assembles them (blocks are disjoint)
        glob = np.zeros((nt, n), np.int64)
        for k in range(nt):
            glob[k, offs[k]:offs[k] + cnt[k]] = idx[k * (hi - lo): k * (hi - lo) + cnt[k]] + 1
        t = torch.from_numpy(glob)
        dist.all_reduce(t)
        if rank == 0:
            q.put((total, t.numpy() - 1))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_routing_equals_single_rank_order(world):
    rng = np.random.default_rng(world)
    conf = rng.random(10_007)
    conf[::9] = 0.5
    thr = workloads.make_grid(0.05)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_route_worker, args=(r, world, port, conf, thr, q))
             for r in range(world)]
    for p in procs:
        p.start()
    total, glob = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n = len(conf)
    idx = np.zeros(len(thr) * n, np.int64)
    cnt = np.zeros(len(thr), np.int64)
    lib.port().dso_route(abi.ptr(conf), n, abi.ptr(thr), len(thr), 0, abi.ptr(idx), abi.ptr(cnt))
    assert np.array_equal(total, cnt)
    for k in range(len(thr)):
        assert np.array_equal(glob[k, :cnt[k]], idx[k * n: k * n + cnt[k]])


def _plan_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = dict(np.load(os.path.join(os.path.dirname(__file__), "golden", "config4.npz")))
        pro = g["problems"]
        lo, hi = ddist.shard_range(len(pro), world, rank)
        mine = np.ascontiguousarray(pro[lo:hi])
        out = np.zeros(hi - lo, abi.PLAN)
        st = np.zeros(hi - lo, np.int32)
        lib.port().dso_plan_batch(abi.ptr(mine), hi - lo, abi.ptr(g["cascades"]),
                                  abi.ptr(g["grid_values"]), abi.ptr(g["grid_offsets"]),
                                  abi.ptr(out), abi.ptr(st), 2)
        parts = [None] * world
        dist.all_gather_object(parts, out.tobytes())
        if rank == 0:
            q.put(b"".join(parts))
    finally:
        dist.destroy_process_group()


def test_sharded_planner_equals_reference_plans():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_plan_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = np.frombuffer(q.get(timeout=120), abi.PLAN)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = dict(np.load(os.path.join(os.path.dirname(__file__), "golden", "config4.npz")))
    assert got.tobytes() == g["want_solve"].tobytes()


def test_shard_range_and_offsets():
    assert [ddist.shard_range(10, 3, r) for r in range(3)] == [(0, 3), (3, 6), (6, 10)]
    offs = ddist.exclusive_offsets(np.array([[2, 0], [3, 1], [1, 4]]))
    assert offs.tolist() == [[0, 0], [2, 0], [5, 1]]
    with pytest.raises(ValueError):
        ddist.shard_range(5, 2, 2)


def test_curve_shards_combine_exactly_at_decay_one():
    """S7 with decay 1: integer bin counts add across shards exactly (8(e))."""
    rng = np.random.default_rng(0)
    conf = rng.random(5000)
    whole = np.zeros((), abi.CURVE)
    lib.port().dso_curve_observe(abi.ptr(whole), abi.ptr(conf), len(conf), 1.0)
    parts = []
    for r in range(2):
        lo, hi = ddist.shard_range(len(conf), 2, r)
        c = np.zeros((), abi.CURVE)
        s = np.ascontiguousarray(conf[lo:hi])
        lib.port().dso_curve_observe(abi.ptr(c), abi.ptr(s), len(s), 1.0)
        parts.append(c)
    assert np.array_equal(parts[0]["bin_mass"] + parts[1]["bin_mass"], whole["bin_mass"])


def _decode_key(key, p, cas, gv, go):
    """Packed selection key -> (x1, x2, b1, b2, threshold) (ds_plan_keys layout)."""
    key = int(key)
    c = cas[p["cascade"]]
    G = int(go[p["grid"] + 1] - go[p["grid"]])
    t_idx = G - 1 - (key >> 40)
    x1 = key & 0xFFF
    tot = (key >> 28) & 0xFFF
    b1 = int(c["light"]["batch"][255 - ((key >> 20) & 0xFF)])
    b2 = int(c["heavy"]["batch"][255 - ((key >> 12) & 0xFF)])
    return x1, tot - x1, b1, b2, float(gv[go[p["grid"]] + t_idx])


def _tplan_worker(rank, world, port, name, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = dict(np.load(os.path.join(os.path.dirname(__file__), "golden", f"{name}.npz")))
        pro, cas, gv, go = g["problems"], g["cascades"], g["grid_values"], g["grid_offsets"]
        G = int(max(go[1:] - go[:-1]))

        def keys_fn(t_lo, t_hi):
            k = np.zeros(len(pro), np.uint64)
            assert lib.port().dso_plan_keys(abi.ptr(pro), len(pro), abi.ptr(cas), abi.ptr(gv),
                                            abi.ptr(go), t_lo, t_hi, abi.ptr(k)) == 0
            return k
        got = ddist.plan_t_sharded(keys_fn, lambda k: k, G)
        if rank == 0:
            q.put((got, keys_fn(0, G)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,name", [(2, "config4"), (3, "wide_random"), (2, "alloc_random_2024")])
def test_t_sharded_planner_argmin_equals_reference(world, name):
    """Threshold-range sharding: per-rank keys of grid slices,
    MIN all-reduce -> the full search's key, which decodes to the reference's
    plan (golden sets written by the reference itself)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_tplan_worker, args=(r, world, port, name, q))
             for r in range(world)]
    for p in procs:
        p.start()
    got, full = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert np.array_equal(got, full)
    g = dict(np.load(os.path.join(os.path.dirname(__file__), "golden", f"{name}.npz")))
    pro, cas, gv, go = g["problems"], g["cascades"], g["grid_values"], g["grid_offsets"]
    want = g["want_solve"] if "want_solve" in g else g["want"]
    found = 0
    for i in np.flatnonzero(got != ddist.KEY_NONE):
        x1, x2, b1, b2, t = _decode_key(got[i], pro[i], cas, gv, go)
        w = want[i]
        assert (x1, x2, b1, b2, t) == (w["x1"], w["x2"], w["b1"], w["b2"], w["threshold"]), i
        assert w["feasible"] == 1
        found += 1
    grid_mode = np.isin(pro["mode"], [abi.SOLVE, abi.SOLVE_FIXED_BATCHES])
    assert np.array_equal(got != ddist.KEY_NONE, grid_mode & (want["feasible"] == 1))
    assert found >= 5
    # keys in int64 for the reduction keep the unsigned order
    # (keys at and above 2^63 arise on grids longer than 2^23 points)
    k = np.array([0, 5, 2**62, 2**63 - 1, 2**63, 2**63 + 7, 2**64 - 2, int(ddist.KEY_NONE)],
                 np.uint64)
    assert np.array_equal(ddist.keys_from_i64(ddist.keys_to_i64(k)), k)
    assert list(np.argsort(ddist.keys_to_i64(k))) == list(range(len(k)))
    assert ddist.keys_to_i64(k)[-1] == np.iinfo(np.int64).max


def _host_ops_worker(rank, world, port, q):
    """dist.TorchHostOps -- the ds_comm_ops host transport of native.Comm.host --
    over gloo: the byte/key semantics the C library relies on."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ops = ddist.TorchHostOps()
        mine = np.arange(6, dtype=np.uint8) + 10 * rank
        ag = ops.allgather(mine)
        keys = np.array([2**64 - 1, 2**63 + rank, 5 + (world - rank), 2**62 * (rank + 1) % 2**64,
                         2**63 - 1 - rank], np.uint64)
        mn = ops.allreduce_min_u64(keys.copy())
        sizes = [3 * r for r in range(world)]          # rank 0 sends nothing
        send = np.full(sizes[rank], rank + 1, np.uint8)
        gv = ops.gatherv(send, sizes, world - 1)
        q.put((rank, ag, mn, gv))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_torch_host_ops(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_host_ops_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, ag, mn, gv = q.get(timeout=120)
        res[r] = (ag, mn, gv)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want_ag = np.concatenate([np.arange(6, dtype=np.uint8) + 10 * r for r in range(world)])
    keys = [np.array([2**64 - 1, 2**63 + r, 5 + (world - r), 2**62 * (r + 1) % 2**64,
                      2**63 - 1 - r], np.uint64) for r in range(world)]
    want_mn = np.minimum.reduce(keys)
    want_gv = np.concatenate([np.full(3 * r, r + 1, np.uint8) for r in range(world)])
    for r in range(world):
        ag, mn, gv = res[r]
        assert np.array_equal(ag, want_ag)
        assert np.array_equal(mn, want_mn) and mn.dtype == np.uint64
        if r == world - 1:
            assert np.array_equal(gv, want_gv)
        else:
            assert gv is None
