"""GPU: the sharded hot path through the C ABI's multi-GPU entry points
(include/ds_gpu.h "multi-GPU": ds_route_sharded_device, ds_queue_gather_device,
ds_curve_observe_sharded_device, ds_plan_sharded_device, ds_comm_gather_device).

An N-rank run must return what one GPU returns, i.e. the reference's own
values (tests/golden/*.npz, written by the reference): the global heavy
queues in id order (cluster.cpp:290-306), the deferral curve after the global
observation sequence (profiles.cpp:108-120), and the planner's choices
(allocator.cpp:57-67,91-121).

* NCCL, one rank (the box has one GPU; NCCL refuses two ranks on one device).
* Two and three ranks sharing cuda:0 over the host transport (gloo via
  dist.TorchHostOps): every exchange of the N-rank algorithm runs, with
  ragged shards at N = 3."""
import os
import socket

import numpy as np
import pytest

from tests.helpers import route_digest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _golden(name):
    return dict(np.load(os.path.join(ROOT, "tests", "golden", name + ".npz")))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run_sharded(ctx, comm, root):
    """The whole sharded path on this rank; returns what it checked."""
    import torch

    from paper_2411_15381_b200 import abi, native
    world, rank = comm.size, comm.rank
    out = {}
    g = _golden("latent")
    conf = g["conf0"]
    n = len(conf)
    grid = g["route_grid"]
    nt = len(grid)
    lo, hi = native.Comm.shard_range(n, world, rank)
    m = hi - lo
    dev = torch.device("cuda", 0)
    dconf = torch.from_numpy(np.ascontiguousarray(conf[lo:hi])).to(dev)
    thr = torch.from_numpy(grid).to(dev)
    heavy = torch.zeros(nt * max(m, 1), dtype=torch.int64, device=dev)
    counts = torch.zeros(nt, dtype=torch.int64, device=dev)
    offs = torch.zeros(nt, dtype=torch.int64, device=dev)
    tot = torch.zeros(nt, dtype=torch.int64, device=dev)
    st = ctx.stream
    torch.cuda.synchronize()   # inputs made on torch's stream, used on the context's
    # route + routed-count all-gather
    comm.route(dconf.data_ptr(), abi.CONF_F64, m, thr.data_ptr(), nt, lo, heavy.data_ptr(),
               counts.data_ptr(), offs.data_ptr(), tot.data_ptr(), stream=st)
    ctx.synchronize()
    want_counts = g["route_counts"]
    out["totals"] = bool(np.array_equal(tot.cpu().numpy(), want_counts))
    below = np.array([(conf[:lo] < t).sum() for t in grid])
    out["offsets"] = bool(np.array_equal(offs.cpu().numpy(), below))
    # global heavy queues at the root
    is_root = rank == root
    gq = torch.full((nt * n,), -1, dtype=torch.int64, device=dev) if is_root else None
    gc = torch.zeros(nt, dtype=torch.int64, device=dev) if is_root else None
    torch.cuda.synchronize()
    comm.gather_queues(root, heavy.data_ptr(), m, counts.data_ptr(), nt,
                       gq.data_ptr() if is_root else 0, n, gc.data_ptr() if is_root else 0,
                       stream=st)
    ctx.synchronize()
    if is_root:
        gcn = gc.cpu().numpy()
        q = gq.cpu().numpy().reshape(nt, n)
        out["queue_counts"] = bool(np.array_equal(gcn, want_counts))
        out["queue_digests"] = all(route_digest(q[k, :gcn[k]]) == g["route_digest"][k]
                                   for k in range(nt))
    # the global curve on every rank
    cur = torch.from_numpy(g["prior"].reshape(1).view(np.uint8).copy()).to(dev)
    sizes = [native.Comm.shard_range(n, world, r)[1] - native.Comm.shard_range(n, world, r)[0]
             for r in range(world)]
    torch.cuda.synchronize()
    comm.curve_observe(cur.data_ptr(), dconf.data_ptr(), abi.CONF_F64, sizes, 0.999, stream=st)
    ctx.synchronize()
    out["curve_bits"] = cur.cpu().numpy().tobytes() == g["curve_after_0999"].tobytes()
    # planner, one batch sharded by threshold range, keys MIN-all-reduced
    c4 = _golden("config4")
    pro, cas, gv, go = c4["problems"], c4["cascades"], c4["grid_values"], c4["grid_offsets"]
    G = int(max(go[1:] - go[:-1]))
    t_lo, t_hi = native.Comm.shard_range(G, world, rank)

    def dbytes(a):
        return torch.from_numpy(np.ascontiguousarray(a).view(np.uint8).copy()).to(dev)
    dp, dc, dg, do = dbytes(pro), dbytes(cas), dbytes(gv), dbytes(go)
    plans = torch.zeros(len(pro) * abi.PLAN.itemsize, dtype=torch.uint8, device=dev)
    torch.cuda.synchronize()
    comm.plan(dp.data_ptr(), len(pro), dc.data_ptr(), len(cas), dg.data_ptr(), do.data_ptr(),
              len(go) - 1, t_lo, t_hi, plans.data_ptr(), stream=st)
    ctx.synchronize()
    out["plans_t_sharded"] = plans.cpu().numpy().tobytes() == c4["want_solve"].tobytes()
    # planner, problems sharded by index, plans gathered at the root
    plo, phi = native.Comm.shard_range(len(pro), world, rank)
    mine = torch.zeros(max(phi - plo, 1) * abi.PLAN.itemsize, dtype=torch.uint8, device=dev)
    native.check(native.lib().ds_plan_batch_device(
        ctx.handle, native.c_p(dp.data_ptr() + plo * abi.PROBLEM.itemsize), phi - plo,
        native.c_p(dc.data_ptr()), len(cas), native.c_p(dg.data_ptr()),
        native.c_p(do.data_ptr()), len(go) - 1, native.c_p(mine.data_ptr()), native.c_p(st)))
    allp = torch.zeros(len(pro) * abi.PLAN.itemsize, dtype=torch.uint8, device=dev)
    torch.cuda.synchronize()
    total = comm.gather(root, mine.data_ptr(), (phi - plo) * abi.PLAN.itemsize,
                        allp.data_ptr() if is_root else 0, allp.numel() if is_root else 0,
                        stream=st)
    if is_root:
        out["plans_gathered"] = (total == allp.numel() and
                                 allp.cpu().numpy().tobytes() == c4["want_solve"].tobytes())
    return out


def test_nccl_one_rank_sharded_path_matches_reference():
    from paper_2411_15381_b200 import native
    ctx = native.Context(0)
    comm = native.Comm.nccl(ctx, 1, 0, native.Comm.unique_id())
    assert (comm.rank, comm.size) == (0, 1)
    out = _run_sharded(ctx, comm, 0)
    comm.close()
    ctx.close()
    assert out and all(out.values()), out


def _run_edges(ctx, comm, root, n):
    """Ragged and empty shards: n confidences over comm.size ranks (n < size
    leaves ranks with nothing; n = 0 leaves all of them empty). Every rank's
    view must equal one GPU's over the whole sequence."""
    import torch

    from paper_2411_15381_b200 import abi, native, workloads
    world, rank = comm.size, comm.rank
    conf = np.array([0.7, 0.3, 0.5, 0.05, 0.95][:n], np.float64)
    grid = np.array([0.0, 0.3, 0.5, 1.0], np.float64)
    nt = len(grid)
    lo, hi = native.Comm.shard_range(n, world, rank)
    m = hi - lo
    dev = torch.device("cuda", 0)
    dconf = torch.from_numpy(np.concatenate([conf[lo:hi], [0.0]])).to(dev)   # never empty
    thr = torch.from_numpy(grid).to(dev)
    heavy = torch.full((nt * max(m, 1),), -7, dtype=torch.int64, device=dev)
    counts = torch.full((nt,), -7, dtype=torch.int64, device=dev)
    offs = torch.full((nt,), -7, dtype=torch.int64, device=dev)
    tot = torch.full((nt,), -7, dtype=torch.int64, device=dev)
    st = ctx.stream
    torch.cuda.synchronize()
    comm.route(dconf.data_ptr(), abi.CONF_F64, m, thr.data_ptr(), nt, lo, heavy.data_ptr(),
               counts.data_ptr(), offs.data_ptr(), tot.data_ptr(), stream=st)
    ctx.synchronize()
    out = {}
    out["counts"] = bool(np.array_equal(counts.cpu().numpy(),
                                        [(conf[lo:hi] < t).sum() for t in grid]))
    out["totals"] = bool(np.array_equal(tot.cpu().numpy(), [(conf < t).sum() for t in grid]))
    out["offsets"] = bool(np.array_equal(offs.cpu().numpy(), [(conf[:lo] < t).sum() for t in grid]))
    is_root = rank == root
    gq = torch.full((nt * max(n, 1),), -1, dtype=torch.int64, device=dev) if is_root else None
    gc = torch.full((nt,), -1, dtype=torch.int64, device=dev) if is_root else None
    torch.cuda.synchronize()
    comm.gather_queues(root, heavy.data_ptr(), m, counts.data_ptr(), nt,
                       gq.data_ptr() if is_root else 0, n, gc.data_ptr() if is_root else 0,
                       stream=st)
    ctx.synchronize()
    if is_root:
        gcn = gc.cpu().numpy()
        q = gq.cpu().numpy()
        out["queue"] = bool(np.array_equal(gcn, [(conf < t).sum() for t in grid])) and all(
            np.array_equal(q[k * n:k * n + gcn[k]], np.flatnonzero(conf < grid[k]))
            for k in range(nt))
    prior = workloads.uniform_prior()
    cur = torch.from_numpy(prior.reshape(1).view(np.uint8).copy()).to(dev)
    sizes = [native.Comm.shard_range(n, world, r)[1] - native.Comm.shard_range(n, world, r)[0]
             for r in range(world)]
    torch.cuda.synchronize()
    comm.curve_observe(cur.data_ptr(), dconf.data_ptr(), abi.CONF_F64, sizes, 0.999, stream=st)
    ctx.synchronize()
    want = ctx.curve_observe(prior, conf, 0.999) if n else prior
    out["curve_bits"] = cur.cpu().numpy().tobytes() == np.asarray(want).tobytes()
    # byte gather with empty contributions
    mine = torch.arange(8 * m, dtype=torch.uint8, device=dev) + 8 * lo
    allb = torch.zeros(8 * max(n, 1), dtype=torch.uint8, device=dev)
    torch.cuda.synchronize()
    total = comm.gather(root, mine.data_ptr() if m else 0, 8 * m,
                        allb.data_ptr() if is_root else 0, allb.numel() if is_root else 0,
                        stream=st)
    ctx.synchronize()
    if is_root:
        out["gather"] = total == 8 * n and bool(
            np.array_equal(allb.cpu().numpy()[:8 * n], np.arange(8 * n, dtype=np.uint8)))
    return out


def _host_worker(rank, world, port, root, q, edge_n=None):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    from paper_2411_15381_b200 import dist as ddist
    from paper_2411_15381_b200 import native
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        ctx = native.Context(0)
        comm = native.Comm.host(ctx, world, rank, ddist.TorchHostOps())
        out = _run_sharded(ctx, comm, root) if edge_n is None else _run_edges(ctx, comm, root, edge_n)
        comm.close()
        ctx.close()
        q.put((rank, out, None))
    except Exception as e:   # report, do not hang the parent
        import traceback
        q.put((rank, {}, traceback.format_exc() + str(e)))
    finally:
        dist.destroy_process_group()


def _spawn(world, root, edge_n=None):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_host_worker, args=(r, world, port, root, q, edge_n))
             for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, out, err = q.get(timeout=300)
        assert err is None, err
        res[r] = out
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("world,root", [(2, 0), (3, 2)])
def test_host_transport_ranks_on_one_gpu_match_reference(world, root):
    res = _spawn(world, root)
    for r, out in res.items():
        assert all(out.values()), (r, out)
    assert "queue_digests" in res[root] and "plans_gathered" in res[root]


@pytest.mark.parametrize("world,root,n", [(3, 1, 2), (3, 0, 5), (2, 1, 0), (4, 3, 1)])
def test_host_transport_empty_and_ragged_shards(world, root, n):
    """Ranks with no queries still take part in every exchange: counts,
    global offsets and queues, the global curve and byte gathers equal one
    GPU's results."""
    res = _spawn(world, root, edge_n=n)
    for r, out in res.items():
        assert out and all(out.values()), (r, out)
    assert "queue" in res[root] and "gather" in res[root]


def test_cpp_multi_gpu_driver():
    """integration/ds_multi: the C++ host drives every visible GPU through the
    C ABI (ncclCommInitAll, one thread per GPU) and checks the G-GPU global
    queues, counts and curve bits against one GPU doing all the work."""
    import json
    import subprocess
    exe = os.path.join(ROOT, "integration", "_bin", "ds_multi")
    assert os.path.exists(exe), "build with make -C integration (__graft_entry__.build)"
    r = subprocess.run([exe, "--images-per-gpu", "1200", "--queries", "30000", "--steps", "2",
                        "--warmup", "1"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["gpus"] >= 1
    assert all(line["check"].values()), line
