"""Host time per call (no synchronisation inside the timed span) of the
device-pointer entry points on their bench workloads: what a caller's thread
spends enqueuing one call. Values well above a few microseconds point at
per-call driver queries or allocations on the launch path.

    python tools/host_overhead.py
"""
import ctypes
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2411_15381_b200 import abi, native, workloads  # noqa: E402

ctx = native.Context(0)
L = native.lib()
sp = native.c_p(ctx.stream)
P = native.c_p


def host_us(fn, reps=20):
    for _ in range(3):
        fn()
    ctx.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
        ctx.synchronize()
    return float(np.median(ts) * 1e6)


disc = native.Discriminator(ctx, 2024)
n = 5000
img = torch.empty(n * 512 * 512 * 3, dtype=torch.uint8, device="cuda")
L.ds_synth_images_device(ctx.handle, 1, 0, n, 512, 512, P(img.data_ptr()), sp)
conf = torch.empty(n, dtype=torch.float32, device="cuda")
grid = torch.tensor(workloads.make_grid(0.01), dtype=torch.float64, device="cuda")
heavy = torch.empty(101 * n, dtype=torch.int64, device="cuda")
counts = torch.empty(101, dtype=torch.int64, device="cuda")
curve = torch.from_numpy(workloads.uniform_prior().reshape(1).view(np.uint8).copy()).cuda()
res = {}
res["disc score 5K"] = host_us(lambda: disc.score_device(img.data_ptr(), n, 512, 512, conf.data_ptr(), ctx.stream), 5)
res["route 5K x101"] = host_us(lambda: native.check(L.ds_route_device(
    ctx.handle, P(conf.data_ptr()), abi.CONF_F32, n, P(grid.data_ptr()), 101, 0, P(heavy.data_ptr()),
    P(counts.data_ptr()), sp)))
res["curve 5K"] = host_us(lambda: native.check(L.ds_curve_observe_device(
    ctx.handle, P(curve.data_ptr()), P(conf.data_ptr()), abi.CONF_F32, n, 0.999, sp)))
pro, cas, gv, go, _ = bench.planner_inputs()
d_pro = torch.from_numpy(pro.view(np.uint8).copy()).cuda()
d_cas = torch.from_numpy(cas.view(np.uint8).copy()).cuda()
d_gv = torch.from_numpy(np.ascontiguousarray(gv)).cuda()
d_go = torch.from_numpy(np.ascontiguousarray(go)).cuda()
d_out = torch.empty(len(pro) * abi.PLAN.itemsize, dtype=torch.uint8, device="cuda")
res["plan 4096"] = host_us(lambda: native.check(L.ds_plan_batch_device(
    ctx.handle, P(d_pro.data_ptr()), len(pro), P(d_cas.data_ptr()), len(cas), P(d_gv.data_ptr()),
    P(d_go.data_ptr()), 1, P(d_out.data_ptr()), sp)))
m = workloads.query_model()
lc = torch.empty(1_000_000, dtype=torch.float64, device="cuda")
res["latent 1M"] = host_us(lambda: native.check(L.ds_score_latent_device(
    ctx.handle, abi.ptr(m), 0, 1_000_000, P(lc.data_ptr()), P(0), sp)))
for k, v in res.items():
    print(f"{k:16s} {v:8.1f} us host per call")

# one light batch of 32 (config 1), the chained per-call path
thr1 = torch.full((1,), 0.5, dtype=torch.float64, device="cuda")
heavy1 = torch.empty(32, dtype=torch.int64, device="cuda")
count1 = torch.empty(1, dtype=torch.int64, device="cuda")
conf1 = torch.empty(32, dtype=torch.float32, device="cuda")
print(f"{'batch of 32':16s} {host_us(lambda: native.check(L.ds_disc_batch_complete_device(disc.handle, P(img.data_ptr()), 32, 512, 512, P(conf1.data_ptr()), P(curve.data_ptr()), 0.999, P(thr1.data_ptr()), 1, 0, P(heavy1.data_ptr()), P(count1.data_ptr()), sp)), 50):8.1f} us host per call")
