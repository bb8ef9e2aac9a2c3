"""Times K2 (ds_route_device) on the bench shapes and checks the lists against
numpy: 1M f64 at t = 0.5 (the latent leg), 1M f32 at t = 0.5 (config 5),
5K f32 at the 101 grid thresholds (config 2). CUDA events, 50 launches each.

    python tools/route_speed.py [--ncu]   (--ncu: 3 launches of each, for a capture)
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2411_15381_b200 import abi, native, workloads  # noqa: E402

ncu = "--ncu" in sys.argv
reps = 3 if ncu else 50
ctx = native.Context(0)
L = native.lib()
st = torch.cuda.ExternalStream(ctx.stream)
rng = np.random.default_rng(1)
cases = [("1M f64 t=0.5", rng.random(1_000_000), [0.5]),
         ("1M f32 t=0.5", rng.random(1_000_000).astype(np.float32), [0.5]),
         ("5K f32 x101", rng.random(5000).astype(np.float32), list(workloads.make_grid(0.01))),
         ("16M f64 t=0.5", rng.random(16_000_000), [0.5])]
for name, conf, thr in cases:
    n, nt = len(conf), len(thr)
    dt = abi.CONF_F64 if conf.dtype == np.float64 else abi.CONF_F32
    dc = torch.from_numpy(conf).cuda()
    dthr = torch.tensor(thr, dtype=torch.float64, device="cuda")
    heavy = torch.empty(n * nt, dtype=torch.int64, device="cuda")
    cnt = torch.empty(nt, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()

    def run():
        native.check(L.ds_route_device(ctx.handle, native.c_p(dc.data_ptr()), dt, n,
                                       native.c_p(dthr.data_ptr()), nt, 7, native.c_p(heavy.data_ptr()),
                                       native.c_p(cnt.data_ptr()), native.c_p(ctx.stream)))
    run()
    ctx.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        a.record(st)
        for _ in range(reps):
            run()
        b.record(st)
    torch.cuda.synchronize()
    ms_eager = a.elapsed_time(b) / reps
    # the same launches replayed from a CUDA graph: GPU time, not the host's
    # per-call enqueue rate (which bounds the eager loop for small kernels)
    gs = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=gs):
        for _ in range(reps):
            native.check(L.ds_route_device(ctx.handle, native.c_p(dc.data_ptr()), dt, n,
                                           native.c_p(dthr.data_ptr()), nt, 7,
                                           native.c_p(heavy.data_ptr()), native.c_p(cnt.data_ptr()),
                                           native.c_p(gs.cuda_stream)))
    with torch.cuda.stream(gs):
        g.replay()
        a.record(gs)
        g.replay()
        b.record(gs)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    c = cnt.cpu().numpy()
    h = heavy.cpu().numpy().reshape(nt, n)
    ok = True
    for k, t in enumerate(thr):
        want = np.flatnonzero(conf.astype(np.float64) < t) + 7
        ok &= int(c[k]) == len(want) and np.array_equal(h[k, :c[k]], want)
    nbytes = conf.nbytes + 8 * int(c.sum()) + 8 * nt
    print(f"{name}: {ms * 1000:.2f} us (graph; eager {ms_eager * 1000:.2f}), "
          f"{nbytes / ms / 1e6:.0f} GB/s algorithmic ({nbytes / 1e6:.2f} MB), lists exact: {ok}")
