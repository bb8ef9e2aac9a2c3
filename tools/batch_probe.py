"""Config-1 light batches (32 images): where the per-batch time goes. Times
CUDA graphs of the 157 batches of the 5K pool with (a) the discriminator
only, (b) + curve observe, (c) + route (the bench's batch32 step)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_15381_b200 import abi, native, workloads  # noqa: E402

N, B, H = 5000, int(sys.argv[1]) if len(sys.argv) > 1 else 32, 512
ctx = native.Context(0)
L = native.lib()
disc = native.Discriminator(ctx, 2024)
img = torch.empty(N * H * H * 3, dtype=torch.uint8, device="cuda")
native.check(L.ds_synth_images_device(ctx.handle, 1, 0, N, H, H, native.c_p(img.data_ptr()),
                                      native.c_p(ctx.stream)))
conf = torch.empty(N, dtype=torch.float32, device="cuda")
prior = workloads.uniform_prior()
p_t = torch.from_numpy(prior.reshape(1).view(np.uint8).copy()).cuda()
cur = torch.empty_like(p_t)
thr = torch.tensor([0.5], dtype=torch.float64, device="cuda")
heavy = torch.empty(B, dtype=torch.int64, device="cuda")
cnt = torch.empty(1, dtype=torch.int64, device="cuda")
torch.cuda.synchronize()


def step(sp, what):
    for off in range(0, N, B):
        m = min(B, N - off)
        cp = native.c_p(conf.data_ptr() + 4 * off)
        native.check(L.ds_disc_score_device(disc.handle, native.c_p(img.data_ptr() + off * H * H * 3),
                                            m, H, H, cp, sp))
        if what >= 1:
            native.check(L.ds_curve_observe_device(ctx.handle, native.c_p(cur.data_ptr()), cp,
                                                   abi.CONF_F32, m, 0.999, sp))
        if what >= 2:
            native.check(L.ds_route_device(ctx.handle, cp, abi.CONF_F32, m,
                                           native.c_p(thr.data_ptr()), 1, off,
                                           native.c_p(heavy.data_ptr()), native.c_p(cnt.data_ptr()),
                                           sp))


for what, name in ((0, "disc only"), (1, "disc + curve"), (2, "disc + curve + route")):
    s = torch.cuda.Stream()
    sp = native.c_p(s.cuda_stream)
    with torch.cuda.stream(s):
        step(sp, what)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        step(sp, what)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        g.replay()
        a.record(s)
        for _ in range(3):
            g.replay()
        b.record(s)
    torch.cuda.synchronize()
    nb = (N + B - 1) // B
    print(f"batch {B}: {name:22s} {a.elapsed_time(b) / 3 * 1000 / nb:7.2f} us per batch")
