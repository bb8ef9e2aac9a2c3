"""Config-1 light batch (32 images 512x512): the timeline of one discriminator
launch and the gap to the next. Two launches back to back (same stream), each
with its own trace buffer (ds_disc_trace_device: per-CTA start / end
globaltimer and SM id; CTA 0's clock64 phase stamps). Prints, in ns from the
first CTA start of launch 1: CTA start / end spread of both launches, and
CTA 0's per-tile phases (role rows of disc.cu's DS_TRACE).

    python tools/batch_trace.py [batch]
"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2411_15381_b200 import native  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
H = 512
ctx = native.Context(0)
L = native.lib()
disc = native.Discriminator(ctx, 2024)
img = torch.empty(2 * B * H * H * 3, dtype=torch.uint8, device="cuda")
native.check(L.ds_synth_images_device(ctx.handle, 1, 0, 2 * B, H, H, native.c_p(img.data_ptr()),
                                      native.c_p(ctx.stream)))
conf = torch.empty(2 * B, dtype=torch.float32, device="cuda")
L.ds_disc_trace_device.argtypes = [ctypes.c_void_p] * 2 + [ctypes.c_int64, ctypes.c_int32,
                                                            ctypes.c_int32] + [ctypes.c_void_p] * 3
NT = 8 * 8 * 16
tr = [torch.zeros(NT + 5 * 160, dtype=torch.int64, device="cuda") for _ in range(2)]
sp = native.c_p(ctx.stream)
for _ in range(5):
    disc.score_device(img.data_ptr(), B, H, H, conf.data_ptr(), ctx.stream)
ctx.synchronize()
for i in range(2):
    native.check(L.ds_disc_trace_device(disc.handle, native.c_p(img.data_ptr() + i * B * H * H * 3),
                                        B, H, H, native.c_p(conf.data_ptr() + 4 * i * B),
                                        native.c_p(tr[i].data_ptr()), sp))
ctx.synchronize()
t = [x.cpu().numpy() for x in tr]
ctas = [x[NT:NT + 480].reshape(160, 3) for x in t]
ctas = [c[c[:, 0] > 0] for c in ctas]
t0 = ctas[0][:, 0].min()
for i, c in enumerate(ctas):
    s, e = c[:, 0] - t0, c[:, 1] - t0
    print(f"launch {i}: {len(c)} CTAs  start min {s.min()} med {int(np.median(s))} max {s.max()}  "
          f"end min {e.min()} med {int(np.median(e))} max {e.max()} (ns)")
print(f"gap: launch 1 first start - launch 0 last end = {ctas[1][:, 0].min() - ctas[0][:, 1].max()} ns")
ph = t[0][:NT].reshape(8, 8, 16)
c0 = ph[ph > 0].min() if (ph > 0).any() else 0
for role in range(8):
    for tile in range(2):
        row = ph[role, tile]
        if (row > 0).any():
            print(f"CTA0 role {role} tile {tile}: " +
                  " ".join(str(int(v - c0)) if v else "." for v in row), "(clock64 cycles)")

# the same two launches captured in a CUDA graph (the config-1 bench path):
# kernel-boundary gap without host launch overhead
gs = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
tr2 = [torch.zeros(NT + 5 * 160, dtype=torch.int64, device="cuda") for _ in range(3)]
torch.cuda.synchronize()
with torch.cuda.graph(g, stream=gs):
    for i in range(3):
        native.check(L.ds_disc_trace_device(disc.handle, native.c_p(img.data_ptr()), B, H, H,
                                            native.c_p(conf.data_ptr()),
                                            native.c_p(tr2[i].data_ptr()),
                                            native.c_p(gs.cuda_stream)))
for _ in range(2):
    g.replay()
torch.cuda.synchronize()
c2 = [x.cpu().numpy()[NT:NT + 480].reshape(160, 3) for x in tr2]
c2 = [c[c[:, 0] > 0] for c in c2]
t0 = c2[0][:, 0].min()
for i, c in enumerate(c2):
    print(f"graph launch {i}: start min {c[:, 0].min() - t0} max {c[:, 0].max() - t0}  "
          f"end min {c[:, 1].min() - t0} max {c[:, 1].max() - t0} (ns)")
for i in range(3):
    ph = tr2[i].cpu().numpy()[:NT].reshape(8, 8, 16)
    print(f"graph launch {i} CTA 0: MMA issuer done {int(ph[0, 7, 0] - t0)}, past the cluster "
          f"barrier {int(ph[0, 7, 1] - t0)} (ns)")
