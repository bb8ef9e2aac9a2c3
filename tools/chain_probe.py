"""Config-1 light batches through chained ds_disc_batch_complete_device calls
(programmatic dependent launch): (1) CUDA-graph time per batch of 32 for
several pair sizes (DS_DISC_MIN_PAIR_TILES: pair tiles per SM pair, fewer and
longer-lived pairs) and unchained; (2) the CTA timeline of 6 chained calls
(per-CTA start / end globaltimer, ds_disc_batch_trace_device).

    python tools/chain_probe.py
"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2411_15381_b200 import native, workloads  # noqa: E402

N, B, H = 5000, 32, 512
ctx = native.Context(0)
L = native.lib()
img = torch.empty(N * H * H * 3, dtype=torch.uint8, device="cuda")
native.check(L.ds_synth_images_device(ctx.handle, 1, 0, N, H, H, native.c_p(img.data_ptr()),
                                      native.c_p(ctx.stream)))
conf = torch.empty(N, dtype=torch.float32, device="cuda")
prior = torch.from_numpy(workloads.uniform_prior().reshape(1).view(np.uint8).copy()).cuda()
cur = prior.clone()
thr = torch.full((N // B + 1,), 0.5, dtype=torch.float64, device="cuda")
heavy = torch.empty(N, dtype=torch.int64, device="cuda")
cnt = torch.empty(N // B + 1, dtype=torch.int64, device="cuda")
torch.cuda.synchronize()


def calls(disc, sp):
    for k, off in enumerate(range(0, N, B)):
        m = min(B, N - off)
        disc.batch_complete_device(img.data_ptr() + off * H * H * 3, m, H, H, conf.data_ptr() + 4 * off,
                                   cur.data_ptr(), 0.999, thr.data_ptr() + 8 * k, 1, off,
                                   heavy.data_ptr() + 8 * off, cnt.data_ptr() + 8 * k, sp)


def per_batch_us(disc):
    s = torch.cuda.Stream()
    sp = s.cuda_stream
    calls(disc, sp)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        calls(disc, sp)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        g.replay()
        a.record(s)
        for _ in range(5):
            g.replay()
        b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / 5 / ((N + B - 1) // B)


ref = None
for knob in ("nochain", "1", "2", "3", "4", "6", "8"):
    os.environ.pop("DS_DISC_NO_CHAIN", None)
    os.environ.pop("DS_DISC_MIN_PAIR_TILES", None)
    if knob == "nochain":
        os.environ["DS_DISC_NO_CHAIN"] = "1"
    else:
        os.environ["DS_DISC_MIN_PAIR_TILES"] = knob
    disc = native.Discriminator(ctx, 2024)
    us = per_batch_us(disc)
    cur.copy_(prior)
    calls(disc, 0)
    ctx.synchronize()
    got = (conf.cpu().numpy().tobytes(), cur.cpu().numpy().tobytes())
    ref = ref or got
    print(f"{knob:>8}: {us:6.2f} us per batch of {B}   bits == unchained: {got == ref}", flush=True)
    if knob == "1":
        chain_disc = disc
os.environ.pop("DS_DISC_MIN_PAIR_TILES", None)

# timeline of 6 chained calls
L.ds_disc_batch_trace_device.argtypes = [ctypes.c_void_p] * 2 + [ctypes.c_int64, ctypes.c_int32,
                                         ctypes.c_int32] + [ctypes.c_void_p] * 2 + \
    [ctypes.c_double, ctypes.c_void_p, ctypes.c_int64] + [ctypes.c_void_p] * 4
NT = 8 * 8 * 16
K = 6
tr = [torch.zeros(NT + 5 * 160, dtype=torch.int64, device="cuda") for _ in range(K)]
sp = native.c_p(ctx.stream)
for rep in range(2):
    for i in range(K):
        tr[i].zero_()
    ctx.synchronize()
    for i in range(K):
        off = i * B
        native.check(L.ds_disc_batch_trace_device(
            chain_disc.handle, native.c_p(img.data_ptr() + off * H * H * 3), B, H, H,
            native.c_p(conf.data_ptr() + 4 * off), native.c_p(cur.data_ptr()), 0.999,
            native.c_p(thr.data_ptr()), off, native.c_p(heavy.data_ptr() + 8 * off),
            native.c_p(cnt.data_ptr() + 8 * i), native.c_p(tr[i].data_ptr()), sp))
    ctx.synchronize()
t = [x.cpu().numpy() for x in tr]
ctas = [x[NT:NT + 480].reshape(160, 3) for x in t]
ctas = [c[c[:, 0] > 0] for c in ctas]
t0 = ctas[0][:, 0].min()
for i, c in enumerate(ctas):
    s, e = c[:, 0] - t0, c[:, 1] - t0
    d = e - s
    print(f"call {i}: {len(c)} CTAs  start min {s.min()/1e3:.1f} med {np.median(s)/1e3:.1f} "
          f"max {s.max()/1e3:.1f}  end min {e.min()/1e3:.1f} med {np.median(e)/1e3:.1f} "
          f"max {e.max()/1e3:.1f}  dur min {d.min()/1e3:.1f} med {np.median(d)/1e3:.1f} "
          f"max {d.max()/1e3:.1f} (us)")
# CTA 0's phase stamps (clock64 cycles from its first stamp) in calls 0 and 3
names = {0: "A-builder (0 tile start, 1 chunks stored; tile 0: 5 role entry, 6 L2 prefetch issued, "
            "7/8 chunk 0/1 loads issued)", 3: "A-builder chunk c: a_empty passed", 4: "chunk c stored+signalled",
         1: "epilogue (0 E1 rdy, 1 E1 done, 2+2j/3+2j E2_j, 10/11 E3)",
         2: "MMA (0 tile, 1 G1 issued, 2 G3_3(prev), 3 E1 seen, 4.. dr/rd)",
         5: "MMA a_full seen per chunk"}
for call in (0, 3):
    ph = t[call][:NT].reshape(8, 8, 16)
    pos = ph[:7][ph[:7] > 0]
    c0 = pos.min()
    print(f"call {call} CTA 0 phases (cycles):")
    for role in (0, 1, 2, 3, 4, 5):
        for tile in range(2):
            row = ph[role, tile]
            if (row > 0).any():
                print(f"  role {role} tile {tile}: " +
                      " ".join(str(int(v - c0)) if v else "." for v in row))
    print("  (legend: " + "; ".join(f"{k}: {v}" for k, v in names.items()) + ")")
