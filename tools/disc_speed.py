"""Times ds_disc_score_device alone on 5,000 device-resident 512x512 images
(CUDA events, 3 warm-up + 10 timed launches) and prints images/s -- the quick
A/B harness for kernel variants (build with DS_EXTRA_NVCC=-D... first)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2411_15381_b200 import native  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
    hw = int(sys.argv[2]) if len(sys.argv) > 2 else 512
    ctx = native.Context(0)
    L = native.lib()
    disc = native.Discriminator(ctx, 2024)
    img = torch.empty(n * hw * hw * 3, dtype=torch.uint8, device="cuda")
    native.check(L.ds_synth_images_device(ctx.handle, 1, 0, n, hw, hw, native.c_p(img.data_ptr()),
                                          native.c_p(ctx.stream)))
    conf = torch.empty(n, dtype=torch.float32, device="cuda")
    st = torch.cuda.ExternalStream(ctx.stream)
    for _ in range(3):
        disc.score_device(img.data_ptr(), n, hw, hw, conf.data_ptr(), ctx.stream)
    ctx.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    reps = 10
    a.record(st)
    for _ in range(reps):
        disc.score_device(img.data_ptr(), n, hw, hw, conf.data_ptr(), ctx.stream)
    b.record(st)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    # clock-independent view: CTA 0's SM cycles per pair tile (clock64 trace)
    import ctypes
    L.ds_disc_trace_device.argtypes = [ctypes.c_void_p] * 2 + [ctypes.c_int64, ctypes.c_int32,
                                                                ctypes.c_int32] + [ctypes.c_void_p] * 3
    tr = torch.zeros(8 * 8 * 16 + 5 * 160, dtype=torch.int64, device="cuda")
    native.check(L.ds_disc_trace_device(disc.handle, native.c_p(img.data_ptr()), n, hw, hw,
                                        native.c_p(conf.data_ptr()), native.c_p(tr.data_ptr()),
                                        native.c_p(ctx.stream)))
    ctx.synchronize()
    t = tr[:8 * 8 * 16].view(8, 8, 16)[2, :, 0].cpu().tolist()
    d = sorted(t[i + 1] - t[i] for i in range(1, 7))
    # whole launch: every CTA's clock64 span / its pair tiles, and its SM clock
    allt = tr.cpu().numpy()
    ns = allt[8 * 8 * 16:8 * 8 * 16 + 480].reshape(160, 3)
    cy = allt[8 * 8 * 16 + 480:].reshape(160, 2)
    u = (ns[:, 1] > ns[:, 0]) & (cy[:, 1] > cy[:, 0])
    pair_tiles = (n * (hw // 16) ** 2 // 128 + 1) // 2
    span = cy[u, 1] - cy[u, 0]
    launch_cpt = float(np.median(span)) / (pair_tiles / (u.sum() // 2))
    mhz = float(np.median(span / ((ns[u, 1] - ns[u, 0]) / 1e3)))
    print(f"{os.environ.get('DS_EXTRA_NVCC', 'default')}: {n / ms * 1000:.0f} images/s "
          f"({ms:.3f} ms / {n} images {hw}x{hw}); cycles/tile median {d[len(d) // 2]} "
          f"(tiles 2-7: {d}); launch cycles/pair tile {launch_cpt:.0f} at {mhz:.0f} MHz; conf[0:3] = {[round(x, 6) for x in conf[:3].tolist()]}")


if __name__ == "__main__":
    main()
