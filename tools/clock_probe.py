"""In-kernel SM clock of disc_kernel over a sustained run (config 2: 5,000
512x512 images per launch, back to back).

Every `every`-th launch is a traced one (ds_disc_trace_device): each CTA stamps
clock64 and globaltimer at its start and end, so the launch's real SM clock is
measured inside the kernel, independent of NVML's averaged readings. Prints,
per traced launch: time since start, launch us, median in-kernel MHz, cycles
per pair tile (clock-independent), and NVML's clock/power at that moment.

    python tools/clock_probe.py [seconds=3] [every=20]
"""
import ctypes
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2411_15381_b200 import native  # noqa: E402


def main():
    secs = float(sys.argv[1]) if len(sys.argv) > 1 else 3.0
    every = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    n = 5000
    ctx = native.Context(0)
    L = native.lib()
    L.ds_disc_trace_device.argtypes = [ctypes.c_void_p] * 2 + [ctypes.c_int64, ctypes.c_int32,
                                                                ctypes.c_int32] + [ctypes.c_void_p] * 3
    disc = native.Discriminator(ctx, 2024)
    img = torch.empty(n * 512 * 512 * 3, dtype=torch.uint8, device="cuda")
    native.check(L.ds_synth_images_device(ctx.handle, 1, 0, n, 512, 512,
                                          native.c_p(img.data_ptr()), native.c_p(ctx.stream)))
    conf = torch.empty(n, dtype=torch.float32, device="cuda")
    nt = 8 * 8 * 16
    tr = torch.zeros(nt + 5 * 160, dtype=torch.int64, device="cuda")
    try:
        import pynvml as nv
        nv.nvmlInit()
        h = nv.nvmlDeviceGetHandleByIndex(0)
    except Exception:   # noqa: BLE001
        nv = None
    pair_tiles = (n * 1024 // 128 + 1) // 2
    ctx.synchronize()
    time.sleep(1.0)   # idle: start from the cool state
    t0 = time.time()
    k = 0
    print("t_s   launch_us  mhz_med  mhz_min  cyc/pair_tile  nvml_mhz  nvml_W")
    while time.time() - t0 < secs:
        traced = k % every == 0
        if traced:
            native.check(L.ds_disc_trace_device(disc.handle, native.c_p(img.data_ptr()), n, 512, 512,
                                                native.c_p(conf.data_ptr()),
                                                native.c_p(tr.data_ptr()), native.c_p(ctx.stream)))
            ctx.synchronize()
            t = tr.cpu().numpy()
            ns = t[nt:nt + 480].reshape(160, 3)
            cyc = t[nt + 480:nt + 800].reshape(160, 2)
            u = (ns[:, 1] > ns[:, 0]) & (cyc[:, 1] > cyc[:, 0])
            mhz = (cyc[u, 1] - cyc[u, 0]) / ((ns[u, 1] - ns[u, 0]) / 1e3)
            cpt = np.median(cyc[u, 1] - cyc[u, 0]) / (pair_tiles / (u.sum() // 2))
            us = (ns[u, 1].max() - ns[u, 0].min()) / 1e3
            nvc = nvw = -1
            if nv is not None:
                nvc = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                nvw = nv.nvmlDeviceGetPowerUsage(h) / 1000.0
            print(f"{time.time() - t0:5.2f} {us:9.0f} {np.median(mhz):8.0f} {mhz.min():8.0f} "
                  f"{cpt:13.0f} {nvc:9} {nvw:7.0f}")
        else:
            disc.score_device(img.data_ptr(), n, 512, 512, conf.data_ptr(), ctx.stream)
        k += 1
    ctx.synchronize()


if __name__ == "__main__":
    main()
