"""Runs each hot-path kernel a few times on its bench workload, for ncu:

    ncu --set full --clock-control none --import-source on -k regex:disc_kernel \
        -s 2 -c 1 -o gpurun_out/disc python tools/prof_kernels.py disc
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2411_15381_b200 import abi, native, workloads  # noqa: E402


def main(which):
    ctx = native.Context(0)
    L = native.lib()
    s = native.c_p(ctx.stream)
    if which in ("disc", "all"):
        n = int(os.environ.get("N_IMG", "5000"))
        disc = native.Discriminator(ctx, 2024)
        img = torch.empty(n * 512 * 512 * 3, dtype=torch.uint8, device="cuda")
        native.check(L.ds_synth_images_device(ctx.handle, 1, 0, n, 512, 512,
                                              native.c_p(img.data_ptr()), s))
        conf = torch.empty(n, dtype=torch.float32, device="cuda")
        for _ in range(3):
            disc.score_device(img.data_ptr(), n, 512, 512, conf.data_ptr(), ctx.stream)
        ctx.synchronize()
    if which in ("plan", "all"):
        sys.path.insert(0, ROOT)
        import bench
        pro, cas, grid, offs, _ = bench.planner_inputs()   # the fixture's curves
        for _ in range(3):
            ctx.plan_batch(pro, cas, grid, offs)
    if which in ("latent", "all"):
        m = workloads.query_model()
        c = torch.empty(1_000_000, dtype=torch.float64, device="cuda")
        for _ in range(3):
            native.check(L.ds_score_latent_device(ctx.handle, abi.ptr(m), 0, 1_000_000,
                                                  native.c_p(c.data_ptr()), native.c_p(0), s))
        ctx.synchronize()
    if which in ("curve", "all"):
        # K3 on the latent leg's 1M confidences (segmented replay) and on 5K
        # (single-CTA replay, the image step's size)
        m = workloads.query_model()
        c = torch.empty(1_000_000, dtype=torch.float64, device="cuda")
        native.check(L.ds_score_latent_device(ctx.handle, abi.ptr(m), 0, 1_000_000,
                                              native.c_p(c.data_ptr()), native.c_p(0), s))
        prior = workloads.uniform_prior()
        p_t = torch.from_numpy(prior.reshape(1).view(np.uint8).copy()).cuda()
        cur = torch.empty_like(p_t)
        for n in (1_000_000, 5_000):
            for _ in range(3):
                cur.copy_(p_t)
                native.check(L.ds_curve_observe_device(ctx.handle, native.c_p(cur.data_ptr()),
                                                       native.c_p(c.data_ptr()), abi.CONF_F64, n,
                                                       0.999, s))
        ctx.synchronize()
    print("done")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "all")
