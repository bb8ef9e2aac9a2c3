"""Writes the discriminator's confidences for N synthetic 512x512 images to
gpurun_out/conf_<tag>.npy (bit-identity checks between builds).

    python tools/disc_dump.py TAG [N=5000]
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2411_15381_b200 import native  # noqa: E402

tag = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 5000
ctx = native.Context(0)
L = native.lib()
disc = native.Discriminator(ctx, 2024)
img = torch.empty(n * 512 * 512 * 3, dtype=torch.uint8, device="cuda")
native.check(L.ds_synth_images_device(ctx.handle, 1, 0, n, 512, 512, native.c_p(img.data_ptr()),
                                      native.c_p(ctx.stream)))
conf = torch.empty(n, dtype=torch.float32, device="cuda")
disc.score_device(img.data_ptr(), n, 512, 512, conf.data_ptr(), ctx.stream)
ctx.synchronize()
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
np.save(os.path.join(ROOT, "gpurun_out", f"conf_{tag}.npy"), conf.cpu().numpy())
print(tag, conf[:4].tolist())
