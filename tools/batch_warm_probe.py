"""Config-1 batches of 32: does the first tile wait on HBM? The same graph of
157 discriminator launches over (a) the 157 distinct batches of the 5K pool
(cold in L2) and (b) one batch 157 times (L2-warm), per-batch time."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_15381_b200 import native  # noqa: E402

N, B, H = 5000, 32, 512
ctx = native.Context(0)
L = native.lib()
disc = native.Discriminator(ctx, 2024)
img = torch.empty(N * H * H * 3, dtype=torch.uint8, device="cuda")
native.check(L.ds_synth_images_device(ctx.handle, 1, 0, N, H, H, native.c_p(img.data_ptr()),
                                      native.c_p(ctx.stream)))
conf = torch.empty(N, dtype=torch.float32, device="cuda")
torch.cuda.synchronize()
for warm in (False, True):
    s = torch.cuda.Stream()
    sp = native.c_p(s.cuda_stream)

    def step():
        for k, off in enumerate(range(0, N, B)):
            src = 0 if warm else off
            native.check(L.ds_disc_score_device(disc.handle,
                                                native.c_p(img.data_ptr() + src * H * H * 3), B,
                                                H, H, native.c_p(conf.data_ptr() + 4 * off), sp))
    with torch.cuda.stream(s):
        step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        step()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        g.replay()
        a.record(s)
        for _ in range(3):
            g.replay()
        b.record(s)
    torch.cuda.synchronize()
    nb = (N + B - 1) // B
    print(f"batch {B} {'L2-warm (same batch)' if warm else 'distinct batches'}: "
          f"{a.elapsed_time(b) / 3 * 1000 / nb:.2f} us per batch")
