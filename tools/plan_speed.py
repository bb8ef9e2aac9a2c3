"""Times ds_plan_batch_device on BASELINE.md's 4,096-problem config-4 batch
(tests/golden/config4_bench.npz; CUDA events over 20 back-to-back calls) and checks the plans against the reference's.

    python tools/plan_speed.py
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2411_15381_b200 import abi, native  # noqa: E402

ctx = native.Context(0)
L = native.lib()
pro, cas, grid, offs, want = bench.planner_inputs()
dev = torch.device("cuda", 0)
d_pro = torch.from_numpy(pro.view(np.uint8).copy()).to(dev)
d_cas = torch.from_numpy(cas.view(np.uint8).copy()).to(dev)
d_grid = torch.from_numpy(np.ascontiguousarray(grid)).to(dev)
d_offs = torch.from_numpy(np.ascontiguousarray(offs)).to(dev)
d_out = torch.empty(len(pro) * abi.PLAN.itemsize, dtype=torch.uint8, device=dev)
sp = native.c_p(ctx.stream)
st = torch.cuda.ExternalStream(ctx.stream)


def call():
    native.check(L.ds_plan_batch_device(ctx.handle, native.c_p(d_pro.data_ptr()), len(pro),
                                        native.c_p(d_cas.data_ptr()), len(cas),
                                        native.c_p(d_grid.data_ptr()), native.c_p(d_offs.data_ptr()),
                                        1, native.c_p(d_out.data_ptr()), sp))


for _ in range(3):
    call()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(st)
for _ in range(20):
    call()
b.record(st)
torch.cuda.synchronize()
eager = a.elapsed_time(b) / 20
ok = d_out.cpu().numpy().view(abi.PLAN).tobytes() == want.tobytes()
print(f"planner {len(pro)} problems: {eager * 1000:.1f} us per call "
      f"({len(pro) / eager * 1000:.3e} problems/s); plans == reference: {ok}")
