"""One launch each of the non-GEMM hot kernels on their bench inputs, for an
ncu capture (tools/ncu_summarize.py turns the CSV into profiles/*.json):

  K1 plan_sweep_kernel : the 4,096-problem config-4 batch (tests/golden/config4_bench.npz)
  K4 latent_kernel     : 1M queries of the cascade model (bench latent leg)
  K2 route_kernel      : those 1M f64 confidences at t = 0.5

    ncu --metrics ... --csv --log-file gpurun_out/x.csv python tools/ncu_kernels.py
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2411_15381_b200 import abi, native, workloads  # noqa: E402

ctx = native.Context(0)
L = native.lib()
sp = native.c_p(ctx.stream)
g = dict(np.load(os.path.join(ROOT, "tests", "golden", "config4_bench.npz")))
pro, cas, gv, go = g["problems"], g["cascades"], g["grid_values"], g["grid_offsets"]


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.uint8).copy()).cuda()


dp, dc, dg, do = dev(pro), dev(cas), dev(gv), dev(go)
out = torch.empty(len(pro) * abi.PLAN.itemsize, dtype=torch.uint8, device="cuda")
n = 1_000_000
conf = torch.empty(n, dtype=torch.float64, device="cuda")
heavy = torch.empty(n, dtype=torch.int64, device="cuda")
cnt = torch.empty(1, dtype=torch.int64, device="cuda")
thr = torch.tensor([0.5], dtype=torch.float64, device="cuda")
qm = workloads.query_model()
torch.cuda.synchronize()
for _ in range(2):   # the second round is the warm one (ncu -c counts both)
    native.check(L.ds_plan_batch_device(ctx.handle, native.c_p(dp.data_ptr()), len(pro),
                                        native.c_p(dc.data_ptr()), len(cas),
                                        native.c_p(dg.data_ptr()), native.c_p(do.data_ptr()),
                                        len(go) - 1, native.c_p(out.data_ptr()), sp))
    native.check(L.ds_score_latent_device(ctx.handle, abi.ptr(qm), 0, n,
                                          native.c_p(conf.data_ptr()), native.c_p(0), sp))
    native.check(L.ds_route_device(ctx.handle, native.c_p(conf.data_ptr()), abi.CONF_F64, n,
                                   native.c_p(thr.data_ptr()), 1, 0, native.c_p(heavy.data_ptr()),
                                   native.c_p(cnt.data_ptr()), sp))
    ctx.synchronize()
print("deferred at 0.5:", int(cnt.item()))
