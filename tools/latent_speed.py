"""Times ds_score_latent_device on 1M queries (CUDA events, 10 launches) and
checks the confidences against the C restatement (the A/B harness for K4)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import lib  # noqa: E402
from paper_2411_15381_b200 import abi, native, workloads  # noqa: E402

n = 1_000_000
ctx = native.Context(0)
L = native.lib()
m = workloads.query_model()
c = torch.empty(n, dtype=torch.float64, device="cuda")
st = torch.cuda.ExternalStream(ctx.stream)


def run():
    native.check(L.ds_score_latent_device(ctx.handle, abi.ptr(m), 0, n, native.c_p(c.data_ptr()),
                                          native.c_p(0), native.c_p(ctx.stream)))


run()
ctx.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(st)
for _ in range(10):
    run()
b.record(st)
torch.cuda.synchronize()
ref = np.zeros(n)
lib.port().dso_sample_queries(abi.ptr(m), 0, n, abi.ptr(ref), None, 8)
got = c.cpu().numpy()
ok = bool(np.array_equal(got.view(np.uint64), ref.view(np.uint64)))
print(f"{os.environ.get('DS_EXTRA_NVCC', 'default')}: latent score 1M: {a.elapsed_time(b) / 10:.4f} ms, "
      f"bit-identical to the port: {ok}")
