"""Times ds_generate_arrivals_device on the bench's 1M-arrival Poisson trace
(400 intervals x 2500 qps, seed 3; CUDA events, 5 calls) and checks the
timestamps against the C restatement."""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import lib  # noqa: E402
from paper_2411_15381_b200 import abi, native  # noqa: E402

ctx = native.Context(0)
L = native.lib()
rates = np.asarray([2500.0] * 400, np.float64)
cap = 1_100_000
out = torch.empty(cap, dtype=torch.float64, device="cuda")
n = native.i64(0)
st = torch.cuda.ExternalStream(ctx.stream)


def run():
    native.check(L.ds_generate_arrivals_device(ctx.handle, abi.ptr(rates), len(rates), 1.0, 3,
                                               abi.ARRIVALS_POISSON, native.c_p(out.data_ptr()),
                                               cap, ctypes.byref(n), native.c_p(ctx.stream)))


run()
ms = []
for _ in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    run()
    b.record(st)
    torch.cuda.synchronize()
    ms.append(a.elapsed_time(b))
got = out[:n.value].cpu().numpy()
m = lib.port().dso_generate_arrivals(abi.ptr(rates), len(rates), 1.0, 3, 0, None, 0)
want = np.zeros(m)
lib.port().dso_generate_arrivals(abi.ptr(rates), len(rates), 1.0, 3, 0, abi.ptr(want), m)
print(f"{'no jump' if os.environ.get('DS_ARRIVALS_NO_JUMP') else 'jump-ahead'}: 1M arrivals "
      f"{min(ms):.3f} ms, bit-identical to the port: {got.tobytes() == want.tobytes()}")
