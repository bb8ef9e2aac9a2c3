"""Times ds_format_queries_csv_device on 1M random QueryRecords (the bench's
csv leg; CUDA events, 5 launches) and checks the bytes against the host-buffer
entry point and against the C restatement on a 200K slice."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import lib  # noqa: E402
from paper_2411_15381_b200 import abi, native  # noqa: E402
from tests import helpers  # noqa: E402

n = 1_000_000
ctx = native.Context(0)
L = native.lib()
rec = helpers.random_query_records(np.random.default_rng(12), n)
drec = torch.from_numpy(rec.view(np.uint8).copy()).cuda()
cap = n * 256 + 4096
dout = torch.empty(cap, dtype=torch.uint8, device="cuda")
nb = native.i64(0)
torch.cuda.synchronize()
st = torch.cuda.ExternalStream(ctx.stream)


def run():
    native.check(L.ds_format_queries_csv_device(ctx.handle, native.c_p(drec.data_ptr()), n,
                                                native.c_p(dout.data_ptr()), cap,
                                                native.ctypes.byref(nb), native.c_p(ctx.stream)))


run()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ms = []
for _ in range(5):
    a.record(st)
    run()
    b.record(st)
    torch.cuda.synchronize()
    ms.append(a.elapsed_time(b))
dev = dout[:nb.value].cpu().numpy().tobytes()
host = ctx.format_queries_csv(rec)
sub = np.ascontiguousarray(rec[:200_000])
m = lib.port().dso_format_queries_csv(abi.ptr(sub), len(sub), None, 0)
want = np.zeros(m, np.uint8)
lib.port().dso_format_queries_csv(abi.ptr(sub), len(sub), abi.ptr(want), m)
got_sub = ctx.format_queries_csv(sub)
print(f"csv 1M rows: {min(ms):.3f} ms ({nb.value / 1e6:.1f} MB), device == host-path: "
      f"{dev == host}, 200K slice == C restatement: {got_sub == want.tobytes()}")
