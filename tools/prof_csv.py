"""Profile helper: one ds_format_queries_csv_device call on 1M QueryRecords
(the bench's csv leg), for ncu."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_15381_b200 import native  # noqa: E402
from tests import helpers  # noqa: E402

ctx = native.Context(0)
rec = helpers.random_query_records(np.random.default_rng(12), 1_000_000)
drec = torch.from_numpy(rec.view(np.uint8).copy()).cuda()
out = torch.empty(len(rec) * 256 + 4096, dtype=torch.uint8, device="cuda")
n = native.i64(0)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    native.check(native.lib().ds_format_queries_csv_device(
        ctx.handle, ctypes.c_void_p(drec.data_ptr()), len(rec), ctypes.c_void_p(out.data_ptr()),
        out.numel(), ctypes.byref(n), ctypes.c_void_p(ctx.stream)))
torch.cuda.synchronize()
print(n.value)
