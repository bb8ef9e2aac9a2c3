"""Profile helper: one ds_generate_arrivals call on the bench's 1M-arrival
trace (run under ncu to get the per-kernel launch list)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_15381_b200.api import default_context  # noqa: E402

ctx = default_context()
rates = np.full(400, 2500.0)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    a = ctx.generate_arrivals(rates, 1.0, 3, 0)
print(len(a))
