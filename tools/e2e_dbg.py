"""e2e timing of macko_spmv_host (pinned host x / y) on the headline matrix, as bench.py times it."""
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_13061_b200 import macko as M  # noqa: E402

R, C = 36864, 12288
dense = torch.empty((R, C), dtype=torch.float16, device="cuda")
M.gen_dense(dense, R, C, 0.5, seed=1234)
dm = M.DeviceMatrix.from_dense(dense)
del dense
hx = torch.empty(C, dtype=torch.int16, pin_memory=True)
hy = torch.empty(R, dtype=torch.int16, pin_memory=True)
hxn, hyn = hx.numpy().view(np.uint16), hy.numpy().view(np.uint16)
hxn[:] = np.arange(C) % 1000
st = torch.cuda.current_stream()
for _ in range(5):
    dm.spmv_host(hxn, hyn, st)
ts = []
for _ in range(50):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    dm.spmv_host(hxn, hyn, st)
    b.record(st)
    b.synchronize()
    ts.append(a.elapsed_time(b) * 1e3)
print(f"e2e median {statistics.median(ts):.2f} us  mean {sum(ts) / len(ts):.2f}")
