"""e2e timing of the bare C-ABI macko_spmv_host call (pinned host x / y), as bench.py measures it.
    MACKO_LIB=... python tools/e2e_time.py --tag X"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_13061_b200 import _lib, macko as M  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--tag", default=os.environ.get("MACKO_LIB", "default"))
a = p.parse_args()
R, C = 36864, 12288
dense = torch.empty((R, C), dtype=torch.float16, device="cuda")
M.gen_dense(dense, R, C, 0.5, seed=1234)
dm = M.DeviceMatrix.from_dense(dense)
del dense
hx = torch.empty(C, dtype=torch.int16, pin_memory=True)
hy = torch.empty(R, dtype=torch.int16, pin_memory=True)
xd = torch.empty(C, dtype=torch.float16, device="cuda")
M.gen_vector(xd, C, seed=4321)
hx.copy_(xd.view(torch.int16).cpu())
hxn, hyn = hx.numpy().view(np.uint16), hy.numpy().view(np.uint16)
st = torch.cuda.current_stream()
dm.spmv_host(hxn, hyn, st)
fn, args = _lib.load().macko_spmv_host, (dm._h, hxn.ctypes.data, hyn.ctypes.data, st.cuda_stream)
for _ in range(10):
    fn(*args)
ts = []
for _ in range(100):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    fn(*args)
    e1.record(st)
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3)
ts.sort()
print(f"{a.tag:20s} e2e us: median {ts[50]:.2f}  mean {sum(ts) / len(ts):.2f}  min {ts[0]:.2f}", flush=True)
