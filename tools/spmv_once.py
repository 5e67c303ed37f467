"""Profiling driver: build one synthetic MACKO matrix on cuda:0 and run a few SpMVs (for ncu)."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_13061_b200 import macko as M  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--rows", type=int, default=36864)
p.add_argument("--cols", type=int, default=12288)
p.add_argument("--density", type=float, default=0.5)
p.add_argument("--reps", type=int, default=3)
p.add_argument("--x-mode", type=int, default=-1)
a = p.parse_args()
dense = torch.empty((a.rows, a.cols), dtype=torch.float16, device="cuda")
M.gen_dense(dense, a.rows, a.cols, a.density, seed=1234)
dm = M.DeviceMatrix.from_dense(dense)
del dense
if a.x_mode != -1:
    dm.configure(a.x_mode)
x = torch.empty(a.cols, dtype=torch.float16, device="cuda")
M.gen_vector(x, a.cols, seed=4321)
y = torch.empty(a.rows, dtype=torch.float16, device="cuda")
flush = torch.ones(256 << 20, dtype=torch.float32, device="cuda")
for _ in range(a.reps):
    flush.sum()
    dm.spmv_into(x, y, torch.cuda.current_stream())
torch.cuda.synchronize()
print("ok", a.rows, a.cols, a.density, dm.pad_nnz)
