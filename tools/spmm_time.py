"""Small-batch SpMM timing per gather split (MACKO_SPMM_XMODE), 36864x12288 @50 % unless given:
    python tools/spmm_time.py [--shape 36864x12288@0.5]"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_13061_b200 import macko as M  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--shape", default="36864x12288@0.5")
p.add_argument("--modes", default="7,0,1,6,8")
a = p.parse_args()
shp, d = a.shape.split("@")
R, C = (int(v) for v in shp.split("x"))
dense = torch.empty((R, C), dtype=torch.float16, device="cuda")
M.gen_dense(dense, R, C, float(d), seed=1234)
dm = M.DeviceMatrix.from_dense(dense)
del dense
st = torch.cuda.current_stream()
for b in (2, 4, 8):
    X = torch.empty((b, C), dtype=torch.float16, device="cuda")
    for i in range(b):
        M.gen_vector(X[i], C, seed=10 + i)
    Y = torch.empty((b, R), dtype=torch.float16, device="cuda")
    ref = None
    for mode in a.modes.split(","):
        os.environ["MACKO_SPMM_XMODE"] = mode
        for _ in range(3):
            dm.spmm_into(X, Y, st)
        torch.cuda.synchronize()
        if ref is None:
            ref = Y.clone()
        same = bool(torch.equal(Y, ref))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 30
        e0.record(st)
        for _ in range(n):
            dm.spmm_into(X, Y, st)
        e1.record(st)
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / n
        print(f"batch {b} x_mode {mode}: {us:8.2f} us  ({us / b:7.2f} us/vector)  y==mode{a.modes.split(',')[0]}: {same}", flush=True)
