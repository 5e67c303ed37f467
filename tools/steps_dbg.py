"""Debug timing: per-launch CUDA-event times of macko_spmv on the headline matrix for several
x_modes, with an L2 flush before each launch (--flush) or back to back."""
import argparse
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_13061_b200 import macko as M  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--rows", type=int, default=36864)
p.add_argument("--cols", type=int, default=12288)
p.add_argument("--density", type=float, default=0.5)
p.add_argument("--modes", default="-1")
p.add_argument("--flush", type=int, default=1)
p.add_argument("--n", type=int, default=40)
p.add_argument("--bits", type=int, default=4)
a = p.parse_args()
R, C = a.rows, a.cols
dense = torch.empty((R, C), dtype=torch.float16, device="cuda")
M.gen_dense(dense, R, C, a.density, seed=1234)
dm = M.DeviceMatrix.from_dense(dense, b_delta=a.bits)
del dense
x = torch.empty(C, dtype=torch.float16, device="cuda")
M.gen_vector(x, C, seed=4321)
y = torch.empty(R, dtype=torch.float16, device="cuda")
st = torch.cuda.current_stream()
flush = torch.ones(256 << 20, dtype=torch.float32, device="cuda")
for mode in [int(m) for m in a.modes.split(",")]:
    dm.configure(mode)
    for _ in range(3):
        dm.spmv_into(x, y, st)
    ts = []
    for i in range(a.n):
        if a.flush:
            flush.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        dm.spmv_into(x, y, st)
        e1.record(st)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    print(f"b{a.bits} d={a.density} mode {dm.launch_info().x_in_smem:2d} flush {a.flush}: median {statistics.median(ts):7.2f} us  min {min(ts):7.2f}  "
          f"GB/s {dm.traffic_bytes / statistics.median(ts) / 1e3:7.1f}")
