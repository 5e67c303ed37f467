"""Per-warp timeline of one SpMV launch from the trace build (make trace):
MACKO_LIB=paper_2511_13061_b200/libmacko_cuda_trace.so python tools/trace_spmv.py --rows 4096 --cols 4096
Stamps (ns, relative to the earliest kernel start): 0 start, 1 plan record loaded, 2 ring filled /
walk set up, 3 griddepcontrol.wait passed, 4 x staged (after __syncthreads), 6 warp done."""
import argparse
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("MACKO_LIB", os.path.join(ROOT, "paper_2511_13061_b200", "libmacko_cuda_trace.so"))
sys.path.insert(0, ROOT)
from paper_2511_13061_b200 import _lib, macko as M  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--rows", type=int, default=4096)
p.add_argument("--cols", type=int, default=4096)
p.add_argument("--density", type=float, default=0.5)
p.add_argument("--flush", type=int, default=1)
p.add_argument("--skew", type=int, default=0, help="macko_dev_set_chain_skew start spread (ns)")
a = p.parse_args()
dense = torch.empty((a.rows, a.cols), dtype=torch.float16, device="cuda")
M.gen_dense(dense, a.rows, a.cols, a.density, seed=1234)
dm = M.DeviceMatrix.from_dense(dense)
if a.skew:
    dm.set_chain_skew(a.skew)
del dense
x = torch.empty(a.cols, dtype=torch.float16, device="cuda")
M.gen_vector(x, a.cols, seed=4321)
y = torch.empty(a.rows, dtype=torch.float16, device="cuda")
flush = torch.ones(256 << 20, dtype=torch.float32, device="cuda")
for _ in range(3):
    dm.spmv_into(x, y)
if a.flush:
    flush.sum()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
dm.spmv_into(x, y)
e1.record()
torch.cuda.synchronize()
L = _lib.load()
L.macko_trace_read.argtypes = [C.c_void_p, C.c_size_t]
L.macko_trace_slot_counter.restype = C.c_uint
buf = np.zeros(8 * 148 * 32 * 8, np.uint64)
assert L.macko_trace_read(buf.ctypes.data, buf.size) == 0
t = buf.reshape(8, 148 * 32, 8)[(L.macko_trace_slot_counter() - 1) % 8].astype(np.int64)  # the last launch
ok = t[:, 0] > 0
t0 = t[ok, 0].min()
rel = (t[ok] - t0) / 1e3
print(f"event time {e0.elapsed_time(e1) * 1e3:.2f} us; warps {ok.sum()}")
for i, name in [(0, "start"), (1, "record"), (5, "mbar init"), (7, "ring issued"), (2, "walk set"), (3, "gdc.wait"),
                (4, "x staged"), (6, "done")]:
    col = rel[:, i][t[ok, i] > 0]
    if col.size:
        print(f"{name:10s} min {col.min():7.2f}  med {np.median(col):7.2f}  p90 {np.percentile(col, 90):7.2f}  max {col.max():7.2f} us")
# tail analysis: per-CTA spread of the done stamps
done = np.where(t[:, 6] > 0, (t[:, 6] - t0) / 1e3, np.nan).reshape(148, 32)
cta_max = np.nanmax(done, axis=1)
cta_min = np.nanmin(done, axis=1)
print(f"per-CTA last warp: min {np.nanmin(cta_max):.2f} med {np.nanmedian(cta_max):.2f} max {np.nanmax(cta_max):.2f} us; "
      f"within-CTA spread med {np.nanmedian(cta_max - cta_min):.2f} max {np.nanmax(cta_max - cta_min):.2f} us")
order = np.argsort(cta_max)
print("slowest CTAs:", [(int(i), round(float(cta_max[i]), 1)) for i in order[-6:]])
print("fastest CTAs:", [(int(i), round(float(cta_max[i]), 1)) for i in order[:6]])
# done time vs warp index within the CTA (scheduler priority?) and vs SMSP (warp % 4)
rel_done = done - np.nanmedian(done, axis=1, keepdims=True)
print("done - CTA median by warp index (us):", " ".join(f"{v:+.1f}" for v in np.nanmean(rel_done, axis=0)))
print("by SMSP (warp % 4):", [round(float(np.nanmean(rel_done[:, k::4])), 2) for k in range(4)])
print("percentiles of done - CTA median:", [round(float(np.nanpercentile(rel_done, q)), 2) for q in (1, 10, 50, 90, 99)])
