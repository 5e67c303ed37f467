"""Is the per-warp completion spread of one SpMV launch deterministic?  Two traced launches of the
same matrix (trace build, make trace): correlation of each warp's done time relative to its CTA's
median, and of that with the warp's element count and row count (from the plan records).
    MACKO_LIB=paper_2511_13061_b200/libmacko_cuda_trace.so python tools/trace_corr.py"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("MACKO_LIB", os.path.join(ROOT, "paper_2511_13061_b200", "libmacko_cuda_trace.so"))
sys.path.insert(0, ROOT)
from paper_2511_13061_b200 import _lib, macko as M  # noqa: E402

R, C = (int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "36864x12288").split("x"))
dense = torch.empty((R, C), dtype=torch.float16, device="cuda")
M.gen_dense(dense, R, C, 0.5, seed=1234)
dm = M.DeviceMatrix.from_dense(dense)
del dense
x = torch.empty(C, dtype=torch.float16, device="cuda")
M.gen_vector(x, C, seed=4321)
y = torch.empty(R, dtype=torch.float16, device="cuda")
L = _lib.load()
L.macko_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
L.macko_trace_slot_counter.restype = ctypes.c_uint
flush = torch.ones(256 << 20, dtype=torch.float32, device="cuda")


def one():
    for _ in range(3):
        dm.spmv_into(x, y)
    flush.sum()
    torch.cuda.synchronize()
    dm.spmv_into(x, y)
    torch.cuda.synchronize()
    buf = np.zeros(8 * 148 * 32 * 8, np.uint64)
    assert L.macko_trace_read(buf.ctypes.data, buf.size) == 0
    t = buf.reshape(8, 148, 32, 8)[(L.macko_trace_slot_counter() - 1) % 8].astype(np.int64)
    done = (t[:, :, 6] - t[:, :, 0].min()) / 1e3
    return done - np.median(done, axis=1, keepdims=True), done


a, da = one()
b, db = one()
recs, _ = dm.plan_records()
rec = recs[: 148 * 32]
elems = (rec[:, 4].astype(np.int64) - rec[:, 3].astype(np.int64)).reshape(148, 32)
units = rec[:, 0].reshape(148, 32).astype(np.float64)
ok = np.isfinite(a) & np.isfinite(b)
print(f"done spread within CTA: p1 {np.percentile(a, 1):.2f} p99 {np.percentile(a, 99):.2f} us")
print(f"corr(run1, run2) of done - CTA median: {np.corrcoef(a[ok], b[ok])[0, 1]:.3f}")
e = elems - elems.mean(axis=1, keepdims=True)
print(f"corr(done - median, elements - CTA mean): {np.corrcoef(a[ok], e[ok])[0, 1]:.3f}")
print(f"corr(CTA last warp run1, run2): {np.corrcoef(da.max(axis=1), db.max(axis=1))[0, 1]:.3f}")
print("CTA last warp (us): run1 min/med/max", np.round([da.max(1).min(), np.median(da.max(1)), da.max(1).max()], 2),
      "run2", np.round([db.max(1).min(), np.median(db.max(1)), db.max(1).max()], 2))
print("mean done - CTA median by warp index:", " ".join(f"{v:+.1f}" for v in ((a + b) / 2).mean(axis=0)))

# ---- what predicts a warp's lateness: regression on plan features (both runs averaged)
h = dm.download()
rp = h.row_pointers.astype(np.int64)
T = np.where(rp[1:] > rp[:-1], (rp[1:] - (rp[:-1] & ~7) + 255) // 256, 0)
n_r = np.where(T >= 8, T // 8, 1)
rows_of = np.zeros(148 * 32)
for k in range(148 * 32):
    u_left, r, j = int(rec[k, 0]), int(rec[k, 1]), int(rec[k, 2])
    cnt = 0
    while u_left > 0:
        take = min(int(n_r[r]) - j, u_left)
        cnt += 1
        u_left -= take
        r += 1
        j = 0
    rows_of[k] = cnt
splits = ((rec[:, 8].view(np.int32) >= 0).astype(int) + (rec[:, 9].view(np.int32) >= 0).astype(int)).astype(np.float64)
y_dev = ((a + b) / 2).reshape(-1)
wi = np.tile(np.arange(32), 148).astype(np.float64)
el = elems.reshape(-1).astype(np.float64)
# deviations from the CTA mean for the per-warp features
def dev(v):
    v = v.reshape(148, 32)
    return (v - v.mean(axis=1, keepdims=True)).reshape(-1)
X = np.stack([dev(el), dev(rows_of), dev(splits), dev(wi)], axis=1)
ok = np.isfinite(y_dev)
coef, *_ = np.linalg.lstsq(X[ok], y_dev[ok], rcond=None)
pred = X @ coef
r2 = 1 - np.var(y_dev[ok] - pred[ok]) / np.var(y_dev[ok])
print("regression of done - CTA median (us) on [elements, rows, split pieces, warp index] deviations:")
print("  coef:", [f"{c:.3e}" for c in coef], f" R^2 {r2:.3f}")
print(f"  elements std {dev(el).std():.0f}, rows std {dev(rows_of).std():.2f}, splits std {dev(splits).std():.2f}")
print(f"  us per 1000 elements {coef[0] * 1e3:.3f}; us per row {coef[1]:.3f}; us per split piece {coef[2]:.3f}; us per warp index {coef[3]:.4f}")
