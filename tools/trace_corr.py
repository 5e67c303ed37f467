"""Is the per-warp completion spread of one SpMV launch deterministic?  Two traced launches of the
same matrix (trace build, make trace): correlation of each warp's done time relative to its CTA's
median, and of that with the warp's element count and row count (from the plan records).
    MACKO_LIB=paper_2511_13061_b200/libmacko_cuda_trace.so python tools/trace_corr.py"""
import ctypes as C
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
L.macko_trace_read.argtypes = [C.c_void_p, C.c_size_t]
flush = torch.ones(256 << 20, dtype=torch.float32, device="cuda")


def one():
    for _ in range(3):
        dm.spmv_into(x, y)
    flush.sum()
    torch.cuda.synchronize()
    dm.spmv_into(x, y)
    torch.cuda.synchronize()
    buf = np.zeros(148 * 32 * 8, np.uint64)
    assert L.macko_trace_read(buf.ctypes.data, buf.size) == 0
    t = buf.reshape(148, 32, 8).astype(np.int64)
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
