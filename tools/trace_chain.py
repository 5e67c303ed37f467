"""Op-by-op timeline of the PDL-chained decoder SpMVs (trace build, make trace): one token of the
32-layer Llama2-7B chain is replayed; the last 8 SpMV launches (kTraceSlots) are read back and,
for each op, the first warp start, plan records, griddepcontrol.wait passed, x staged and warp
completion percentiles are printed relative to the first op's first warp.
    MACKO_LIB=paper_2511_13061_b200/libmacko_cuda_trace.so python tools/trace_chain.py"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("MACKO_LIB", os.path.join(ROOT, "paper_2511_13061_b200", "libmacko_cuda_trace.so"))
sys.path.insert(0, ROOT)
from paper_2511_13061_b200 import _lib, macko as M  # noqa: E402
from paper_2511_13061_b200 import decoder_chain as D  # noqa: E402

ch = D.SparseDecoderChain(D.LLAMA2_7B, density=0.5)
M.gen_vector(ch.acts["h"], D.LLAMA2_7B.hidden, seed=1)
L = _lib.load()
L.macko_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
L.macko_trace_slot_counter.restype = ctypes.c_uint
S = 8
g = ch.capture(pdl=True)  # warm-up token + captured token: slots are baked into the graph nodes
c1 = L.macko_trace_slot_counter()
c0 = c1 - ch.kernels_per_token
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
buf = np.zeros(S * 148 * 32 * 8, np.uint64)
assert L.macko_trace_read(buf.ctypes.data, buf.size) == 0
t = buf.reshape(S, 148 * 32, 8).astype(np.int64)
order = [(c1 - S + i) % S for i in range(S)]  # oldest first
base = None
names = ["start", "record", "walk set", "gdc.wait", "x staged", "mbar", "done", "ring issued"]
print(f"launches this token: {c1 - c0}; last {S} ops (oldest first), us relative to the first op's first warp")
prev_done = None
for k, slot in enumerate(order):
    tt = t[slot]
    ok = tt[:, 0] > 0
    if base is None:
        base = tt[ok, 0].min()
    rel = (tt - base) / 1e3
    def q(i, p):
        col = rel[ok, i][tt[ok, i] > 0]
        return np.percentile(col, p) if col.size else float("nan")
    line = (f"op {k}: start {q(0, 0):8.2f}..{q(0, 100):8.2f}  gdc {q(3, 50):8.2f} (max {q(3, 100):8.2f})  "
            f"x staged {q(4, 50):8.2f}  done p10/50/90/max {q(6, 10):8.2f} {q(6, 50):8.2f} {q(6, 90):8.2f} {q(6, 100):8.2f}")
    if prev_done is not None:
        line += f"  | gap last-done(prev) -> gdc(max) {q(3, 100) - prev_done:6.2f}"
    prev_done = q(6, 100)
    print(line, flush=True)
    cta_last = np.where(tt[:, 6] > 0, rel[:, 6], np.nan).reshape(148, 32)
    cl = np.nanmax(cta_last, axis=1)
    print(f"      CTA last warp min/med/max {np.nanmin(cl):8.2f} {np.nanmedian(cl):8.2f} {np.nanmax(cl):8.2f}; "
          f"CTA first start min/max {np.nanmin(rel[ok, 0]):8.2f} {np.nanmax(rel[ok, 0]):8.2f}")

# the prologue of each op's latest-starting CTA, stage by stage (median over its warps)
print("latest-starting CTA per op: stage stamps (median over its warps), us")
for k, slot in enumerate(order):
    tt = t[slot]
    rel = (tt - base) / 1e3
    st = np.where(tt[:, 0] > 0, rel[:, 0], np.nan).reshape(148, 32)
    c = int(np.nanargmax(np.nanmin(st, axis=1)))
    rows = rel.reshape(148, 32, 8)[c]
    vals = {n: np.median(rows[:, i][tt.reshape(148, 32, 8)[c][:, i] > 0]) for i, n in enumerate(names)}
    print(f"op {k} CTA {c}: " + "  ".join(f"{n} {vals[n]:8.2f}" for n in
                                            ["start", "record", "mbar", "ring issued", "walk set", "gdc.wait", "x staged", "done"]))
