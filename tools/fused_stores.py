"""Fused all-gather stores on one GPU: the SpMV's peer table gets this rank's own y plus one local
buffer standing in for a remote rank's y, so the kernel's peer-store path runs without NVLink.
Checks the stand-in equals y and times fused vs plain launches (events, no flush).  Under ncu,
the write-request counts of the fused launch are the NVLink write packets a real peer would see:
  ncu --metrics lts__t_requests_srcunit_tex_op_write.sum,smsp__inst_executed_op_global_st.sum \
      -k regex:macko_spmv python tools/fused_stores.py 36864 12288 0.5 --iters 1
"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2511_13061_b200 import macko as M  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("rows", type=int)
ap.add_argument("cols", type=int)
ap.add_argument("density", type=float)
ap.add_argument("--iters", type=int, default=200)
args = ap.parse_args()

dev = torch.device("cuda", 0)
A = torch.empty(args.rows, args.cols, dtype=torch.float16, device=dev)
M.gen_dense(A, args.rows, args.cols, args.density, seed=3)
dm = M.DeviceMatrix.from_dense(A)
del A
x = torch.empty(args.cols, dtype=torch.float16, device=dev)
M.gen_vector(x, args.cols, seed=4)
y = torch.zeros(args.rows, dtype=torch.float16, device=dev)
other = torch.full((args.rows,), -1.0, dtype=torch.float16, device=dev)
flags = torch.zeros(2, dtype=torch.int32, device=dev)
dm.set_peers([y.data_ptr(), other.data_ptr()], [flags.data_ptr(), flags.data_ptr() + 4])
dm.set_peer_bank(1, [y.data_ptr(), other.data_ptr()])
dm.spmv_into(x, y, peers=True)
torch.cuda.synchronize()
peer_ok = torch.equal(y.view(torch.int16), other.view(torch.int16))
y2 = torch.zeros_like(y)
dm.spmv_into(x, y2)
dm.spmv_into(x, y2, pdl=True)  # the chain instance without peers (ncu: compare with the fused launch)
torch.cuda.synchronize()
assert torch.equal(y.view(torch.int16), y2.view(torch.int16)), "fused y differs from plain y"


def timed(fn):
    for _ in range(10):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(args.iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) * 1e3 / args.iters


if args.iters > 1:
    tp = timed(lambda: dm.spmv_into(x, y2))
    tf = timed(lambda: dm.spmv_into(x, y, peers=True))
    print(f"{args.rows}x{args.cols}@{args.density}: plain {tp:.2f} us  fused(1 stand-in peer) {tf:.2f} us  peer copy {'ok' if peer_ok else 'DIFFERS'}")
else:
    print(f"peer copy {'ok' if peer_ok else 'DIFFERS'}")
dm.set_peers([], [])
dm.close()
