"""Per-op timeline of the persistent chain kernel (trace build, thread 0 of every CTA):
MACKO_LIB=.../libmacko_cuda_trace.so python tools/trace_chain.py [--layers 8]
Stamps per op k < 32: 0 loop top, 1 barrier passed, 2 x staged, 3 thread 0's warp done with op k,
4 op k+1 set up (record + first fills issued)."""
import argparse
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("MACKO_LIB", os.path.join(ROOT, "paper_2511_13061_b200", "libmacko_cuda_trace.so"))
sys.path.insert(0, ROOT)
from paper_2511_13061_b200 import _lib, decoder_chain as D, macko as M  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--layers", type=int, default=8)
a = p.parse_args()
ch = D.SparseDecoderChain(D.ChainShape(a.layers, 4096, 11008), density=0.5)
M.gen_vector(ch.acts["h"], 4096, seed=1)
for _ in range(2):
    ch.forward_token_persistent()
torch.cuda.synchronize()
L = _lib.load()
L.macko_trace_read.argtypes = [C.c_void_p, C.c_size_t]
buf = np.zeros(148 * 32 * 8, np.uint64)
assert L.macko_trace_read(buf.ctypes.data, buf.size) == 0
t = buf.reshape(148, 32, 8).astype(np.int64)
t0 = t[:, 0, 0].min()
r = (t - t0) / 1e3
names = ["qkv", "o", "gate_up", "down"]
print("op       top(max)  barrier(min/max)   staged(max)  done(min/med/max)      next set(max)")
for k in range(min(32, 4 * a.layers)):
    print(f"{k:2d} {names[k % 4]:8s} {r[:, k, 0].max():8.2f}  {r[:, k, 1].min():8.2f}/{r[:, k, 1].max():8.2f}  "
          f"{r[:, k, 2].max():8.2f}  {r[:, k, 3].min():8.2f}/{np.median(r[:, k, 3]):8.2f}/{r[:, k, 3].max():8.2f}  "
          f"{r[:, k, 4].max():8.2f}")
