"""Decode-chain timing for kernel variants: the 32-layer Llama2-7B SpMV chain (BASELINE config 4),
PDL-chained SpMVs in one CUDA graph per token, CUDA events around each replay.
    MACKO_LIB=build/variants/libmacko_cuda_X.so python tools/chain_time.py --tag X"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_13061_b200 import decoder_chain as D  # noqa: E402
from paper_2511_13061_b200 import macko as M  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--tokens", type=int, default=20)
p.add_argument("--tag", default=os.environ.get("MACKO_LIB", "default"))
a = p.parse_args()
ch = D.SparseDecoderChain(D.LLAMA2_7B, density=0.5)
M.gen_vector(ch.acts["h"], D.LLAMA2_7B.hidden, seed=1)
g = ch.capture(pdl=True)
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.tokens)]
for e0, e1 in evs:
    e0.record()
    g.replay()
    e1.record()
torch.cuda.synchronize()
us = sorted(e0.elapsed_time(e1) * 1e3 for e0, e1 in evs)
print(f"{a.tag:30s} chain: median {us[len(us) // 2]:8.1f} us/token  min {us[0]:8.1f}  "
      f"{ch.traffic_bytes / (us[len(us) // 2] * 1e-6) / 1e9:7.1f} GB/s", flush=True)
