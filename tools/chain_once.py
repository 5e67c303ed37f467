"""Profiling driver: build the Llama2-7B decode chain and run a few tokens with plain stream
launches (PDL on), so ncu sees every SpMV of the chain."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_13061_b200 import decoder_chain as D  # noqa: E402
from paper_2511_13061_b200 import macko as M  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--layers", type=int, default=32)
p.add_argument("--tokens", type=int, default=2)
p.add_argument("--pdl", type=int, default=1)
a = p.parse_args()
ch = D.SparseDecoderChain(D.ChainShape(a.layers, 4096, 11008), density=0.5)
M.gen_vector(ch.acts["h"], 4096, seed=1)
for _ in range(a.tokens):
    ch.forward_token(pdl=bool(a.pdl))
torch.cuda.synchronize()
print("ok")
