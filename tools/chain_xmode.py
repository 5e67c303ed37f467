"""Timing: Llama2-7B decode chain, PDL graph vs persistent kernel, for a forced x_mode."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_13061_b200 import decoder_chain as D  # noqa: E402
from paper_2511_13061_b200 import macko as M  # noqa: E402

ch = D.SparseDecoderChain(D.LLAMA2_7B, density=0.5)
M.gen_vector(ch.acts["h"], 4096, seed=1)
for xm in [int(v) for v in sys.argv[1:]] or [-1]:
    for mats in ch.mats:
        for m in mats.values():
            m.configure(xm)
    ch._chain = None
    g = ch.capture(pdl=True)
    s = torch.cuda.Stream()
    ch.forward_token_persistent()
    torch.cuda.synchronize()
    gp = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gp, stream=s):
        ch.forward_token_persistent(s)
    for name, graph in (("pdl", g), ("persistent", gp)):
        for _ in range(3):
            graph.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            graph.replay()
        b.record()
        b.synchronize()
        print(f"x_mode {xm} {name}: {a.elapsed_time(b) / 10 * 1e3:.1f} us/token")
