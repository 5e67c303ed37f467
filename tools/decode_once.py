"""One Llama2-7B decode step (MACKO linears) for an ncu launch list: per-kernel durations."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_13061_b200 import llama as L  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "macko"
torch.cuda.set_device(0)
w = L.LlamaWeights(L.LLAMA2_7B, density=0.5, keep_dense=(kind == "dense"), macko=(kind == "macko"))
d = L.LlamaDecoder(w, kind)
d.reset()
for _ in range(3):
    d.step()
torch.cuda.synchronize()
d.step()  # the profiled step (ncu -s skips the build and warm-up launches)
torch.cuda.synchronize()
