"""Debug: order-0/1 SpMV vs the oracle on random shapes, one case at a time (first failure)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_2511_13061_b200 import macko as M  # noqa: E402
from tests.helpers import b200_y, to_dev, to_host_u16  # noqa: E402

order = int(sys.argv[1]) if len(sys.argv) > 1 else 1
rng = np.random.default_rng(5)
cases = [(1, 1, 1.0), (1, 3000, 0.5), (3, 5000, 0.5), (64, 64, 0.5), (1000, 16000, 0.5), (333, 777, 0.3),
         (4096, 4096, 0.5), (5000, 300, 0.9), (20, 70000, 0.5)]
cases += [(int(rng.integers(1, 3000)), int(rng.integers(1, 9000)), float(rng.choice([0.01, 0.1, 0.5, 0.9, 1.0])))
          for _ in range(20)]
for R, C, d in cases:
    A = O.gen_dense(R, C, d, R * 7 + C)
    if R > 3:
        A[1::3] = 0
    x = O.gen_vector(C, 9)
    m = O.encode_dense(A)
    dm = M.DeviceMatrix.from_dense(to_dev(A))
    dm.set_order(order)
    y = to_host_u16(M.spmv(dm, to_dev(x)))
    torch.cuda.synchronize()
    ref = b200_y(order, m, x)
    bad = np.flatnonzero(y != ref)
    print((R, C, d), "ok" if bad.size == 0 else f"BAD {bad.size} first rows {bad[:8]}", flush=True)
    dm.close()
