import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_13061_b200 import macko as M
for R, C in ((4096, 4096), (12288, 4096)):
    dense = torch.empty((R, C), dtype=torch.float16, device="cuda")
    M.gen_dense(dense, R, C, 0.5, seed=1)
    dm = M.DeviceMatrix.from_dense(dense)
    x = torch.empty(C, dtype=torch.float16, device="cuda"); M.gen_vector(x, C, seed=2)
    y = torch.empty(R, dtype=torch.float16, device="cuda")
    for skew in (0, 2000):
        dm.set_chain_skew(skew)
        li = dm.launch_info()
        recs, splits = dm.plan_records()
        el = (recs[:, 4].astype(np.int64) - recs[:, 3].astype(np.int64)).reshape(li.grid, -1).sum(1)
        for pdl in (False, True):
            for _ in range(3): dm.spmv_into(x, y, pdl=pdl)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(50): dm.spmv_into(x, y, pdl=pdl)
            e1.record(); torch.cuda.synchronize()
            print(R, C, "skew", skew, "pdl", pdl, f"{e0.elapsed_time(e1)*1e3/50:.2f} us", "splits", li.n_split_rows,
                  "units", li.n_units, "cta elems first/last", el[:3], el[-3:], flush=True)
