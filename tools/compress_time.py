"""Wall time of macko_dev_from_dense (dense 36864x12288 fp16 @50 % already on the device), repeated:
the first call pays lazy module loading and first-touch allocation; later calls reuse cached
device blocks (capi BlockCache; MACKO_NO_BLOCK_CACHE=1 disables it).  MACKO_TIMING=1 prints phases."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_13061_b200 import macko as M  # noqa: E402

torch.cuda.set_device(0)
R, C = 36864, 12288
dense = torch.empty((R, C), dtype=torch.float16, device="cuda")
M.gen_dense(dense, R, C, 0.5, seed=1234)
for i in range(int(os.environ.get("REPS", "4"))):
    torch.cuda.synchronize()
    t = time.perf_counter()
    dm = M.DeviceMatrix.from_dense(dense)
    torch.cuda.synchronize()
    print("from_dense wall ms", round((time.perf_counter() - t) * 1e3, 3), flush=True)
    dm.close()
