import torch, time, os, sys
sys.path.insert(0, '.')
from paper_2511_13061_b200 import macko as M
torch.cuda.set_device(0)
R, C = 36864, 12288
dense = torch.empty((R, C), dtype=torch.float16, device="cuda")
M.gen_dense(dense, R, C, 0.5, seed=1234)
for i in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    dm = M.DeviceMatrix.from_dense(dense)
    torch.cuda.synchronize(); print("from_dense wall ms", (time.perf_counter() - t) * 1e3, flush=True)
    dm.close()
