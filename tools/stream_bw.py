"""Sustained vs burst HBM streaming on this box (context for the SpMV's roofline fraction):
a copy (read + write) and a read-only reduction over 1 GiB, timed with CUDA events, before and
after a soak of back-to-back SpMVs, with the SM clock sampled (NVML)."""
import os
import statistics
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_13061_b200 import macko as M  # noqa: E402

import pynvml  # noqa: E402

pynvml.nvmlInit()
nv = pynvml.nvmlDeviceGetHandleByIndex(0)


def timed(fn, n, nbytes):
    clocks, stop = [], threading.Event()

    def samp():
        while not stop.is_set():
            clocks.append(pynvml.nvmlDeviceGetClockInfo(nv, pynvml.NVML_CLOCK_SM))
            time.sleep(0.005)

    th = threading.Thread(target=samp)
    th.start()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for a, b in evs:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    ms = statistics.median(a.elapsed_time(b) for a, b in evs)
    return nbytes / (ms * 1e-3) / 1e9, ms * 1e3, statistics.median(clocks) if clocks else float("nan")


N = 1 << 29  # 1 GiB of fp16
a = torch.ones(N, dtype=torch.float16, device="cuda")
b = torch.empty_like(a)
R, C = 36864, 12288
dense = torch.empty((R, C), dtype=torch.float16, device="cuda")
M.gen_dense(dense, R, C, 0.5, seed=1234)
dm = M.DeviceMatrix.from_dense(dense)
del dense
x = torch.empty(C, dtype=torch.float16, device="cuda")
M.gen_vector(x, C, seed=4321)
y = torch.empty(R, dtype=torch.float16, device="cuda")
for label in ("burst", "after 2 s soak"):
    if label != "burst":
        t_end = time.time() + 2.0
        while time.time() < t_end:
            for _ in range(20):
                dm.spmv_into(x, y)
            torch.cuda.synchronize()
    for name, fn, nb, n in (("copy 1GiB", lambda: b.copy_(a), 4 * N, 20),
                            ("read 1GiB (sum)", lambda: a.sum(), 2 * N, 20),
                            ("spmv 36864x12288@0.5", lambda: dm.spmv_into(x, y), dm.traffic_bytes, 100)):
        gbs, us, mhz = timed(fn, n, nb)
        print(f"{label:16s} {name:22s} {gbs:8.1f} GB/s  {us:9.2f} us  sm {mhz:6.0f} MHz", flush=True)
