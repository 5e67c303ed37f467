"""Kernel experiments: per-launch CUDA-event times of the SpMV for several densities / shapes, with
the SM clock sampled (NVML) during the timed launches, so variants built with different -D
knobs (MACKO_LIB=path/to/variant.so) compare in SM cycles, not only µs.

    MACKO_LIB=build/variants/libX.so python tools/spmv_time.py --shapes 36864x12288@0.5,11008x4096@0.5
"""
import argparse
import os
import statistics
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_13061_b200 import macko as M  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--shapes", default="36864x12288@0.5")
p.add_argument("--n", type=int, default=100)
p.add_argument("--soak", type=float, default=0.5)
p.add_argument("--x-mode", type=int, default=-1)
p.add_argument("--bits", type=int, default=4, help="b_delta of the format")
p.add_argument("--tag", default=os.environ.get("MACKO_LIB", "default"))
p.add_argument("--no-flush", action="store_true", help="never flush L2 between launches (L2-resident runs)")
p.add_argument("--check", type=int, default=1, help="compare y with the oracle order (small shapes only)")
a = p.parse_args()

try:
    import pynvml

    pynvml.nvmlInit()
    nv = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
except Exception:  # pragma: no cover
    nv = None


def sample_clock(stop, out):
    while not stop.is_set():
        if nv is not None:
            out.append(pynvml.nvmlDeviceGetClockInfo(nv, pynvml.NVML_CLOCK_SM))
        time.sleep(0.005)


st = torch.cuda.current_stream()
l2 = torch.cuda.get_device_properties(0).L2_cache_size
flush = torch.ones(max(2 * l2, 256 << 20) // 4, dtype=torch.float32, device="cuda")
for spec in a.shapes.split(","):
    shp, d = spec.split("@")
    R, C = (int(v) for v in shp.split("x"))
    d = float(d)
    dense = torch.empty((R, C), dtype=torch.float16, device="cuda")
    M.gen_dense(dense, R, C, d, seed=1234)
    dm = M.DeviceMatrix.from_dense(dense, b_delta=a.bits)
    x = torch.empty(C, dtype=torch.float16, device="cuda")
    M.gen_vector(x, C, seed=4321)
    y = torch.empty(R, dtype=torch.float16, device="cuda")
    if a.x_mode != -1:
        dm.configure(a.x_mode)
    ok = "-"
    if a.check and R * C <= 64 << 20:
        from oracle import oracle as O
        from tests.helpers import b200_y, to_host_u16

        dm.spmv_into(x, y, st)
        torch.cuda.synchronize()
        hm = dm.download()
        m = O.Macko(hm.rows, hm.cols, a.bits, hm.values, hm.packed_deltas, hm.row_pointers)
        ok = "ok" if (to_host_u16(y) == b200_y(m, to_host_u16(x))).all() else "MISMATCH"
    del dense
    need_flush = dm.traffic_bytes < 3 * l2 and not a.no_flush
    t_end = time.time() + a.soak
    while time.time() < t_end:
        for _ in range(10):
            dm.spmv_into(x, y, st)
        torch.cuda.synchronize()
    clocks, stop = [], threading.Event()
    th = threading.Thread(target=sample_clock, args=(stop, clocks))
    th.start()
    ts = []
    for i in range(a.n):
        if need_flush:
            flush.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        dm.spmv_into(x, y, st)
        e1.record(st)
        if need_flush:
            e1.synchronize()
        ts.append((e0, e1))
    torch.cuda.synchronize()
    stop.set()
    th.join()
    us = [e0.elapsed_time(e1) * 1e3 for e0, e1 in ts]
    med = statistics.median(us)
    if need_flush:  # per-launch events after a flush tick in ~2.05 us steps: amortise instead
        ea, eb, ec, ed = (torch.cuda.Event(enable_timing=True) for _ in range(4))
        ea.record(st)
        for _ in range(a.n):
            flush.sum()
            dm.spmv_into(x, y, st)
        eb.record(st)
        ec.record(st)
        for _ in range(a.n):
            flush.sum()
        ed.record(st)
        torch.cuda.synchronize()
        med = (ea.elapsed_time(eb) - ec.elapsed_time(ed)) * 1e3 / a.n
    # back-to-back launches (no flush): the mean over the whole run resolves below the event tick
    mean = ts[0][0].elapsed_time(ts[-1][1]) * 1e3 / a.n if not need_flush else float("nan")
    mhz = statistics.median(clocks) if clocks else float("nan")
    li = dm.launch_info()
    print(f"{a.tag:40s} {R}x{C}@{d}: {med:8.2f} us  {dm.traffic_bytes / med / 1e3:7.1f} GB/s  "
          f"sm {mhz:6.0f} MHz  {med * mhz / 1e3:7.1f} kcyc  mean {mean:8.2f} us  x_mode {li.x_in_smem} y {ok}", flush=True)
    dm.close()
    torch.cuda.empty_cache()
