#!/usr/bin/env python
"""bench.py — MACKO SpMV on B200 (BASELINE.json metric: effective HBM GB/s & µs,
36864x12288 fp16 @ 50 % sparsity vs cuBLAS GEMV).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--sweep] [--chain] [--strong] [--fused] [--no-decode] [--no-cpu-baseline]

One step = one SpMV y = A·x over the resident MACKO matrix (GPU-compressed from a synthetic
random-unstructured fp16 matrix of the configured shape; inputs resident in HBM).

N > 1 ranks (one per GPU; `--gpus N` re-launches itself under torch.distributed.run when
WORLD_SIZE is unset): weak scaling of the headline — rank g owns rows [g·R, (g+1)·R) of an
(N·R) x C matrix; a step is NCCL broadcast(x) + the slab SpMV + NCCL all_gather(y), timed on the
device and reduced as the max over ranks.  Beside it, `strong` reports BASELINE config 5
(131072x32768 @50 / 90 %, rows/N per rank): per-rank SpMV µs, the collectives' µs alone, the full
NCCL step and the step with the all-gather fused into the SpMV kernel (peer stores over NVLink).

`value` = algorithmic bytes of all ranks (spmv_traffic) / device time of one
step.  Inputs larger than 3x L2 stream from HBM every step; smaller ones get an L2 flush (a read
of a 2xL2 buffer) before every step, outside the step's events.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import socket
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SpMV effective HBM GB/s & µs, 36864×12288 fp16 @50% sparsity vs cuBLAS GEMV"
HEADLINE = dict(rows=36864, cols=12288, density=0.5)
CONFIG5 = dict(rows=131072, cols=32768)
SEED_A, SEED_X = 1234, 4321


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=100)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--rows", type=int, default=HEADLINE["rows"])
    p.add_argument("--cols", type=int, default=HEADLINE["cols"])
    p.add_argument("--density", type=float, default=HEADLINE["density"])
    p.add_argument("--sweep", action="store_true", help="30/50/70/90 %% sparsity, Llama shapes, 131072x32768")
    p.add_argument("--chain", action="store_true", help="Llama2-7B 32-layer decode SpMV chain (config 4) vs cuBLAS")
    p.add_argument("--no-decode", action="store_true", help="skip the Llama2-7B decode E2E (MACKO vs cuBLAS tokens/s)")
    p.add_argument("--strong", action="store_true", help="config 5 strong scaling also at N = 1")
    p.add_argument("--chain-tokens", type=int, default=20)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--soak-s", type=float, default=0.0, help="untimed back-to-back SpMVs before the timed steps")
    p.add_argument("--sustain-s", type=float, default=1.5,
                   help="then this long back-to-back and the K steps again under the settled power-cap clocks (0: skip)")
    p.add_argument("--x-mode", type=int, default=-1, help="x gathers: -1 auto, 0 texture, 1 smem table, 6/7/8/10 split")
    p.add_argument("--ctas", type=int, default=0, help="cap on SpMV CTAs (k/4 of the persistent grid, 0 = all)")
    p.add_argument("--fused", action="store_true", help="N > 1: also the chain with the all-gather fused into the SpMV")
    return p.parse_args()


def maybe_spawn(args) -> None:
    """`--gpus N` without a launcher: re-exec under torch.distributed.run, one rank per GPU."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ or args.impl == "reference":
        return
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def sparsity_pct(d: float) -> int:
    return int(round((1 - d) * 100))


def workload_config(R: int, C: int, d: float, world: int) -> dict:
    """The `config` object — identical in both arms (same_config)."""
    sp = sparsity_pct(d)
    if world > 1:
        wl = (f"{R}x{C} fp16 @{sp}% sparsity per rank (random unstructured), weak scaling: {world * R}x{C} "
              f"row-sharded over {world} GPUs, NCCL broadcast x + all_gather y per SpMV")
    else:
        wl = f"{R}x{C} fp16 @{sp}% sparsity (random unstructured), single SpMV"
    return {"workload": wl, "rows": R * world, "rows_per_rank": R, "cols": C, "density": d, "b_delta": 4,
            "parallelism": f"row-shard x{world}" if world > 1 else "single GPU"}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ---------------------------------------------------------------------------------- clocks
_NVML_SAMPLER = r"""
import sys, time, pynvml
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(int(sys.argv[1]))
reasons = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
print("max", pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM), flush=True)
while True:
    t = time.time()
    try:
        c = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
    except Exception:
        c = -1
    try:
        r = int(reasons(h))
    except Exception:
        r = -1
    try:
        w = pynvml.nvmlDeviceGetPowerUsage(h) / 1e3
    except Exception:
        w = -1.0
    print(f"{t:.6f} {c} {r} {w:.1f}", flush=True)
    time.sleep(0.001)
"""


class ClockSampler:
    """SM clock, throttle reasons and power of one GPU, sampled every ~1 ms by a separate process
    (NVML; no GIL shared with the launching thread).  `mark()` brackets a timed region with
    wall-clock stamps; `summary()` keeps the samples inside it."""
    REASON_BITS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap",
                   0x80: "hw_power_brake_slowdown"}

    def __init__(self, index: int):
        self.proc = None
        self.sm_max = None
        try:
            self.proc = subprocess.Popen([sys.executable, "-c", _NVML_SAMPLER, str(index)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            first = self.proc.stdout.readline().split()  # ready: NVML initialised
            self.sm_max = float(first[1]) if len(first) == 2 and first[0] == "max" else None
        except Exception:
            self.proc = None
        self.lines = []

    def collect(self):
        """Stop the sampler; returns the samples (t, sm_mhz, reasons, watts)."""
        if self.proc is None:
            return []
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        self.proc = None
        rows = []
        for line in out.splitlines():
            parts = line.split()
            if len(parts) == 4:
                try:
                    rows.append((float(parts[0]), float(parts[1]), int(parts[2]), float(parts[3])))
                except ValueError:
                    pass
        self.lines = rows
        return rows

    def summary(self, t0: float, t1: float):
        rows = [r for r in self.lines if t0 <= r[0] <= t1 and r[1] > 0]
        widened = 0.0
        while not rows and widened < 0.05 and self.lines:  # a short region between two polls: the
            widened += 0.002                                  # nearest samples, window stated below
            rows = [r for r in self.lines if t0 - widened <= r[0] <= t1 + widened and r[1] > 0]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": self.sm_max, "reasons": ["no samples"], "source": "nvml"}
        reasons = sorted({n for r in rows if r[2] >= 0 for b, n in self.REASON_BITS.items() if r[2] & b})
        return {"sm_mhz": statistics.median(r[1] for r in rows), "sm_max_mhz": self.sm_max,
                "sm_mhz_min": min(r[1] for r in rows), "reasons": reasons, "samples": len(rows),
                "power_w_median": round(statistics.median(r[3] for r in rows), 1),
                "source": "nvml every ~1 ms (separate process) during the timed steps" + (
                    f" (region shorter than the poll interval: samples within {widened * 1e3:.0f} ms of it)" if widened else "")}


# ---------------------------------------------------------------------------------- reference arm
def run_reference(args, rank: int, world: int):
    """The reference's own CPU path (oracle/_ref: the reference fp16.cpp / bitpack.cpp / headers
    + SPEC-restated bodies) on the box's host cores, same config / metric / unit.  Rows are
    independent, so at N > 1 the sample is one rank's slab of the (N·R) x C matrix: GB/s is a
    rate, and the whole job's time is N x the slab's."""
    if rank != 0:
        return
    from oracle import oracle as O

    kind = "reference" if O.ref_available() else "port"
    threads = host_cores()
    R, C, d = args.rows, args.cols, args.density
    n = max(world, args.gpus)
    t0 = time.time()
    A = O.gen_dense_rows(0, R, C, d, SEED_A, False, threads)
    if kind == "reference":
        rm = O.RefMatrix.encode(A, 4)
        m = rm.to_macko(R, C, 4)
        run = lambda x: rm.spmv(x, R, threads)  # noqa: E731
    else:
        m = O.encode_dense(A, 4, threads)
        run = lambda x: O.reference_spmv(m, x, threads)  # noqa: E731
    del A
    build_s = time.time() - t0
    x = O.gen_vector(C, SEED_X)
    bytes_sample = O.spmv_traffic_bytes(R, C, m.pad_nnz, 4)
    t1 = time.perf_counter()
    run(x)
    one = time.perf_counter() - t1
    steps = args.steps
    budget = 120.0
    if one * (steps + args.warmup) > budget:  # keep the whole arm within a few minutes
        steps = max(3, int(budget / max(one, 1e-6)) - args.warmup)
    for _ in range(min(max(args.warmup, 1), 3)):
        run(x)
    times = []
    for _ in range(steps):
        t1 = time.perf_counter()
        run(x)
        times.append(time.perf_counter() - t1)
    ms = statistics.median(times) * 1e3
    gbs = bytes_sample / (ms * 1e-3) / 1e9
    sample = (f"{'rows [0, %d) of the %dx%d matrix (one rank slab; rows independent), ' % (R, n * R, C) if n > 1 else ''}"
              f"{R}x{C} @{sparsity_pct(d)}% sparsity, reference_spmv (reference encoder build {build_s:.1f} s), "
              f"{steps} timed steps (median), {threads} threads std::thread row partition, CPU {cpu_model()}")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(gbs, 3), "unit": "GB/s", "n_gpus": n,
        "steps": steps, "warmup": args.warmup, "ms_per_step": round(ms * n, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f16", "data": "synthetic (counter-hash generator)",
        "config": workload_config(R, C, d, n),
        "pad_nnz_sample": m.pad_nnz, "bytes_per_spmv_sample": bytes_sample,
        "cpu_baseline": {"value": round(gbs, 3), "unit": "GB/s", "cores": threads, "kind": kind, "sample": sample},
        "e2e": {"value": round(gbs, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------- timing helpers
class Timer:
    """CUDA-event timing on the launching stream with an optional L2 flush before every rep."""

    def __init__(self, torch, stream, flush_buf):
        self.torch, self.stream, self.flush_buf = torch, stream, flush_buf

    def flush(self):
        self.flush_buf.sum()  # reads 2x L2 of clean lines: evicts without dirty write-back

    def run(self, fn, reps: int, warmup: int = 3, flush: bool = False):
        torch = self.torch
        for _ in range(warmup):
            fn()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
        torch.cuda.synchronize()
        for a, b in evs:
            if flush:
                self.flush()
            a.record(self.stream)
            fn()
            b.record(self.stream)
        torch.cuda.synchronize()
        return [a.elapsed_time(b) for a, b in evs]  # ms

    def device_ms(self, fn, reps: int, flush: bool, warmup: int = 3) -> float:
        """Per-call device time (ms): median of per-call events back to back, or, with an L2 flush
        before every call, the amortised mean (run_amortized)."""
        if flush:
            return self.run_amortized(fn, reps, warmup)
        return statistics.median(self.run(fn, reps, warmup))

    def run_amortized(self, fn, reps: int, warmup: int = 3) -> float:
        """Mean device time (ms) of fn with an L2 flush before every rep: one event pair around
        reps x (flush; fn) minus one around reps x flush.  On B200 an event recorded right after
        the flush kernel ticks in ~2.05 us steps, so per-rep events quantise kernels of 10-30 us by
        up to 10 %; the two long intervals do not."""
        torch = self.torch
        for _ in range(warmup):
            self.flush()
            fn()
        a, b, c, d = (torch.cuda.Event(enable_timing=True) for _ in range(4))
        torch.cuda.synchronize()
        a.record(self.stream)
        for _ in range(reps):
            self.flush()
            fn()
        b.record(self.stream)
        c.record(self.stream)
        for _ in range(reps):
            self.flush()
        d.record(self.stream)
        torch.cuda.synchronize()
        return max(a.elapsed_time(b) - c.elapsed_time(d), 1e-6) / reps


def allmax(torch, dist, dev, vals):
    t = torch.tensor(vals, device=dev, dtype=torch.float64)
    if dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


def cublas_hsh_gemv():
    """cublasHSHgemvStridedBatched (fp16 in/out, fp32 compute) through the cuBLAS torch loaded —
    the GEMV the paper compares against."""
    import torch

    lib = None
    for name in ("libcublas.so.12", os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cublas", "lib",
                                                 "libcublas.so.12")):
        try:
            lib = ctypes.CDLL(name)
            break
        except OSError:
            continue
    if lib is None:
        return None
    fn = lib.cublasHSHgemvStridedBatched
    c = ctypes
    fn.argtypes = [c.c_void_p, c.c_int, c.c_int, c.c_int, c.POINTER(c.c_float), c.c_void_p, c.c_int, c.c_longlong,
                   c.c_void_p, c.c_int, c.c_longlong, c.POINTER(c.c_float), c.c_void_p, c.c_int, c.c_longlong, c.c_int]
    fn.restype = c.c_int
    setstream = lib.cublasSetStream_v2
    setstream.argtypes = [c.c_void_p, c.c_void_p]
    alpha, beta = c.c_float(1.0), c.c_float(0.0)

    def run(A, x, y):  # A row-major R x C = column-major C x R; y = op_T(A_cm) x
        R, C = A.shape
        h = torch.cuda.current_blas_handle()
        setstream(h, torch.cuda.current_stream().cuda_stream)
        st = fn(h, 1, C, R, c.byref(alpha), A.data_ptr(), C, R * C, x.data_ptr(), 1, C, c.byref(beta),
                y.data_ptr(), 1, R, 1)
        if st != 0:
            raise RuntimeError(f"cublasHSHgemvStridedBatched status {st}")

    return run


def dense_baseline(torch, timer, dense, x, reps, flush):
    """The faster of cublasGemmEx (torch.mv: fp16 in/out, fp32 compute) and
    cublasHSHgemvStridedBatched on the same dense matrix."""
    R, C = dense.shape
    y1 = torch.empty(R, dtype=torch.float16, device=dense.device)
    y2 = torch.empty(R, dtype=torch.float16, device=dense.device)
    out = {}
    out["cublasGemmEx (torch.mv)"] = timer.device_ms(lambda: torch.mv(dense, x, out=y1), reps, flush) * 1e3
    hsh = cublas_hsh_gemv()
    if hsh is not None:
        hsh(dense, x, y2)
        torch.cuda.synchronize()
        if torch.allclose(y1.float(), y2.float(), rtol=2e-2, atol=1e-2):
            out["cublasHSHgemvStridedBatched"] = timer.device_ms(lambda: hsh(dense, x, y2), reps, flush) * 1e3
    best = min(out, key=out.get)
    return best, out[best], {k: round(v, 2) for k, v in out.items()}


# ---------------------------------------------------------------------------------- our arm
def main():
    args = parse()
    maybe_spawn(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    from paper_2511_13061_b200 import macko as M
    from paper_2511_13061_b200.sharded import RowShardedSpmv, device_local_spmv

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    torch.backends.cuda.matmul.allow_fp16_reduced_precision_reduction = False
    stream = torch.cuda.current_stream()
    peak, peak_src = load_peaks()
    R, C, d = args.rows, args.cols, args.density
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush_buf = torch.ones(max(2 * l2, 256 << 20) // 4, dtype=torch.float32, device=dev)
    timer = Timer(torch, stream, flush_buf)

    # ---- build the rank's slab on the device: generator -> GPU compressor (no host copies)
    dense = torch.empty((R, C), dtype=torch.float16, device=dev)
    M.gen_dense(dense, R, C, d, seed=SEED_A, row0=rank * R)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dm = M.DeviceMatrix.from_dense(dense)
    torch.cuda.synchronize()
    compress_s = time.perf_counter() - t0  # first call: lazy module loading, allocator first touch
    dm.close()  # a rebuild (the matrix's device blocks are reused from the library's block cache)
    t0 = time.perf_counter()
    dm = M.DeviceMatrix.from_dense(dense)
    torch.cuda.synchronize()
    compress_warm_s = time.perf_counter() - t0
    if args.x_mode != -1 or args.ctas:
        dm.configure(args.x_mode, args.ctas)
    x = torch.empty(C, dtype=torch.float16, device=dev)
    M.gen_vector(x, C, seed=SEED_X)
    y = torch.empty(R, dtype=torch.float16, device=dev)
    bytes_rank = dm.traffic_bytes
    need_flush = bytes_rank < 3 * l2

    sharded = None
    if world > 1:
        sharded = RowShardedSpmv(R * world, C, device_local_spmv(dm, stream), device=dev)

    def step():
        if sharded is not None:
            sharded(x)
        else:
            dm.spmv_into(x, y, stream)

    # ---- dense cuBLAS GEMV on the same matrix (before freeing the dense copy)
    dense_best = None
    if rank == 0:
        dense_best = dense_baseline(torch, timer, dense, x, max(10, min(args.steps, 50)), need_flush)
    del dense
    torch.cuda.empty_cache()

    # ---- warmup, then the timed region: exactly K steps, per-step device events around the step
    # only, clocks sampled during it (rank 0's GPU)
    sampler = ClockSampler(local) if rank == 0 else None
    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()

    def soak(seconds):
        t_end = time.time() + seconds
        while time.time() < t_end:
            for _ in range(20):
                dm.spmv_into(x, y, stream)
            torch.cuda.synchronize()

    def timed_steps():
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.time()
        for i in range(args.steps):
            if need_flush:
                timer.flush()
            evs[i][0].record(stream)
            step()
            evs[i][1].record(stream)
        torch.cuda.synchronize()
        t1 = time.time()
        if world > 1:
            dist.barrier()
        step_ms = [a.elapsed_time(b) for a, b in evs]
        mean, med = allmax(torch, dist, dev, [sum(step_ms) / len(step_ms), statistics.median(step_ms)])
        return mean, med, (t0, t1)

    soak(args.soak_s)
    launches0 = M.kernel_launches()
    ms_mean, ms_med, clocks = timed_steps()
    launches = M.kernel_launches() - launches0
    total_bytes = bytes_rank * world
    value = total_bytes / (ms_mean * 1e-3) / 1e9
    # ---- kernel-only roofline of the dominant kernel (the rank's SpMV)
    kern_ms = ms_mean
    coll_us = None
    if world > 1:
        kern_ms = allmax(torch, dist, dev, [timer.device_ms(lambda: dm.spmv_into(x, y, stream), min(args.steps, 50),
                                                            need_flush)])[0]
        cm = timer.run(lambda: (sharded.broadcast_x(x), sharded.gather_y()), min(args.steps, 50))
        coll_us = allmax(torch, dist, dev, [statistics.mean(cm)])[0] * 1e3
    achieved = bytes_rank / (kern_ms * 1e-3) / 1e9

    # ---- e2e through the public API with pinned host buffers (H2D x, SpMV, D2H y, synchronise)
    hx = torch.empty(C, dtype=torch.int16, pin_memory=True)
    hx.copy_(x.view(torch.int16).cpu())
    if world == 1:
        hy = torch.empty(R, dtype=torch.int16, pin_memory=True)
        hxn, hyn = hx.numpy().view(np.uint16), hy.numpy().view(np.uint16)
        dm.spmv_host(hxn, hyn, stream)  # validated once through the Python wrapper ...
        from paper_2511_13061_b200 import _lib as _L
        _c_fn = _L.load().macko_spmv_host  # ... then timed as the bare C-ABI call a C/C++ caller makes
        _c_args = (dm._h, hxn.ctypes.data, hyn.ctypes.data, M._stream_ptr(stream))

        def e2e_fn():  # C-ABI macko_spmv_host: x pulled from pinned host memory, y written back, synchronises
            if _c_fn(*_c_args) != 0:
                raise RuntimeError("macko_spmv_host failed")
        d2h = 2 * R
    else:
        hy = torch.empty(R * world, dtype=torch.int16, pin_memory=True)

        def e2e_fn():  # rank 0's host x -> every rank's host y
            if rank == 0:
                x.view(torch.int16).copy_(hx, non_blocking=True)
            yy = sharded(x)
            hy.copy_(yy.view(torch.int16), non_blocking=True)
            torch.cuda.current_stream().synchronize()
        d2h = 2 * R * world
    e2e_ms = timer.run(e2e_fn, min(args.steps, 100), flush=need_flush)
    e2e_mean = allmax(torch, dist, dev, [sum(e2e_ms) / len(e2e_ms)])[0]
    e2e_val = total_bytes / (e2e_mean * 1e-3) / 1e9

    # ---- small-batch SpMM (batch 1/2/4/8 stream the matrix once)
    spmm = run_spmm(M, torch, dm, timer, stream, need_flush) if (rank == 0 and hasattr(dm, "spmm_into")) else None

    # ---- the same K steps again once the power cap has settled the clocks (back-to-back SpMVs for
    # --sustain-s first): what a long stream of SpMVs sustains.  Last of the SpMV measurements, so
    # the e2e and SpMM figures above are taken at the same (burst) clocks as the headline.
    sustained = None
    if args.sustain_s > 0:
        soak(args.sustain_s)
        s_mean, s_med, s_win = timed_steps()
        sustained = {"value": round(total_bytes / (s_mean * 1e-3) / 1e9, 2), "ms_per_step": round(s_mean, 5),
                     "us_per_step_median": round(s_med * 1e3, 2), "after_soak_s": args.sustain_s}
    if sampler is not None:
        sampler.collect()
        clocks = sampler.summary(*clocks)
        if sustained is not None:
            sustained["clocks"] = sampler.summary(*s_win)

    cpu_src = dm.download() if (rank == 0 and world == 1 and not args.no_cpu_baseline) else None
    li = dm.launch_info()
    pad_nnz = dm.pad_nnz
    sweep = run_sweep(M, torch, dev, stream, timer, peak) if (args.sweep and rank == 0) else None
    strong = None
    if world > 1 or args.strong:
        del dm, sharded
        torch.cuda.empty_cache()
        dm = None
        strong = run_strong(args, M, torch, dist, dev, stream, timer, world, rank, peak)
    chain = None
    if args.chain:
        if dm is not None:
            dm.close()
        torch.cuda.empty_cache()
        chain = run_chain(args, torch, dist, dev, world, rank, peak)
    decode = None
    if not args.no_decode and world == 1 and rank == 0:
        if dm is not None:
            dm.close()
            dm = None
        torch.cuda.empty_cache()
        decode = run_decode(torch, dev)

    # ---- CPU baselines (rank 0, N = 1): reference SpMV on the same matrix, 1 thread and all cores
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cpu_src, C, d)

    if rank == 0:
        traffic = load_traffic(R, C, d)
        kname = f"macko_spmv<{li.x_in_smem},4>"
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_mean, 5), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f16", "data": "synthetic (counter-hash generator, random unstructured)",
            "config": workload_config(R, C, d, world),
            "us_per_spmv": round(kern_ms * 1e3, 2), "us_per_step_median": round(ms_med * 1e3, 2),
            "timing": {"l2": ("flushed before every step (sum over a 2xL2 buffer, outside the step events)" if need_flush
                              else f"not flushed: inputs larger than L2 ({bytes_rank / 2**20:.0f} MiB per step vs "
                                   f"{l2 / 2**20:.0f} MiB L2; ncu: L2 hit rate < 1 % back to back)"),
                       "soak_s": args.soak_s, "events": "CUDA events on the launching stream, max over ranks",
                       "clocks": "sampled during the K timed steps only"},
            "matrix": {"pad_nnz_per_rank": pad_nnz, "bytes_per_spmv_per_rank": bytes_rank, "grid": li.grid,
                       "block": li.block, "x_mode": li.x_in_smem, "split_rows": li.n_split_rows},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": traffic, "peak_source": peak_src,
                         "kernel": kname, "us": round(kern_ms * 1e3, 2),
                         "algorithmic_bytes": "spmv_traffic (SPEC.md:336): values + packed deltas (16-B tails) "
                                              "+ 4(R+1) + 2C + 2R per SpMV"},
            "e2e": {"value": round(e2e_val, 2), "unit": "GB/s", "h2d_bytes_per_step": 2 * C, "d2h_bytes_per_step": d2h,
                    "us_per_call": round(e2e_mean * 1e3, 2),
                    "api": ("macko_spmv_host (bare C-ABI call via ctypes, pinned host x / y, synchronising)" if world == 1 else
                            "pinned H2D x on rank 0 + RowShardedSpmv + D2H y on every rank")},
            "compress_s": round(compress_s, 4), "compress_warm_s": round(compress_warm_s, 4),
            "gpu_launches": launches,
            "clocks": clocks,
            "sustained": sustained,
            "cpu_baseline": cpu,
        }
        if coll_us is not None:
            line["collectives_us"] = round(coll_us, 2)
        if dense_best is not None:
            api, dus, all_apis = dense_best
            line["dense_cublas_gemv"] = {
                "api": api, "us": round(dus, 2), "apis_us": all_apis,
                "GBps_effective": round((2 * R * C + 2 * R + 2 * C) / (dus * 1e-6) / 1e9, 1),
                "macko_speedup": round(dus / (kern_ms * 1e3), 3)}
        for k, v in (("spmm", spmm), ("sweep", sweep), ("strong", strong), ("chain", chain), ("decode", decode)):
            if v is not None:
                line[k] = v
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def load_traffic(R, C, d):
    """DRAM bytes per launch of the SpMV from the committed ncu --set full capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f)
        k = f"{R}x{C}@{d}"
        if k in t:
            return t[k]["dram_bytes_per_launch"]
    except Exception:
        pass
    return None


def run_spmm(M, torch, dm, timer, stream, need_flush):
    """Small-batch SpMM Y = A X (X: C x b) for b = 1, 2, 4, 8: one pass over the matrix."""
    out = {}
    for b in (1, 2, 4, 8):
        X = torch.empty((b, dm.cols), dtype=torch.float16, device="cuda")
        for i in range(b):
            M.gen_vector(X[i], dm.cols, seed=SEED_X + i)
        Y = torch.empty((b, dm.rows), dtype=torch.float16, device="cuda")
        us = timer.device_ms(lambda: dm.spmm_into(X, Y, stream), 30, need_flush) * 1e3
        out[f"batch{b}"] = {"us": round(us, 2), "us_per_vector": round(us / b, 2)}
    return out


def run_strong(args, M, torch, dist, dev, stream, timer, world, rank, peak):
    """BASELINE config 5: 131072x32768 @50 / 90 %, rows/N per rank (strong scaling)."""
    from paper_2511_13061_b200.sharded import FusedRowShardedSpmv, RowShardedSpmv, device_local_spmv

    R, C = CONFIG5["rows"], CONFIG5["cols"]
    out = []
    for d in (0.5, 0.1):
        r0, r1 = M.shard_rows(R, world, rank)
        dense = torch.empty((r1 - r0, C), dtype=torch.float16, device=dev)
        M.gen_dense(dense, r1 - r0, C, d, seed=SEED_A, row0=r0)
        dm = M.DeviceMatrix.from_dense(dense)
        del dense
        torch.cuda.empty_cache()
        x = torch.empty(C, dtype=torch.float16, device=dev)
        M.gen_vector(x, C, seed=SEED_X)
        y = torch.empty(r1 - r0, dtype=torch.float16, device=dev)
        total = float(dm.traffic_bytes)  # algorithmic bytes of the whole matrix: sum over the slabs
        if world > 1:
            tb = torch.tensor([total], device=dev, dtype=torch.float64)
            dist.all_reduce(tb)
            total = tb.item()
        reps = min(args.steps, 30)
        kern = allmax(torch, dist, dev, [statistics.mean(timer.run(lambda: dm.spmv_into(x, y, stream), reps))])[0]
        rec = {"shape": f"{R}x{C}", "sparsity": sparsity_pct(d), "rows_per_rank": r1 - r0, "n_gpus": world,
               "bytes_total": int(total), "spmv_us_per_rank": round(kern * 1e3, 2),
               "spmv_frac_per_rank": round(dm.traffic_bytes / (kern * 1e-3) / 1e9 / peak, 4)}
        if world > 1:
            sh = RowShardedSpmv(R, C, device_local_spmv(dm, stream), device=dev)
            coll = allmax(torch, dist, dev, [statistics.mean(timer.run(lambda: (sh.broadcast_x(x), sh.gather_y()), reps))])[0]
            stp = allmax(torch, dist, dev, [statistics.mean(timer.run(lambda: sh(x), reps))])[0]
            rec.update({"collectives_us": round(coll * 1e3, 2), "nccl_step_us": round(stp * 1e3, 2),
                        "nccl_GBps": round(total / (stp * 1e-3) / 1e9, 1)})
            if r1 - r0 == R // world:
                fused = FusedRowShardedSpmv(dm, R, dev)
                ys = [fused(x, stream)]
                fs = allmax(torch, dist, dev, [statistics.mean(timer.run(lambda: fused(x, stream), reps))])[0]
                rec.update({"fused_step_us": round(fs * 1e3, 2), "fused_GBps": round(total / (fs * 1e-3) / 1e9, 1)})
                torch.cuda.synchronize()
                dist.barrier()
                fused.close()
                del ys
        else:
            rec["GBps"] = round(total / (kern * 1e-3) / 1e9, 1)
        out.append(rec)
        dm.close()
        torch.cuda.empty_cache()
    return out


def run_chain(args, torch, dist, dev, world, rank, peak):
    """Config 4: Llama2-7B decode SpMV chain (32 layers x {qkv, o, gate_up, down}) at 50 %,
    PDL-chained SpMVs in one CUDA graph per token; N > 1: row slabs + NCCL all_gather per SpMV
    (and, with --fused, the all-gather fused into the SpMVs).  Beside it (N = 1) the same chain over
    dense fp16 weights with torch.mv (cuBLAS GEMV), also graph-captured."""
    from paper_2511_13061_b200 import decoder_chain as D
    from paper_2511_13061_b200 import macko as M

    t0 = time.time()
    ch = D.SparseDecoderChain(D.LLAMA2_7B, density=0.5, keep_dense=(world == 1), fused=(args.fused and world > 1))
    build_s = time.time() - t0
    M.gen_vector(ch.acts["h"], D.LLAMA2_7B.hidden, seed=SEED_X)
    g = None if ch.fused else ch.capture(pdl=True)

    def time_graph(graph, n):
        for _ in range(3):
            graph.replay()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
        for a, b in evs:
            a.record()
            graph.replay()
            b.record()
        torch.cuda.synchronize()
        return allmax(torch, dist, dev, [sum(a.elapsed_time(b) for a, b in evs) / n])[0]

    def time_tokens(n):  # fused all-gather: plain stream launches (flag targets grow per SpMV)
        for _ in range(3):
            ch.forward_token(pdl=True)
        torch.cuda.synchronize()
        dist.barrier()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
        for a, b in evs:
            a.record()
            ch.forward_token(pdl=True)
            b.record()
        torch.cuda.synchronize()
        return allmax(torch, dist, dev, [sum(a.elapsed_time(b) for a, b in evs) / n])[0]

    n = max(3, args.chain_tokens)
    ms = time_tokens(n) if ch.fused else time_graph(g, n)
    bytes_rank = ch.traffic_bytes
    total_bytes = bytes_rank * world
    out = {
        "workload": "Llama2-7B decoder stack, 32 layers x {qkv 12288x4096, o 4096x4096, gate_up 22016x4096, "
                    "down 4096x11008} @50% sparsity, batch-1 decode SpMV chain (q/k/v and gate/up row-stacked), "
                    "random-init",
        "n_gpus": world, "parallelism": f"row-shard x{world}" + (
            (" + all-gather fused into each SpMV (peer stores + flags)" if ch.fused else " + NCCL all_gather per SpMV")
            if world > 1 else ""),
        "spmvs_per_token": ch.kernels_per_token,
        "launch": ("PDL-chained SpMV + flag-wait kernels, stream launches" if ch.fused else
                   "PDL-chained SpMV kernels, one CUDA graph per token"),
        "us_per_token": round(ms * 1e3, 2), "tokens_per_s": round(1e3 / ms, 2),
        "bytes_per_token": total_bytes, "GBps": round(total_bytes / (ms * 1e-3) / 1e9, 1),
        "frac_per_gpu": round(bytes_rank / (ms * 1e-3) / 1e9 / peak, 4), "build_s": round(build_s, 2),
        "l2": "not flushed: 8.1 GB of weights per token streams from HBM", "timed_tokens": n,
    }
    if world == 1:
        dch = D.DenseDecoderChain(ch)
        dch.acts["h"].copy_(ch.acts["h"])
        dg = dch.capture()
        dms = time_graph(dg, n)
        out.update({"cublas_us_per_token": round(dms * 1e3, 2), "cublas_tokens_per_s": round(1e3 / dms, 2),
                    "cublas_GBps": round(dch.traffic_bytes / (dms * 1e-3) / 1e9, 1),
                    "speedup_vs_cublas": round(dms / ms, 3)})
        del dch, dg
    ch.close()
    del ch, g
    torch.cuda.empty_cache()
    return out


def run_decode(torch, dev):
    """Llama2-7B decode: a random-init 32-layer model with MACKO linears vs the
    same model with dense cuBLAS linears, tokens/s at batch 1."""
    try:
        from paper_2511_13061_b200 import llama
    except ImportError:
        return None
    return llama.bench_decode(torch, dev)


def cpu_baseline(h, C, d):
    """The reference CPU SpMV (oracle/_ref: reference sources) on the same matrix, 1 thread and all
    host cores, plus BASELINE config 1 (4096x4096 @50 %: reference format build + SpMV)."""
    try:
        from oracle import oracle as O
    except Exception as e:  # pragma: no cover
        return {"value": None, "unit": "GB/s", "cores": 0, "kind": "port", "sample": f"oracle unavailable: {e}"}
    kind = "reference" if O.ref_available() else "port"
    threads = host_cores()
    m = O.Macko(h.rows, h.cols, 4, h.values, h.packed_deltas, h.row_pointers)
    x = O.gen_vector(C, SEED_X)
    if kind == "reference":
        rm = O.RefMatrix.from_macko(m)
        runner = lambda t: (lambda: rm.spmv(x, m.rows, t))  # noqa: E731
    else:
        runner = lambda t: (lambda: O.reference_spmv(m, x, t))  # noqa: E731

    def timeit(fn, min_reps, budget_s):
        fn()
        ts = []
        t0 = time.time()
        while len(ts) < min_reps or (time.time() - t0 < budget_s and len(ts) < 50):
            t1 = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t1)
        return statistics.median(ts) * 1e3

    bytes_step = O.spmv_traffic_bytes(m.rows, C, m.pad_nnz, 4)
    ms_all = timeit(runner(threads), 5, 8.0)
    ms_one = timeit(runner(1), 2, 3.0)
    # config 1: 4096^2 @50 %, the reference's format build (csr_from_dense + macko_from_csr) + SpMV
    A1 = O.gen_dense(4096, 4096, 0.5, SEED_A)
    x1 = O.gen_vector(4096, SEED_X)
    tb = []
    for _ in range(3):
        t1 = time.perf_counter()
        r1 = O.RefMatrix.encode(A1, 4) if kind == "reference" else None
        if r1 is None:
            m1 = O.encode_dense(A1, 4)
        tb.append(time.perf_counter() - t1)
    if kind == "reference":
        c1_one = timeit(lambda: r1.spmv(x1, 4096, 1), 5, 2.0)
        c1_all = timeit(lambda: r1.spmv(x1, 4096, threads), 5, 2.0)
    else:
        c1_one = timeit(lambda: O.reference_spmv(m1, x1, 1), 5, 2.0)
        c1_all = timeit(lambda: O.reference_spmv(m1, x1, threads), 5, 2.0)
    return {"value": round(bytes_step / (ms_all * 1e-3) / 1e9, 3), "unit": "GB/s", "cores": threads, "kind": kind,
            "ms_per_spmv": round(ms_all, 3),
            "one_thread": {"value": round(bytes_step / (ms_one * 1e-3) / 1e9, 3), "unit": "GB/s", "cores": 1,
                           "ms_per_spmv": round(ms_one, 3)},
            "config1_4096x4096": {"format_build_ms_1thread": round(statistics.median(tb) * 1e3, 2),
                                  "spmv_ms_1thread": round(c1_one, 3), f"spmv_ms_{threads}threads": round(c1_all, 3)},
            "sample": f"the same {m.rows}x{C} matrix (downloaded from the GPU), reference_spmv, median of >= 5 reps "
                      f"({threads} threads) / >= 2 reps (1 thread), std::thread row partition, CPU {cpu_model()}"}


def run_sweep(M, torch, dev, stream, timer, peak):
    """30/50/70/90 % sparsity at 36864x12288, the Llama2-7B linear shapes at 50 % and the
    131072x32768 shapes of config 5 (whole matrix and an N = 8 row slab) at 50 / 90 %."""
    out = []
    cfgs = [(36864, 12288, 0.7), (36864, 12288, 0.5), (36864, 12288, 0.3), (36864, 12288, 0.1),
            (4096, 4096, 0.5), (11008, 4096, 0.5), (4096, 11008, 0.5),
            (131072, 32768, 0.5), (131072, 32768, 0.1), (16384, 32768, 0.5), (16384, 32768, 0.1)]
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    for R, C, d in cfgs:
        dense = torch.empty((R, C), dtype=torch.float16, device=dev)
        M.gen_dense(dense, R, C, d, seed=SEED_A)
        dm = M.DeviceMatrix.from_dense(dense)
        x = torch.empty(C, dtype=torch.float16, device=dev)
        M.gen_vector(x, C, seed=SEED_X)
        y = torch.empty(R, dtype=torch.float16, device=dev)
        flush = dm.traffic_bytes < 3 * l2
        us = timer.device_ms(lambda: dm.spmv_into(x, y, stream), 50, flush, warmup=5) * 1e3
        api, dus, apis = dense_baseline(torch, timer, dense, x, 30, flush)
        gbs = dm.traffic_bytes / (us * 1e-6) / 1e9
        out.append({"shape": f"{R}x{C}", "sparsity": sparsity_pct(d), "us": round(us, 2), "GBps": round(gbs, 1),
                    "x_mode": dm.launch_info().x_in_smem, "l2_flush": flush, "frac": round(gbs / peak, 4),
                    "cublas_us": round(dus, 2), "cublas_api": api, "speedup": round(dus / us, 3),
                    "bytes": dm.traffic_bytes})
        del dense
        dm.close()
        torch.cuda.empty_cache()
    return out


if __name__ == "__main__":
    main()
