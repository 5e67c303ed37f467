#!/usr/bin/env python
"""bench.py — MACKO SpMV on B200 (BASELINE.json metric: effective HBM GB/s & µs,
36864x12288 fp16 @ 50 % sparsity vs cuBLAS GEMV).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--sweep]

One step = one SpMV y = A·x over the resident MACKO matrix (GPU-compressed from a synthetic
random-unstructured fp16 matrix).  N > 1 (torchrun, one rank per GPU): weak scaling — every
rank owns a 36864-row slab of an (N·36864)x12288 matrix; a step is NCCL broadcast(x) + SpMV +
NCCL all_gather(y), timed on the device and reduced as the max over ranks.

`value` = algorithmic bytes of all ranks (spmv_traffic) / device time of one
step.  L2 is flushed (read of a 2xL2 buffer) before every step, outside the step's events.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SpMV effective HBM GB/s & µs, 36864×12288 fp16 @50% sparsity vs cuBLAS GEMV"
HEADLINE = dict(rows=36864, cols=12288, density=0.5)
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
    p.add_argument("--sweep", action="store_true", help="also report 30/50/70/90 %% sparsity and Llama shapes")
    p.add_argument("--chain", action="store_true",
                   help="also report the Llama2-7B 32-layer decode SpMV chain (config 4) vs a dense cuBLAS chain")
    p.add_argument("--chain-tokens", type=int, default=20)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--soak-s", type=float, default=1.0, help="untimed load before timing (clock sampling)")
    p.add_argument("--x-mode", type=int, default=-1, help="x gathers: -1 auto, 0 texture only, 1 smem table only, 6..9 smem + texture split")
    p.add_argument("--ctas", type=int, default=0, help="cap on SpMV CTAs per SM (0 = occupancy maximum)")
    p.add_argument("--fused", action="store_true",
                   help="N > 1: all-gather of y fused into the SpMV kernel (peer stores over NVLink + flags; "
                        "x replicated, no broadcast) instead of NCCL broadcast + all_gather")
    return p.parse_args()


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
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        rows = []
        for line in out.strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), parts[2:6], float(parts[6])))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        loaded = [r for r in rows if r[3] > 0] or rows
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in loaded for i, v in enumerate(r[2]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(r[0] for r in loaded), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows), "samples_under_load": len(loaded)}


# ---------------------------------------------------------------------------------- reference arm
def run_reference(args, rank: int):
    """The reference's own CPU path (oracle/_ref: reference fp16.cpp / bitpack.cpp / headers +
    SPEC-restated bodies) on the box's host cores, same config / metric / unit."""
    if rank != 0:
        return
    from oracle import oracle as O

    kind = "reference" if O.ref_available() else "port"
    threads = host_cores()
    R, C, d = args.rows, args.cols, args.density
    t0 = time.time()
    # bounded sample: full-width row slab; full matrix unless the build would be too slow
    rows_s = R
    A = O.gen_dense(rows_s, C, d, SEED_A)
    if kind == "reference":
        rm = O.RefMatrix.encode(A, 4)
        m = rm.to_macko(rows_s, C, 4)
        run = lambda x: rm.spmv(x, rows_s, threads)  # noqa: E731
    else:
        m = O.encode_dense(A, 4)
        run = lambda x: O.reference_spmv(m, x, threads)  # noqa: E731
    del A
    build_s = time.time() - t0
    x = O.gen_vector(C, SEED_X)
    bytes_step = O.spmv_traffic_bytes(rows_s, C, m.pad_nnz, 4)
    t1 = time.perf_counter()
    run(x)
    one = time.perf_counter() - t1
    steps = args.steps
    budget = 120.0
    if one * (steps + args.warmup) > budget:  # keep the whole arm within a few minutes
        steps = max(3, int(budget / max(one, 1e-6)) - args.warmup)
    for _ in range(min(args.warmup, 3)):
        run(x)
    times = []
    for _ in range(steps):
        t1 = time.perf_counter()
        run(x)
        times.append(time.perf_counter() - t1)
    ms = statistics.median(times) * 1e3
    gbs = bytes_step / (ms * 1e-3) / 1e9
    sample = (f"{rows_s}x{C} @{int(round((1 - d) * 100))}% sparsity (full workload), reference_spmv, "
              f"{steps} timed steps (median), {threads} threads std::thread row partition, build {build_s:.1f}s, "
              f"CPU {cpu_model()}")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(gbs, 3), "unit": "GB/s", "n_gpus": args.gpus,
        "steps": steps, "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f16", "data": "synthetic",
        "config": {"workload": f"{R}x{C} fp16 @{int(round((1 - d) * 100))}% sparsity, single SpMV", "rows": rows_s,
                   "cols": C, "density": d, "b_delta": 4, "pad_nnz": m.pad_nnz, "bytes_per_spmv": bytes_step},
        "cpu_baseline": {"value": round(gbs, 3), "unit": "GB/s", "cores": threads, "kind": kind, "sample": sample},
        "e2e": {"value": round(gbs, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------- our arm
def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
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
    sparsity_pct = int(round((1 - d) * 100))

    # ---- build the rank's slab on the device: generator -> GPU compressor (no host copies)
    dense = torch.empty((R, C), dtype=torch.float16, device=dev)
    M.gen_dense(dense, R, C, d, seed=SEED_A, row0=rank * R)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dm = M.DeviceMatrix.from_dense(dense)
    torch.cuda.synchronize()
    compress_s = time.perf_counter() - t0
    if args.x_mode != -1 or args.ctas:
        dm.configure(args.x_mode, args.ctas)
    x = torch.empty(C, dtype=torch.float16, device=dev)
    M.gen_vector(x, C, seed=SEED_X)
    y = torch.empty(R, dtype=torch.float16, device=dev)
    bytes_rank = dm.traffic_bytes
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = torch.ones(max(2 * l2, 256 << 20) // 4, dtype=torch.float32, device=dev)
    # Inputs several times larger than L2 stream from HBM on every step (verified with ncu on
    # back-to-back launches: L2 hit rate < 1 %, DRAM bytes = algorithmic bytes); smaller inputs
    # get an L2 flush (a read of a 2xL2 buffer) before every step, outside the step events.
    need_flush = bytes_rank < 3 * l2

    def l2_flush(force=False):
        if need_flush or force:
            flush.sum()  # reads 2xL2 of clean lines: evicts the matrix without dirty write-back

    # N > 1: rows [rank*R, (rank+1)*R) of an (N*R) x C matrix; NCCL broadcast(x) + SpMV + all_gather(y)
    sharded = None
    if world > 1:
        if args.fused:
            from paper_2511_13061_b200.sharded import FusedRowShardedSpmv

            fused = FusedRowShardedSpmv(dm, R * world, dev)
            sharded = lambda xx: fused(xx, stream)  # noqa: E731
        else:
            sharded = RowShardedSpmv(R * world, C, device_local_spmv(dm, stream), device=dev)

    def step():
        if sharded is not None:
            sharded(x)
        else:
            dm.spmv_into(x, y, stream)

    # ---- dense cuBLAS GEMV on the same matrix (before freeing the dense copy)
    dense_us = None
    if rank == 0:
        yd = torch.empty(R, dtype=torch.float16, device=dev)
        for _ in range(3):
            torch.mv(dense, x, out=yd)
        ts = []
        for _ in range(max(10, min(args.steps, 50))):
            l2_flush()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch.mv(dense, x, out=yd)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        dense_us = statistics.median(ts) * 1e3
    del dense
    torch.cuda.empty_cache()

    # ---- warmup + soak (clock sampling covers soak + timed region)
    sampler = ClockSampler(local)
    if rank == 0:
        sampler.start()
    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    t_end = time.time() + args.soak_s
    while time.time() < t_end:
        for _ in range(20):
            dm.spmv_into(x, y, stream)
        torch.cuda.synchronize()

    # ---- timed region: exactly K steps, per-step device events around the step only
    launches0 = M.kernel_launches()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for i in range(args.steps):
        l2_flush()
        evs[i][0].record(stream)
        step()
        evs[i][1].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = M.kernel_launches() - launches0
    clocks = sampler.stop() if rank == 0 else None
    step_ms = [a.elapsed_time(b) for a, b in evs]
    ms_mean = sum(step_ms) / len(step_ms)
    ms_med = statistics.median(step_ms)
    if world > 1:
        t = torch.tensor([ms_mean, ms_med], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_mean, ms_med = t.tolist()
    total_bytes = bytes_rank * world
    value = total_bytes / (ms_mean * 1e-3) / 1e9

    # ---- kernel-only roofline of the dominant kernel (macko_spmv_b4), rank 0 alone
    kern_ms = ms_mean
    if world > 1:
        kts = []
        for _ in range(min(args.steps, 50)):
            l2_flush()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            dm.spmv_into(x, y, stream)
            b.record(stream)
            b.synchronize()
            kts.append(a.elapsed_time(b))
        kern_ms = sum(kts) / len(kts)
    achieved = bytes_rank / (kern_ms * 1e-3) / 1e9

    # ---- e2e through the C-ABI with pinned host buffers (H2D x, kernel, D2H y, sync)
    hx = torch.empty(C, dtype=torch.int16, pin_memory=True)
    hy = torch.empty(R, dtype=torch.int16, pin_memory=True)
    hx.copy_(x.view(torch.int16).cpu())
    hxn, hyn = hx.numpy().view(np.uint16), hy.numpy().view(np.uint16)
    for _ in range(3):
        dm.spmv_host(hxn, hyn, stream)
    e2e_ms = []
    for _ in range(min(args.steps, 100)):
        l2_flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        dm.spmv_host(hxn, hyn, stream)  # synchronises the stream internally
        b.record(stream)
        b.synchronize()
        e2e_ms.append(a.elapsed_time(b))
    e2e_mean = sum(e2e_ms) / len(e2e_ms)
    if world > 1:
        t = torch.tensor([e2e_mean], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_mean = t.item()
    e2e_val = total_bytes / (e2e_mean * 1e-3) / 1e9

    cpu_src = dm.download() if (rank == 0 and world == 1 and not args.no_cpu_baseline) else None
    li = dm.launch_info()
    pad_nnz = dm.pad_nnz
    sweep = None
    if args.sweep and rank == 0:
        sweep = run_sweep(M, torch, dev, stream, l2_flush, peak)

    chain = None
    if args.chain:
        del dm
        torch.cuda.empty_cache()
        chain = run_chain(args, torch, dist, dev, world, rank, peak)

    # ---- CPU baseline (rank 0, N = 1): reference SpMV on the same matrix, host cores
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cpu_src, C, d)

    if rank == 0:
        traffic = load_traffic(R, C, d)
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_mean, 5), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f16", "data": "synthetic (counter-hash generator, random unstructured)",
            "us_per_spmv": round(kern_ms * 1e3, 2), "us_per_step_median": round(ms_med * 1e3, 2),
            "config": {
                "workload": f"{R}x{C} fp16 @{sparsity_pct}% sparsity (random unstructured), single SpMV"
                + ((f" per rank, {R * world}x{C} row-sharded, all-gather of y fused into the SpMV (peer stores + flags)"
                    if args.fused else f" per rank, {R * world}x{C} row-sharded, NCCL broadcast x + all_gather y")
                   if world > 1 else ""),
                "rows_per_rank": R, "cols": C, "density": d, "b_delta": 4, "pad_nnz": pad_nnz,
                "bytes_per_spmv_per_rank": bytes_rank, "parallelism": f"row-shard x{world}",
                "l2": ("flushed before every step (sum over a 2xL2 buffer, outside the step events)" if need_flush else
                       f"not flushed: inputs larger than L2 ({bytes_rank / 2**20:.0f} MiB per step vs {l2 / 2**20:.0f} MiB L2; "
                       "ncu: L2 hit rate < 1 % back to back)"),
                "grid": li.grid, "block": li.block, "ctas_per_sm": li.ctas_per_sm, "split_rows": li.n_split_rows,
            },
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": traffic, "peak_source": peak_src,
                         "kernel": f"macko_spmv<{li.x_in_smem},4>", "us": round(kern_ms * 1e3, 2)},
            "e2e": {"value": round(e2e_val, 2), "unit": "GB/s", "h2d_bytes_per_step": 2 * C,
                    "d2h_bytes_per_step": 2 * R, "us_per_call": round(e2e_mean * 1e3, 2)},
            "dense_cublas_gemv": None if dense_us is None else {
                "us": round(dense_us, 2), "GBps_effective": round((2 * R * C + 2 * R + 2 * C) / (dense_us * 1e-6) / 1e9, 1),
                "GBps_vs_macko_bytes": round(bytes_rank / (dense_us * 1e-6) / 1e9, 1),
                "macko_speedup": round(dense_us / (kern_ms * 1e3), 3), "api": "torch.mv (cuBLAS), fp32 compute"},
            "compress_s": round(compress_s, 4),
            "gpu_launches": launches,
            "clocks": clocks,
            "cpu_baseline": cpu,
        }
        if sweep is not None:
            line["sweep"] = sweep
        if chain is not None:
            line["chain"] = chain
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def load_traffic(R, C, d):
    """DRAM bytes per launch of macko_spmv_b4 from the committed ncu --set full capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f)
        k = f"{R}x{C}@{d}"
        if k in t:
            return t[k]["dram_bytes_per_launch"]
    except Exception:
        pass
    return None


def run_chain(args, torch, dist, dev, world, rank, peak):
    """Config 4: Llama2-7B decode chain (32 layers x {qkv, o, gate_up, down}) at 50 % sparsity,
    PDL-chained SpMVs in one CUDA graph per token; N > 1: row slabs + NCCL all_gather per SpMV.
    Weights stream from HBM (8.1 GB per token >> L2): no flush.  Beside it (N = 1) the same
    chain with dense fp16 weights through torch.mv (cuBLAS GEMV), also graph-captured."""
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
        ms = sum(a.elapsed_time(b) for a, b in evs) / n
        if world > 1:
            t = torch.tensor([ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = t.item()
        return ms

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
        t = torch.tensor([sum(a.elapsed_time(b) for a, b in evs) / n], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    n = max(3, args.chain_tokens)
    launches0 = M.kernel_launches()
    ms_graph = time_tokens(n) if ch.fused else time_graph(g, n)
    launches_graph = M.kernel_launches() - launches0
    bytes_rank = ch.traffic_bytes
    total_bytes = bytes_rank * world
    ms_pers = None
    if world == 1:
        # the token as one persistent cooperative kernel (weights prefetched across the barriers)
        gp = torch.cuda.CUDAGraph()
        sp = torch.cuda.Stream()
        ch.forward_token_persistent()
        torch.cuda.synchronize()
        with torch.cuda.graph(gp, stream=sp):
            ch.forward_token_persistent(sp)
        ms_pers = time_graph(gp, n)
    ms = min(ms_graph, ms_pers) if ms_pers is not None else ms_graph
    out = {
        "workload": "Llama2-7B decoder stack, 32 layers x {qkv 12288x4096, o 4096x4096, gate_up 22016x4096, "
                    "down 4096x11008} @50% sparsity, batch-1 decode (q/k/v and gate/up row-stacked), random-init",
        "n_gpus": world, "parallelism": f"row-shard x{world}" + (
            (" + all-gather fused into each SpMV (peer stores + flags)" if ch.fused else " + NCCL all_gather per SpMV")
            if world > 1 else ""),
        "spmvs_per_token": ch.kernels_per_token,
        "launch": ("one persistent cooperative kernel per token (grid barrier between dependent SpMVs, "
                   "weights prefetched across it)" if ms == ms_pers else
                   "PDL-chained SpMV + flag-wait kernels, stream launches" if ch.fused else
                   "PDL-chained SpMV kernels, one CUDA graph per token"),
        "us_per_token": round(ms * 1e3, 2), "tokens_per_s": round(1e3 / ms, 2),
        "us_per_token_pdl_graph": round(ms_graph * 1e3, 2),
        "us_per_token_persistent": None if ms_pers is None else round(ms_pers * 1e3, 2),
        "bytes_per_token": total_bytes, "GBps": round(total_bytes / (ms * 1e-3) / 1e9, 1),
        "frac_per_gpu": round(bytes_rank / (ms * 1e-3) / 1e9 / peak, 4), "build_s": round(build_s, 2),
        "l2": "not flushed: 8.1 GB of weights per token streams from HBM",
        "timed_tokens": n, "host_launch_calls_in_timed_region": launches_graph,
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


def cpu_baseline(dm, C, d):
    try:
        from oracle import oracle as O
    except Exception as e:  # pragma: no cover
        return {"value": None, "unit": "GB/s", "cores": 0, "kind": "port", "sample": f"oracle unavailable: {e}"}
    kind = "reference" if O.ref_available() else "port"
    threads = host_cores()
    h = dm  # host MackoMatrix downloaded from the GPU
    m = O.Macko(h.rows, h.cols, 4, h.values, h.packed_deltas, h.row_pointers)
    x = O.gen_vector(C, SEED_X)
    if kind == "reference":
        rm = O.RefMatrix.from_macko(m)
        run = lambda: rm.spmv(x, m.rows, threads)  # noqa: E731
    else:
        run = lambda: O.reference_spmv(m, x, threads)  # noqa: E731
    run()
    ts = []
    t_start = time.time()
    while len(ts) < 5 or (time.time() - t_start < 10 and len(ts) < 50):
        t1 = time.perf_counter()
        run()
        ts.append(time.perf_counter() - t1)
        if time.time() - t_start > 30:
            break
    ms = statistics.median(ts) * 1e3
    bytes_step = O.spmv_traffic_bytes(m.rows, C, m.pad_nnz, 4)
    return {"value": round(bytes_step / (ms * 1e-3) / 1e9, 3), "unit": "GB/s", "cores": threads, "kind": kind,
            "ms_per_spmv": round(ms, 3),
            "sample": f"the same {m.rows}x{C} matrix (downloaded from the GPU), reference_spmv, median of {len(ts)} "
                      f"reps, {threads} threads, CPU {cpu_model()}"}


def run_sweep(M, torch, dev, stream, l2_flush, peak):
    """30/50/70/90 % sparsity at 36864x12288, the Llama2-7B linear shapes at 50 % and the
    131072x32768 shapes of config 5 (whole matrix and an N = 8 row slab) at 50 / 90 %."""
    out = []
    cfgs = [(36864, 12288, 0.7), (36864, 12288, 0.5), (36864, 12288, 0.3), (36864, 12288, 0.1),
            (4096, 4096, 0.5), (11008, 4096, 0.5), (4096, 11008, 0.5),
            # config 5: 131072x32768 (whole matrix on one GPU, and the row slab of one rank at N = 8)
            (131072, 32768, 0.5), (131072, 32768, 0.1), (16384, 32768, 0.5), (16384, 32768, 0.1)]
    for R, C, d in cfgs:
        dense = torch.empty((R, C), dtype=torch.float16, device=dev)
        M.gen_dense(dense, R, C, d, seed=SEED_A)
        dm = M.DeviceMatrix.from_dense(dense)
        x = torch.empty(C, dtype=torch.float16, device=dev)
        M.gen_vector(x, C, seed=SEED_X)
        y = torch.empty(R, dtype=torch.float16, device=dev)
        yd = torch.empty(R, dtype=torch.float16, device=dev)

        big = dm.traffic_bytes >= 3 * torch.cuda.get_device_properties(dev).L2_cache_size

        def timeit(fn, n=50):
            for _ in range(5):
                fn()
            ts = []
            for _ in range(n):
                if not big:
                    l2_flush(force=True)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                fn()
                b.record(stream)
                b.synchronize()
                ts.append(a.elapsed_time(b))
            return statistics.median(ts) * 1e3

        us = timeit(lambda: dm.spmv_into(x, y, stream))
        dus = timeit(lambda: torch.mv(dense, x, out=yd))
        gbs = dm.traffic_bytes / (us * 1e-6) / 1e9
        out.append({"shape": f"{R}x{C}", "sparsity": round(1 - d, 2), "us": round(us, 2), "GBps": round(gbs, 1),
                    "x_mode": dm.launch_info().x_in_smem, "l2_flush": not big,
                    "frac": round(gbs / peak, 4), "cublas_us": round(dus, 2), "speedup": round(dus / us, 3),
                    "bytes": dm.traffic_bytes})
        del dense, dm
        torch.cuda.empty_cache()
    return out


if __name__ == "__main__":
    main()
