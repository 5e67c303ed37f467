"""Batch-1 decode chain of sparse linears — BASELINE.json config 4: "Llama2-7B full decoder stack
of 32 layers' sparse linears at 50 %, batch-1 decode SpMV chain, row-sharded over 1/2/4/8 B200".

The paper's end-to-end use: every linear of a decoder layer is a MACKO
matrix and one generated token is a chain of SpMVs.  Per layer (the stand-in for
attention and the MLP activation — only the SpMV chain is timed):

    qkv = W_qkv h          W_qkv = [W_v; W_q; W_k]   (3H x H, rows stacked: rows are independent,
    o   = W_o v            v = qkv[0:H]                so the stacked encoding is the three
    gu  = W_gu o           W_gu = [W_up; W_gate]       encodings concatenated; the
    h'  = W_down u         u = gu[0:I]                 consumed slice first keeps it 512-B aligned)

so a token is 4 dependent SpMVs per layer (128 for Llama2-7B: H = 4096, I = 11008, 8.1 GB of
MACKO data at 50 % sparsity).  The chain is launched with programmatic dependent launch (each
SpMV's plan load and first matrix fills overlap the previous kernel's tail) and captured into a
CUDA graph.  Row sharding (N > 1): rank g owns the row slab g of every linear and the outputs are
all-gathered (NCCL) after each SpMV, so every rank holds the full activation.

`DenseDecoderChain` is the same chain over dense fp16 weights with torch.mv (cuBLAS GEMV, fp32
compute) — the baseline the paper compares against.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, List, Optional, Tuple

import os

import torch
import torch.distributed as dist

from . import macko as M

LINEARS = ("qkv", "o", "gate_up", "down")


@dataclass(frozen=True)
class ChainShape:
    layers: int = 32
    hidden: int = 4096
    inter: int = 11008

    def shape(self, name: str) -> Tuple[int, int]:
        H, I = self.hidden, self.inter
        return {"qkv": (3 * H, H), "o": (H, H), "gate_up": (2 * I, H), "down": (H, I)}[name]


LLAMA2_7B = ChainShape(32, 4096, 11008)


def weight_seed(base: int, layer: int, name: str) -> int:
    return base + 16 * layer + LINEARS.index(name)


def _x_slice(shape: ChainShape, name: str, acts: Dict[str, torch.Tensor]) -> torch.Tensor:
    H, I = shape.hidden, shape.inter
    if name == "qkv":
        return acts["h"]
    if name == "o":
        return acts["qkv"][:H]  # v
    if name == "gate_up":
        return acts["o"]
    return acts["gate_up"][:I]  # up


def _out_name(name: str) -> str:
    return "h" if name == "down" else name


# Start spread of a chained SpMV's CTAs the plans may be skewed for (macko_dev_set_chain_skew;
# tools/trace_chain.py measures ~2 us between the first and the last CTA of each op).  Measured on
# the 32-layer chain: 0 -> 2288, 1000 -> 2325, 2000 -> 2376, 3000 -> 2474 us per token, so the
# equal split stays the default.
CHAIN_SKEW_NS = int(os.environ.get("MACKO_CHAIN_SKEW_NS", "0"))
CHAIN_X_MODE = int(os.environ.get("MACKO_CHAIN_XMODE", "-1"))


class SparseDecoderChain:
    """The decode chain over MACKO matrices built on the GPU (generator -> GPU compressor)."""

    def __init__(self, shape: ChainShape = LLAMA2_7B, density: float = 0.5, seed: int = 0x5EEDA000,
                 device: Optional[torch.device] = None, keep_dense: bool = False, group=None, fused: bool = False,
                 chain_skew_ns: int = CHAIN_SKEW_NS):
        self.shape = shape
        self.device = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.mats: List[Dict[str, M.DeviceMatrix]] = []
        self.dense: List[Dict[str, torch.Tensor]] = []
        self.bounds: Dict[str, Tuple[int, int]] = {}
        H, I = shape.hidden, shape.inter
        self.acts = {"h": torch.zeros(H, dtype=torch.float16, device=self.device),
                     "qkv": torch.zeros(3 * H, dtype=torch.float16, device=self.device),
                     "o": torch.zeros(H, dtype=torch.float16, device=self.device),
                     "gate_up": torch.zeros(2 * I, dtype=torch.float16, device=self.device)}
        self.local = {}
        for name in LINEARS:
            R, C = shape.shape(name)
            r0, r1 = M.shard_rows(R, self.world, self.rank)
            self.bounds[name] = (r0, r1)
            if self.world > 1:
                self.local[name] = torch.zeros(r1 - r0, dtype=torch.float16, device=self.device)
        for layer in range(shape.layers):
            mats, dense = {}, {}
            for name in LINEARS:
                R, C = shape.shape(name)
                r0, r1 = self.bounds[name]
                w = torch.empty((r1 - r0, C), dtype=torch.float16, device=self.device)
                M.gen_dense(w, r1 - r0, C, density, seed=weight_seed(seed, layer, name), row0=r0)
                mats[name] = M.DeviceMatrix.from_dense(w)
                if chain_skew_ns:  # PDL-chained: late CTAs start up to ~2 us after the first
                    mats[name].set_chain_skew(chain_skew_ns)
                if CHAIN_X_MODE >= 0:  # experiments: force the gather split of every chain matrix
                    mats[name].configure(CHAIN_X_MODE)
                if keep_dense:
                    dense[name] = w
                else:
                    del w
            self.mats.append(mats)
            self.dense.append(dense)
        torch.cuda.synchronize(self.device)
        self.graph: Optional[torch.cuda.CUDAGraph] = None
        self.fused = fused
        if fused:
            self._setup_fused()

    def _setup_fused(self) -> None:
        """Fused all-gather (MACKO_SPMV_PEERS): every slab SpMV stores its rows into every rank's
        activation buffer and counts its CTAs into every rank's flag array; the next SpMV waits
        for all ranks' counters (macko_wait_flags).  IPC handles are exchanged over the group."""
        dev = self.device.index if self.device.index is not None else torch.cuda.current_device()
        self.flags = torch.zeros(self.world, dtype=torch.int32, device=self.device)
        self._ops_done = 0
        self._grid = self.mats[0][LINEARS[0]].launch_info().grid
        mine = {k: M.ipc_handle(v) for k, v in self.acts.items()}
        mine["flags"] = M.ipc_handle(self.flags)
        if self.world > 1:
            allh = [None] * self.world
            dist.all_gather_object(allh, mine, group=self.group)
        else:
            allh = [mine]
        self._bases, self._opened = {}, []
        own = {k: v.data_ptr() for k, v in self.acts.items()}
        own["flags"] = self.flags.data_ptr()
        ptrs = []
        for p, h in enumerate(allh):
            if p == self.rank:
                ptrs.append(own)
                continue
            d = {}
            for k, (handle, off) in h.items():
                if handle not in self._bases:
                    self._bases[handle] = M.ipc_open(handle, dev)
                    self._opened.append(self._bases[handle])
                d[k] = self._bases[handle] + off
            ptrs.append(d)
        for mats in self.mats:
            for name, m in mats.items():
                r0 = self.bounds[name][0]
                m.set_peers([ptrs[p][_out_name(name)] + 2 * r0 for p in range(self.world)],
                            [ptrs[p]["flags"] + 4 * self.rank for p in range(self.world)])

    # -- accounting -------------------------------------------------------------------------
    @property
    def traffic_bytes(self) -> int:
        """Algorithmic bytes of one token on this rank (sum of spmv_traffic of its slabs)."""
        return sum(m.traffic_bytes for mats in self.mats for m in mats.values())

    @property
    def kernels_per_token(self) -> int:
        return self.shape.layers * len(LINEARS)

    # -- execution --------------------------------------------------------------------------
    def _spmv(self, layer: int, name: str, stream, pdl: bool) -> None:
        x = _x_slice(self.shape, name, self.acts)
        out = self.acts[_out_name(name)]
        if self.fused:
            r0, r1 = self.bounds[name]
            self.mats[layer][name].spmv_into(x, out[r0:r1], stream, pdl=pdl, peers=True)
            self._ops_done += 1
            M.wait_flags(self.flags, self.world, self._ops_done * self._grid, stream)
        elif self.world == 1:
            self.mats[layer][name].spmv_into(x, out, stream, pdl=pdl)
        else:
            self.mats[layer][name].spmv_into(x, self.local[name], stream, pdl=pdl)
            dist.all_gather_into_tensor(out, self.local[name], group=self.group)

    def forward_token(self, stream=None, pdl: bool = True) -> torch.Tensor:
        """One token through every layer (stream-ordered; h is updated in place)."""
        for layer in range(self.shape.layers):
            for name in LINEARS:
                # the first kernel of a token follows the previous token's last SpMV: chained too
                self._spmv(layer, name, stream, pdl)
        return self.acts["h"]

    def capture(self, pdl: bool = True) -> torch.cuda.CUDAGraph:
        """Capture forward_token into a CUDA graph (kernel nodes keep their PDL edges)."""
        if self.fused:
            raise ValueError("fused all-gather waits on growing flag targets: not graph-capturable")
        s = torch.cuda.Stream(device=self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(s):
            self.forward_token(s, pdl)  # warm-up: texture objects for each x buffer, allocations
        torch.cuda.current_stream(self.device).wait_stream(s)
        torch.cuda.synchronize(self.device)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            self.forward_token(s, pdl)
        self.graph = g
        return g

    def close(self) -> None:
        for ptr in getattr(self, "_opened", []):
            M.ipc_close(ptr)
        self._opened = []
        for mats in self.mats:
            for m in mats.values():
                m.close()
        self.mats = []
        self.dense = []


class DenseDecoderChain:
    """The same chain over dense fp16 weights: torch.mv = cuBLAS GEMV with fp32 compute."""

    def __init__(self, sparse: SparseDecoderChain):
        if not sparse.dense or not sparse.dense[0]:
            raise ValueError("build the SparseDecoderChain with keep_dense=True")
        self.sparse = sparse
        self.shape = sparse.shape
        self.acts = {k: torch.zeros_like(v) for k, v in sparse.acts.items()}
        self.graph: Optional[torch.cuda.CUDAGraph] = None

    @property
    def traffic_bytes(self) -> int:
        return sum(2 * w.numel() + 2 * w.shape[0] + 2 * w.shape[1] for d in self.sparse.dense for w in d.values())

    def forward_token(self) -> torch.Tensor:
        for layer in range(self.shape.layers):
            for name in LINEARS:
                torch.mv(self.sparse.dense[layer][name], _x_slice(self.shape, name, self.acts),
                         out=self.acts[_out_name(name)])
        return self.acts["h"]

    def capture(self) -> torch.cuda.CUDAGraph:
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            self.forward_token()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            self.forward_token()
        self.graph = g
        return g
