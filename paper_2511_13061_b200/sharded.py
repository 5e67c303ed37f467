"""Row-sharded MACKO SpMV across GPUs (one process per GPU, torch.distributed).

A large matrix (or every linear of a layer stack) is cut into contiguous equal-row slabs
(macko_shard_rows; slab encodings equal the global encoding sliced).  Rank g owns
rows [r0_g, r1_g) as its own MACKO matrix.  One step:

    broadcast(x, src=0)  ->  y_g = A_g x  (libmacko_cuda on the rank's GPU)  ->  all_gather(y_g)

The exchange is the path's real data movement (north_star: "x broadcast and y all-gathered by
NCCL over NVLink"); over NVSwitch these messages (x: 2C bytes, y: 2R bytes) are latency bound.
The same class runs over gloo on CPU tensors in the tests, with the per-rank compute supplied
by the caller.
"""
from __future__ import annotations

from typing import Callable, Optional

import torch
import torch.distributed as dist

from . import macko as M


def slab_bounds(rows: int, world: int, rank: int) -> tuple[int, int]:
    """[r0, r1) of `rank` (macko_shard_rows: floor(rows*g/N) cut points)."""
    return M.shard_rows(rows, world, rank)


class RowShardedSpmv:
    """y = A x for a row-sharded A.

    local_spmv(x, y_local) computes the rank's slab product into y_local (for the GPU path this
    is DeviceMatrix.spmv_into).  x is broadcast from rank 0 and the slabs are gathered in rank
    order, so every rank ends with the full y.
    """

    def __init__(self, rows: int, cols: int, local_spmv: Callable[[torch.Tensor, torch.Tensor], None],
                 device: Optional[torch.device] = None, dtype: torch.dtype = torch.float16, group=None):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.rows, self.cols = rows, cols
        self.bounds = [slab_bounds(rows, self.world, g) for g in range(self.world)]
        self.r0, self.r1 = self.bounds[self.rank]
        self.local_spmv = local_spmv
        self.device = device if device is not None else torch.device("cpu")
        self.dtype = dtype
        self.equal = len({b - a for a, b in self.bounds}) == 1
        self.y_local = torch.empty(self.r1 - self.r0, dtype=dtype, device=self.device)
        self.y = torch.empty(rows, dtype=dtype, device=self.device)
        self._parts = [self.y[a:b] for a, b in self.bounds]

    def broadcast_x(self, x: torch.Tensor) -> torch.Tensor:
        if self.world > 1:
            dist.broadcast(x, src=0, group=self.group)
        return x

    def gather_y(self) -> torch.Tensor:
        if self.world == 1:
            self.y.copy_(self.y_local)
        elif self.equal and self.device.type == "cuda":
            dist.all_gather_into_tensor(self.y, self.y_local, group=self.group)
        else:
            # uneven slabs (sizes differ by at most one row): gather padded slabs
            width = max(b - a for a, b in self.bounds)
            send = torch.zeros(width, dtype=self.dtype, device=self.device)
            send[: self.y_local.numel()].copy_(self.y_local)
            parts = [torch.empty(width, dtype=self.dtype, device=self.device) for _ in range(self.world)]
            dist.all_gather(parts, send, group=self.group)
            for dst, src in zip(self._parts, parts):
                dst.copy_(src[: dst.numel()])
        return self.y

    def __call__(self, x: torch.Tensor) -> torch.Tensor:
        self.broadcast_x(x)
        self.local_spmv(x, self.y_local)
        return self.gather_y()


def device_local_spmv(dm: "M.DeviceMatrix", stream=None) -> Callable[[torch.Tensor, torch.Tensor], None]:
    """The GPU per-rank compute: libmacko_cuda SpMV of the rank's slab."""

    def run(x: torch.Tensor, y: torch.Tensor) -> None:
        dm.spmv_into(x, y, stream)

    return run


def nccl_sharded_spmv(dm: "M.DeviceMatrix", nccl_comm: int, x: torch.Tensor, y: torch.Tensor, root: int = 0,
                      stream=None) -> torch.Tensor:
    """One sharded step inside libmacko_cuda (macko_sharded_spmv): NCCL broadcast of x from
    `root`, this rank's slab SpMV into its part of y, in-place NCCL all-gather of y.  `nccl_comm`
    is an ncclComm_t (as an int); dm is this rank's slab of a y.numel() x x.numel() matrix."""
    from . import _lib

    _lib.check(_lib.load().macko_sharded_spmv(dm.handle, nccl_comm, root, x.data_ptr(), y.data_ptr(), y.numel(),
                                              M._stream_ptr(stream)))
    return y
