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


class FusedRowShardedSpmv:
    """Row-sharded y = A x whose all-gather is fused into the SpMV kernel: every rank's kernel
    stores its slab's rows straight into every rank's full-y buffer (CUDA IPC / P2P over NVLink)
    and counts its CTAs into every rank's flag array; a step ends with a stream-ordered wait until
    all ranks' CTAs have signalled (MACKO_SPMV_PEERS, macko_wait_flags).  x must already be
    identical on every rank.

    The output is double-buffered by step parity (peer banks 0 / 1), so `y = fused(y)` is safe:
    step k writes the buffer that was step k-1's x, and a rank only starts step k after every
    rank's CTAs of step k-1 signalled — which they do after their last read of x.  The returned
    buffer is valid until the call after next.

    Setup exchanges IPC handles over `group` (any backend; gloo works).  Every rank's slab must
    use the same launch grid (same GPU model), which the flag target assumes.
    """

    def __init__(self, dm: "M.DeviceMatrix", rows_total: int, device: torch.device, group=None):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.dm = dm
        self.r0, self.r1 = slab_bounds(rows_total, self.world, self.rank)
        if dm.rows != self.r1 - self.r0:
            raise ValueError("slab rows do not match this rank's share of rows_total")
        self.ys = [torch.zeros(rows_total, dtype=torch.float16, device=device) for _ in range(2)]
        self.flags = torch.zeros(self.world, dtype=torch.int32, device=device)
        self.grid = dm.launch_info().grid
        self.epoch = 0
        dev = device.index if device.index is not None else torch.cuda.current_device()
        mine = ([M.ipc_handle(y) for y in self.ys], M.ipc_handle(self.flags), self.r0)
        if self.world > 1:
            allh = [None] * self.world
            dist.all_gather_object(allh, mine, group=group)
        else:
            allh = [mine]
        self._opened, self._bases = [], {}
        peer_y, peer_f = [[], []], []
        for p, (hys, (hf, of), _) in enumerate(allh):
            for b, (hy, oy) in enumerate(hys):
                yb = self.ys[b].data_ptr() if p == self.rank else self._open(hy, dev) + oy
                peer_y[b].append(yb + 2 * self.r0)
            fb = self.flags.data_ptr() if p == self.rank else self._open(hf, dev) + of
            peer_f.append(fb + 4 * self.rank)
        dm.set_peers(peer_y[0], peer_f)
        dm.set_peer_bank(1, peer_y[1])

    def _open(self, handle: bytes, dev: int) -> int:
        # one mapping per allocation (y and flags may come from the same caching-allocator segment)
        if handle not in self._bases:
            self._bases[handle] = M.ipc_open(handle, dev)
            self._opened.append(self._bases[handle])
        return self._bases[handle]

    @property
    def y(self) -> torch.Tensor:
        """The buffer the last call filled."""
        return self.ys[(self.epoch + 1) % 2]

    def __call__(self, x: torch.Tensor, stream=None) -> torch.Tensor:
        bank = self.epoch % 2
        out = self.ys[bank]
        xs, xe = x.data_ptr(), x.data_ptr() + 2 * x.numel()
        if xs < out.data_ptr() + 2 * out.numel() and out.data_ptr() < xe:
            raise ValueError("x overlaps this step's output buffer (pass the previous step's y or another buffer)")
        self.epoch += 1
        self.dm.spmv_into(x, out[self.r0:self.r1], stream, peers=True, bank=bank)
        M.wait_flags(self.flags, self.world, self.epoch * self.grid, stream)
        return out

    def close(self) -> None:
        self.dm.set_peers([], [])
        for ptr in self._opened:
            M.ipc_close(ptr)
        self._opened = []
