"""`MackoLinear`: an nn.Linear replacement for batch-1 decode over a MACKO weight (the paper's
end-to-end use, PAPER.md:86,496-510 — every linear of a pruned LLM becomes an SpMV).

The fp16 weight is compressed once on the GPU (bit-exact MACKO format, b_delta = 4 by default);
forward(x) for x of shape [in_features] or [1, ..., 1, in_features] is one sm_100a SpMV (fp32
accumulate, one RNE) plus the optional bias; batches of up to 8 vectors are one small-batch SpMM
(macko_dev_spmm: the weight streams from HBM once per 8 vectors; row b bit-identical to the SpMV of
vector b), larger batches run in groups of 8.  There is no CPU fallback: the module requires the
CUDA library and a CUDA weight.
"""
from __future__ import annotations

from typing import Optional

import torch
from torch import nn

from . import _lib
from . import macko as M


@torch.library.custom_op("macko::spmv", mutates_args=())
def spmv_op(handle: int, x: torch.Tensor, rows: int) -> torch.Tensor:
    """y = A x as a registered torch operator (torch.ops.macko.spmv): `handle` is a live
    DeviceMatrix's C-ABI handle, x a contiguous fp16 CUDA vector.  Launches on the current stream
    (CUDA-graph capturable); no CPU implementation exists."""
    if not x.is_cuda or x.dtype != torch.float16 or x.dim() != 1:
        raise ValueError("macko::spmv takes a 1-D fp16 CUDA tensor")
    x = x.contiguous()
    y = torch.empty(rows, dtype=torch.float16, device=x.device)
    stream = torch.cuda.current_stream(x.device).cuda_stream
    _lib.check(_lib.load().macko_dev_spmv(handle, x.data_ptr(), y.data_ptr(), stream))
    return y


@spmv_op.register_fake
def _spmv_fake(handle: int, x: torch.Tensor, rows: int) -> torch.Tensor:
    return x.new_empty(rows)


@torch.library.custom_op("macko::spmm", mutates_args=())
def spmm_op(handle: int, X: torch.Tensor, rows: int) -> torch.Tensor:
    """Y = (A X^T)^T for a batch X of 1..8 fp16 CUDA row vectors (batch x cols) as a registered
    torch operator (torch.ops.macko.spmm); Y is batch x rows.  Launches on the current stream."""
    if not X.is_cuda or X.dtype != torch.float16 or X.dim() != 2 or not 1 <= X.shape[0] <= 8:
        raise ValueError("macko::spmm takes a (1..8) x cols fp16 CUDA tensor")
    X = X.contiguous()
    Y = torch.empty((X.shape[0], rows), dtype=torch.float16, device=X.device)
    stream = torch.cuda.current_stream(X.device).cuda_stream
    _lib.check(_lib.load().macko_dev_spmm(handle, X.data_ptr(), X.shape[1], Y.data_ptr(), rows, X.shape[0], stream))
    return Y


@spmm_op.register_fake
def _spmm_fake(handle: int, X: torch.Tensor, rows: int) -> torch.Tensor:
    return X.new_empty((X.shape[0], rows))


class MackoLinear(nn.Module):
    def __init__(self, matrix: M.DeviceMatrix, bias: Optional[torch.Tensor] = None):
        super().__init__()
        self.matrix = matrix
        self.in_features = matrix.cols
        self.out_features = matrix.rows
        if bias is not None:
            self.register_buffer("bias", bias.detach().to(torch.float16).contiguous())
        else:
            self.bias = None

    @classmethod
    def from_linear(cls, linear: nn.Linear, b_delta: int = 4) -> "MackoLinear":
        """Compress an (already pruned) nn.Linear's weight on its CUDA device."""
        w = linear.weight.detach()
        if not w.is_cuda:
            raise ValueError("MackoLinear needs a CUDA weight (no CPU fallback)")
        w16 = w.to(torch.float16).contiguous()
        dm = M.DeviceMatrix.from_dense(w16, b_delta=b_delta)
        return cls(dm, linear.bias)

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        if x.shape[-1] != self.in_features:
            raise ValueError(f"expected last dimension {self.in_features}, got {x.shape[-1]}")
        lead = x.shape[:-1]
        xs = x.reshape(-1, self.in_features).to(torch.float16).contiguous()
        h = self.matrix.handle
        if xs.shape[0] == 1:
            out = torch.ops.macko.spmv(h, xs[0], self.out_features).unsqueeze(0)
        elif self.matrix.b_delta != 4:  # the SpMM kernel is built for the paper's 4-bit deltas
            out = torch.stack([torch.ops.macko.spmv(h, xs[i], self.out_features) for i in range(xs.shape[0])])
        else:  # groups of up to 8 vectors: one pass over the weight per group
            out = torch.cat([torch.ops.macko.spmm(h, xs[i:i + 8], self.out_features) for i in range(0, xs.shape[0], 8)])
        if self.bias is not None:
            out = out + self.bias
        return out.reshape(*lead, self.out_features)

    def extra_repr(self) -> str:
        return (f"in_features={self.in_features}, out_features={self.out_features}, "
                f"pad_nnz={self.matrix.pad_nnz}, b_delta={self.matrix.b_delta}, bias={self.bias is not None}")
