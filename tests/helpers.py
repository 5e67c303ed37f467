"""Shared test helpers (tolerance bound, torch <-> numpy fp16-bit transfers)."""
import numpy as np

from oracle import oracle as O
from paper_2511_13061_b200 import macko as M

UNIT_STEPS = M.unit_steps()  # csrc/common.cuh kUnitSteps: the kernel's canonical reduction granularity


def b200_y(m, x):
    """The oracle emulation of the GPU's summation order (mo_b200_order_spmv: the ROMA walk,
    per-lane sequential, xor-tree per unit of UNIT_STEPS steps, units in order)."""
    return O.b200_order_spmv(m, x, UNIT_STEPS)


def tol_bound(dense: np.ndarray, x: np.ndarray, y_ref: np.ndarray):
    """Float-mode tolerance:
    |y - y_ref| <= ulp16(|y_ref|) + 2*n*2^-24*sum_i |a_i x_i|   (n = stored nonzeros of the row)."""
    a = dense.view(np.float16).astype(np.float64)
    xf = x.view(np.float16).astype(np.float64)
    s = np.abs(a) @ np.abs(xf)
    n = (dense & 0x7FFF != 0).sum(axis=1)
    yr = y_ref.view(np.float16).astype(np.float64)
    ulp = np.spacing(np.abs(y_ref.view(np.float16))).astype(np.float64)
    return ulp + 2 * n * 2.0**-24 * s, yr


def within_bound(dense, x, y, y_ref) -> bool:
    bound, yr = tol_bound(dense, x, y_ref)
    dy = np.abs(y.view(np.float16).astype(np.float64) - yr)
    return bool((dy <= bound).all())


def to_dev(a: np.ndarray, device="cuda"):
    import torch

    a = np.ascontiguousarray(a)
    if a.dtype == np.uint16:
        return torch.from_numpy(a.view(np.int16).copy()).to(device).view(torch.float16)
    return torch.from_numpy(a.copy()).to(device)


def to_host_u16(t) -> np.ndarray:
    import torch

    return t.detach().contiguous().view(torch.int16).cpu().numpy().view(np.uint16)
