"""Operand handling for the drop-in facade (the reference's ``as_matrix``
contract, linalg.py:30-39, moved onto the device).

Accepted operands: numpy arrays / array-likes (returned results are numpy),
CPU torch tensors (uploaded; results come back as CPU tensors; pinned memory
gives asynchronous copies) and CUDA tensors (results stay on the device).
float32 operands run the FP32 (3xTF32) path, everything else is promoted to
float64 like the reference.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _ops
from ._ops import F32, F64


class Operand:
    __slots__ = ("t", "kind", "name")

    def __init__(self, t, kind, name):
        self.t, self.kind, self.name = t, kind, name


def _torch_dtype_for(dt) -> torch.dtype:
    return F32 if dt in (np.float32, F32) else F64


def upload(a, name: str = "matrix", device=None, dtype=None, check_finite: bool = True) -> Operand:
    dev = _ops.require_cuda(device)
    if isinstance(a, torch.Tensor):
        kind = "cuda" if a.is_cuda else "cpu"
        want = dtype or (a.dtype if a.dtype in (F32, F64) else F64)
        t = a
    else:
        arr = np.asarray(a)
        kind = "numpy"
        want = dtype or _torch_dtype_for(arr.dtype.type)
        if arr.ndim == 2 and arr.size:
            arr = np.ascontiguousarray(arr, dtype=np.float32 if want == F32 else np.float64)
        t = torch.from_numpy(arr) if arr.ndim == 2 and arr.size else torch.empty(arr.shape)
    if t.dim() != 2:
        raise ValueError(f"{name} must be 2-D, got ndim={t.dim()}")
    if t.numel() == 0:
        raise ValueError(f"{name} must be non-empty")
    if t.device != dev or t.dtype != want:
        t = t.to(device=dev, dtype=want, non_blocking=True)
    if t.stride(1) != 1 or t.stride(0) < t.shape[1]:
        t = t.contiguous()
    op = Operand(t, kind, name)
    if check_finite:
        ensure_finite(op)
    return op


def ensure_finite(op: Operand, nonfinite: torch.Tensor | None = None) -> None:
    """Raise ValueError on non-finite entries (one fused device reduction)."""
    if nonfinite is None:
        nonfinite = torch.zeros(1, dtype=torch.int64, device=op.t.device)
        _ops.sumsq(op.t, nonfinite=nonfinite)
    if int(nonfinite.item()) != 0:
        raise ValueError(f"{op.name} contains non-finite entries")


def common_dtype(*ops: Operand) -> torch.dtype:
    return F32 if all(o.t.dtype == F32 for o in ops) else F64


def as_dtype(op: Operand, dtype) -> torch.Tensor:
    return op.t if op.t.dtype == dtype else _ops.cast(op.t, dtype)


def download(t: torch.Tensor, kind: str):
    """Result back to the caller's kind.  Host results land in PINNED memory
    (pageable device->host copies of the 0.5 GB U run at a fraction of the
    link rate); numpy results are views of those pinned tensors."""
    if kind == "cuda":
        return t
    host = torch.empty(tuple(t.shape), dtype=t.dtype, pin_memory=True)
    host.copy_(t, non_blocking=True)
    torch.cuda.current_stream(t.device).synchronize()
    return host if kind == "cpu" else host.numpy()
