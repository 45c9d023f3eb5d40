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
    if isinstance(a, DeviceMatrix):
        op = a.resident()
        if dtype is not None and op.t.dtype != dtype:
            op = Operand(_ops.cast(op.t, dtype), op.kind, name)
        if check_finite and not a.finite:
            ensure_finite(op)
            a.finite = True
        return op
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
    if not t.is_cuda:
        # host operands land in 128-byte rows (_ops.empty2d): the TMA / tcgen05
        # paths (K2 v2's row copies, randsvd's in-kernel split of A) need them,
        # and an unaligned n would otherwise fall back to slower kernels
        if t.dtype != want:
            t = t.to(dtype=want)
        dst = _ops.empty2d(t.shape[0], t.shape[1], want, dev)
        dst.copy_(t, non_blocking=t.is_pinned())
        t = dst
    else:
        if t.device != dev or t.dtype != want:
            t = t.to(device=dev, dtype=want, non_blocking=True)
        per = 128 // t.element_size()
        if t.stride(1) != 1 or t.stride(0) < t.shape[1] or (
                t.stride(0) % per and _aligned_copy_fits(t)):
            # a device operand with unaligned rows: one padded copy (when it
            # fits) instead of the fallback kernels for every product
            dst = _ops.empty2d(t.shape[0], t.shape[1], t.dtype, dev)
            dst.copy_(t)
            t = dst
    op = Operand(t, kind, name)
    if check_finite:
        ensure_finite(op)
    return op


def _aligned_copy_fits(t: torch.Tensor) -> bool:
    """Room for a padded copy of t (allocator counters, no device sync)."""
    need = 2 * t.shape[0] * (t.shape[1] + 32) * t.element_size() + (1 << 30)
    return _ops._device_total(t.device) - torch.cuda.memory_allocated(t.device) >= need


class Streamed:
    """A host matrix bound for the device in row blocks: ``t`` is the device
    destination (128-byte rows), allocated but not yet filled; ``blocks()``
    issues the H2D copy of each block on a side stream and makes the current
    stream wait for it, so a consumer can start on block b while blocks
    b+1.. are still on the link (the range finder sketches behind the copy)."""

    BLOCK_BYTES = 1 << 30

    def __init__(self, src: torch.Tensor, dst: torch.Tensor):
        self.src, self.t = src, dst
        self.rows_per_block = max(1, self.BLOCK_BYTES // max(1, src.shape[1] * src.element_size()))
        self.done = False

    def blocks(self):
        m = self.t.shape[0]
        dev = self.t.device
        side = torch.cuda.Stream(dev)
        cur = torch.cuda.current_stream(dev)
        side.wait_stream(cur)   # the destination's allocation is ordered on cur
        for r0 in range(0, m, self.rows_per_block):
            r1 = min(m, r0 + self.rows_per_block)
            with torch.cuda.stream(side):
                self.t[r0:r1].copy_(self.src[r0:r1], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(side)
            cur.wait_event(ev)
            yield r0, r1
        self.t.record_stream(side)
        self.done = True


def upload_streamed(a, name: str = "matrix", device=None):
    """(Operand, Streamed | None): like upload(check_finite=False), except that
    a host 2-D float32/float64 matrix is NOT copied yet -- the caller drives
    the copy block by block through Streamed.blocks()."""
    if isinstance(a, DeviceMatrix):
        return a.take()
    dev = _ops.require_cuda(device)
    if isinstance(a, torch.Tensor) and (a.is_cuda or a.dim() != 2 or a.dtype not in (F32, F64)):
        return upload(a, name, device, check_finite=False), None
    if isinstance(a, torch.Tensor):
        src, kind = a, "cpu"
    else:
        arr = np.asarray(a)
        if arr.ndim != 2 or arr.size == 0:
            return upload(a, name, device, check_finite=False), None
        want = np.float32 if _torch_dtype_for(arr.dtype.type) == F32 else np.float64
        src, kind = torch.from_numpy(np.ascontiguousarray(arr, dtype=want)), "numpy"
    if src.numel() == 0:
        raise ValueError(f"{name} must be non-empty")
    if src.stride(1) != 1:
        src = src.contiguous()
    dst = _ops.empty2d(src.shape[0], src.shape[1], src.dtype, dev)
    return Operand(dst, kind, name), Streamed(src, dst)


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


class DeviceMatrix:
    """A host matrix uploaded ONCE for a sequence of reference calls, e.g. the
    drop-in pair ``range_finder_sketched(A, spec)`` then ``randsvd(A, Q)``
    (power.py:141, :181), each of which would otherwise copy ``a`` to the
    device again.  Nothing is copied at construction: the first call that
    takes the matrix streams it in row blocks behind its own sketch (as
    ``rsvd`` does); later calls use the resident copy.  Results keep the
    caller's kind (numpy in, numpy out).  The caller must not modify ``a``
    while the handle is in use (the device copy would not follow)."""

    def __init__(self, a, device=None):
        self.op, self._streamed = upload_streamed(a, "a", device)
        self.finite = False      # set by the first call that tested every entry
        self._taken = False

    @property
    def shape(self):
        return tuple(self.op.t.shape)

    @property
    def dtype(self):
        return self.op.t.dtype

    def take(self):
        """(Operand, Streamed | None) for the first consumer; (Operand, None) after."""
        if self._streamed is not None and not self._taken:
            self._taken = True
            return self.op, self._streamed
        return self.resident(), None

    def resident(self) -> Operand:
        """The operand with every row on the device."""
        st = self._streamed
        if st is not None and not st.done:
            if self._taken:      # a consumer stopped part way: copy it all again
                self.op.t.copy_(st.src, non_blocking=True)
                st.done = True
            else:
                self._taken = True
                for _ in st.blocks():
                    pass
        return self.op


def device_matrix(a, device=None) -> DeviceMatrix:
    """Upload handle for reusing one device copy of ``a`` across calls."""
    if isinstance(a, DeviceMatrix):
        return a
    return DeviceMatrix(a, device)
