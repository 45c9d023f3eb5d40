"""Direct-to-device ingestion of the reference's file formats (SURVEY.md §8(f)
row 3; reference data_io.py:99-255, formats in pkg/README.md "File formats").

* ``.skpw`` (magic ``SKPW``, version byte 1, rows/cols as little-endian u64,
  row-major little-endian float64): ``read_skpw`` memory-maps the file and
  streams row blocks through two pinned staging buffers into a device tensor
  (optionally only a row range -- one rank's slab), casting to float32 on the
  device when asked; the float64 host copy the reference makes is skipped.
  Header checks and messages follow data_io.read_binary.
* MatrixMarket (array / coordinate, real, general / symmetric): parsed on the
  host with the reference's validations and line-numbered messages
  (data_io.read_matrix_market), assembled in a pinned buffer and uploaded;
  symmetric storage is expanded.
"""
from __future__ import annotations

import os
import struct

import numpy as np
import torch

from . import _ops
from ._ops import F32, F64

_MAGIC = b"SKPW"
_VERSION = 1
_HEADER = 21


def _skpw_header(path) -> tuple[int, int]:
    size = os.path.getsize(path)
    with open(path, "rb") as fh:
        head = fh.read(_HEADER)
    if len(head) < _HEADER:
        raise ValueError(f"{path}: truncated header ({len(head)} bytes)")
    if head[:4] != _MAGIC:
        raise ValueError(f"{path}: bad magic {head[:4]!r}")
    if head[4] != _VERSION:
        raise ValueError(f"{path}: unsupported version {head[4]}")
    rows, cols = struct.unpack("<QQ", head[5:21])
    expected = _HEADER + rows * cols * 8
    if size != expected:
        raise ValueError(f"{path}: expected {expected} bytes, got {size}")
    return rows, cols


def skpw_shape(path) -> tuple[int, int]:
    """(rows, cols) of a .skpw file (header validated)."""
    return _skpw_header(path)


def read_skpw(path, device=None, dtype=torch.float64, rows: tuple[int, int] | None = None,
              block_bytes: int = 64 << 20, check_finite: bool = True) -> torch.Tensor:
    """Rows [r0, r1) (all by default) of a .skpw file as a device tensor with
    128-byte aligned rows (the layout every libskp kernel prefers).  Raises
    ValueError like the reference for truncated / corrupt files and for
    non-finite data (as_matrix, linalg.py:30-39)."""
    dev = _ops.require_cuda(device)
    if dtype not in (F64, F32):
        raise ValueError("dtype must be torch.float64 or torch.float32")
    m, n = _skpw_header(path)
    r0, r1 = (0, m) if rows is None else rows
    if not 0 <= r0 <= r1 <= m:
        raise ValueError(f"row range {rows} outside 0..{m}")
    out = _ops.empty2d(r1 - r0, n, dtype, dev)
    if r1 == r0 or n == 0:
        return out
    data = np.memmap(path, dtype="<f8", mode="r", offset=_HEADER, shape=(m, n))
    per = max(1, block_bytes // (8 * n))
    stage = [torch.empty((per, n), dtype=F64, pin_memory=True) for _ in range(2)]
    dev64 = None if dtype == F64 else _ops.empty2d(min(per, r1 - r0), n, F64, dev)
    done = [None, None]
    cur = torch.cuda.current_stream(dev)
    for bi, b0 in enumerate(range(r0, r1, per)):
        b1 = min(r1, b0 + per)
        buf = stage[bi & 1]
        if done[bi & 1] is not None:
            done[bi & 1].synchronize()          # staging buffer free again
        np.copyto(buf[: b1 - b0].numpy(), data[b0:b1])
        if dtype == F64:
            out[b0 - r0:b1 - r0].copy_(buf[: b1 - b0], non_blocking=True)
        else:
            dev64[: b1 - b0].copy_(buf[: b1 - b0], non_blocking=True)
            out[b0 - r0:b1 - r0].copy_(_ops.cast(dev64[: b1 - b0], F32))
        ev = torch.cuda.Event()
        ev.record(cur)
        done[bi & 1] = ev
    cur.synchronize()
    del data
    if check_finite:
        bad = torch.zeros(1, dtype=torch.int64, device=dev)
        _ops.sumsq(out, nonfinite=bad)
        if int(bad.item()) != 0:
            raise ValueError("binary data contains non-finite entries")
    return out


def write_skpw(a, path) -> None:
    """Write the SKPW format (bit-exact round trip with read_skpw / the reference)."""
    arr = a.detach().to("cpu", torch.float64).numpy() if isinstance(a, torch.Tensor) else np.asarray(a, dtype=np.float64)
    if arr.ndim != 2 or arr.size == 0:
        raise ValueError("a must be a non-empty 2-D matrix")
    if not np.isfinite(arr).all():
        raise ValueError("a contains non-finite entries")
    with open(path, "wb") as fh:
        fh.write(_MAGIC)
        fh.write(bytes([_VERSION]))
        fh.write(struct.pack("<QQ", arr.shape[0], arr.shape[1]))
        fh.write(np.ascontiguousarray(arr, dtype="<f8").tobytes())


def _mm_error(path, lineno: int, message: str) -> ValueError:
    return ValueError(f"{path}:{lineno}: {message}")


def read_matrix_market(path, device=None, dtype=torch.float64) -> torch.Tensor:
    """A real MatrixMarket file (array or coordinate, general or symmetric) as a
    device tensor; symmetric storage expanded.  Malformed headers,
    out-of-bounds indices and non-real fields raise ValueError with the line
    number, as data_io.read_matrix_market does."""
    dev = _ops.require_cuda(device)
    with open(path, "r", encoding="ascii") as fh:
        lines = fh.readlines()
    if not lines:
        raise _mm_error(path, 1, "empty file")
    header = lines[0].split()
    if len(header) != 5 or header[0] != "%%MatrixMarket" or header[1].lower() != "matrix":
        raise _mm_error(path, 1, f"malformed MatrixMarket header: {lines[0].rstrip()!r}")
    fmt, field_kind, symmetry = (tok.lower() for tok in header[2:5])
    if fmt not in ("array", "coordinate"):
        raise _mm_error(path, 1, f"unsupported format {fmt!r}")
    if field_kind != "real":
        raise _mm_error(path, 1, f"unsupported field {field_kind!r} (only real)")
    if symmetry not in ("general", "symmetric"):
        raise _mm_error(path, 1, f"unsupported symmetry {symmetry!r}")
    idx = 1
    while idx < len(lines) and (lines[idx].startswith("%") or not lines[idx].strip()):
        idx += 1
    if idx >= len(lines):
        raise _mm_error(path, len(lines), "missing size line")
    size_tokens = lines[idx].split()
    lineno = idx + 1

    def _int(tok, what, ln):
        try:
            return int(tok)
        except ValueError:
            raise _mm_error(path, ln, f"invalid {what}: {tok!r}") from None

    host = None
    if fmt == "array":
        if len(size_tokens) != 2:
            raise _mm_error(path, lineno, "array size line must be 'rows cols'")
        rows, cols = _int(size_tokens[0], "row count", lineno), _int(size_tokens[1], "column count", lineno)
        if rows < 1 or cols < 1:
            raise _mm_error(path, lineno, "dimensions must be positive")
        if symmetry == "symmetric" and rows != cols:
            raise _mm_error(path, lineno, "symmetric matrices must be square")
        # column-major values (general) or the lower triangle by columns (symmetric)
        total = rows * cols if symmetry == "general" else rows * (rows + 1) // 2
        vals = np.empty(total, dtype=np.float64)
        pos = 0
        for offset, line in enumerate(lines[idx + 1:], start=idx + 2):
            text = line.strip()
            if not text or text.startswith("%"):
                continue
            for tok in text.split():
                if pos >= total:
                    raise _mm_error(path, offset, "more entries than rows*cols")
                try:
                    vals[pos] = float(tok)
                except ValueError:
                    raise _mm_error(path, offset, f"non-real value {tok!r}") from None
                pos += 1
        if pos != total:
            raise _mm_error(path, len(lines), f"expected {total} entries, got {pos}")
        host = torch.zeros((rows, cols), dtype=F64, pin_memory=True)
        hn = host.numpy()
        if symmetry == "general":
            hn[:] = vals.reshape(cols, rows).T
        else:
            jj = np.repeat(np.arange(cols), np.arange(rows, 0, -1))
            ii = np.concatenate([np.arange(j, rows) for j in range(cols)])
            hn[ii, jj] = vals
            hn[jj, ii] = vals
    else:
        if len(size_tokens) != 3:
            raise _mm_error(path, lineno, "coordinate size line must be 'rows cols nnz'")
        rows = _int(size_tokens[0], "row count", lineno)
        cols = _int(size_tokens[1], "column count", lineno)
        nnz = _int(size_tokens[2], "non-zero count", lineno)
        if rows < 1 or cols < 1 or nnz < 0:
            raise _mm_error(path, lineno, "sizes must be positive")
        if symmetry == "symmetric" and rows != cols:
            raise _mm_error(path, lineno, "symmetric matrices must be square")
        host = torch.zeros((rows, cols), dtype=F64, pin_memory=True)
        hn = host.numpy()
        seen = 0
        for offset, line in enumerate(lines[idx + 1:], start=idx + 2):
            text = line.strip()
            if not text or text.startswith("%"):
                continue
            tokens = text.split()
            if len(tokens) != 3:
                raise _mm_error(path, offset, f"expected 'i j value', got {text!r}")
            i, j = _int(tokens[0], "row index", offset), _int(tokens[1], "column index", offset)
            try:
                value = float(tokens[2])
            except ValueError:
                raise _mm_error(path, offset, f"non-real value {tokens[2]!r}") from None
            if not (1 <= i <= rows and 1 <= j <= cols):
                raise _mm_error(path, offset, f"index ({i}, {j}) out of bounds for {rows}x{cols}")
            hn[i - 1, j - 1] = value
            if symmetry == "symmetric":
                hn[j - 1, i - 1] = value
            seen += 1
        if seen != nnz:
            raise _mm_error(path, len(lines), f"expected {nnz} entries, got {seen}")
    out = _ops.empty2d(host.shape[0], host.shape[1], dtype, dev)
    if dtype == F64:
        out.copy_(host, non_blocking=True)
    else:
        tmp = _ops.empty2d(host.shape[0], host.shape[1], F64, dev)
        tmp.copy_(host, non_blocking=True)
        out.copy_(_ops.cast(tmp, F32))
    torch.cuda.current_stream(dev).synchronize()
    bad = torch.zeros(1, dtype=torch.int64, device=dev)
    _ops.sumsq(out, nonfinite=bad)
    if int(bad.item()) != 0:
        raise ValueError("matrix-market data contains non-finite entries")
    return out
