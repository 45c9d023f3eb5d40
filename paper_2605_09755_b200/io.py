"""Direct-to-device ingestion of the reference's file formats (SURVEY.md §8(f)
row 3; reference data_io.py:99-255, formats in pkg/README.md "File formats").

* ``.skpw`` (magic ``SKPW``, version byte 1, rows/cols as little-endian u64,
  row-major little-endian float64): ``read_skpw`` memory-maps the file and
  streams row blocks through two pinned staging buffers into a device tensor
  (optionally only a row range -- one rank's slab), casting to float32 on the
  device when asked; the float64 host copy the reference makes is skipped.
  Header checks and messages follow data_io.read_binary.
* MatrixMarket (array / coordinate, real, general / symmetric): streamed
  line chunk by line chunk (no whole-file ``readlines``), converted a chunk
  at a time, assembled in a pinned buffer and uploaded; symmetric storage is
  expanded.  Validations, messages and line numbers are the reference's
  (data_io.read_matrix_market).
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


class _MMSource:
    """Streams a MatrixMarket file: the banner, then the data lines (blank
    lines and ``%`` comments skipped) in chunks, with their 1-based line
    numbers; ``total`` is the number of lines read so far (the whole file at
    EOF -- the line the reference cites for count mismatches)."""

    CHUNK = 1 << 16

    def __init__(self, path):
        self.path = path
        self._fh = open(path, "r", encoding="ascii")
        self.total = 0

    def close(self):
        self._fh.close()

    def fail(self, lineno: int, message: str) -> ValueError:
        return ValueError(f"{self.path}:{lineno}: {message}")

    def banner(self) -> str | None:
        line = self._fh.readline()
        if line:
            self.total = 1
        return line or None

    def chunks(self):
        """Lists of (lineno, text) for the data lines, CHUNK at a time."""
        buf = []
        for line in self._fh:
            self.total += 1
            text = line.strip()
            if text and not text.startswith("%"):
                buf.append((self.total, text))
                if len(buf) >= self.CHUNK:
                    yield buf
                    buf = []
        if buf:
            yield buf


def _to_ints(src: _MMSource, vals, lines, what: str) -> list:
    try:
        return list(map(int, vals))
    except ValueError:
        for v, ln in zip(vals, lines):
            try:
                int(v)
            except ValueError:
                raise src.fail(ln, f"invalid {what}: {v!r}") from None
        raise


def _to_floats(src: _MMSource, vals, lines) -> list:
    try:
        return list(map(float, vals))
    except ValueError:
        for v, ln in zip(vals, lines):
            try:
                float(v)
            except ValueError:
                raise src.fail(ln, f"non-real value {v!r}") from None
        raise


def _mm_array(src: _MMSource, data, size_line: int, size_tok, symmetric: bool) -> np.ndarray:
    """Dense values in column order (all of column j, or its lower part from
    the diagonal when symmetric), written straight into the flat value buffer."""
    if len(size_tok) != 2:
        raise src.fail(size_line, "array size line must be 'rows cols'")
    rows = _to_ints(src, size_tok[:1], [size_line], "row count")[0]
    cols = _to_ints(src, size_tok[1:], [size_line], "column count")[0]
    if rows < 1 or cols < 1:
        raise src.fail(size_line, "dimensions must be positive")
    if symmetric and rows != cols:
        raise src.fail(size_line, "symmetric matrices must be square")
    want = rows * (rows + 1) // 2 if symmetric else rows * cols
    flat = np.empty(want, dtype=np.float64)
    got = 0
    for chunk in data:
        toks, where = [], []
        for ln, text in chunk:
            parts = text.split()
            toks.extend(parts)
            where.extend([ln] * len(parts))
        room = want - got
        flat[got:got + min(room, len(toks))] = _to_floats(src, toks[:room], where[:room])
        if len(toks) > room:
            raise src.fail(where[room], "more entries than rows*cols")
        got += len(toks)
    if got != want:
        raise src.fail(src.total, f"expected {want} entries, got {got}")
    host = _host_f64(rows, cols, zero=False)
    dense = host.numpy()
    if not symmetric:
        dense[:] = flat.reshape(cols, rows).T
        return host
    # packed lower triangle by columns: column j holds rows j..n-1
    starts = np.concatenate(([0], np.cumsum(np.arange(rows, 0, -1))))
    for j in range(cols):
        seg = flat[starts[j]:starts[j + 1]]
        dense[j:, j] = seg
        dense[j, j:] = seg
    return host


def _mm_coordinate(src: _MMSource, data, size_line: int, size_tok, symmetric: bool):
    if len(size_tok) != 3:
        raise src.fail(size_line, "coordinate size line must be 'rows cols nnz'")
    rows = _to_ints(src, size_tok[:1], [size_line], "row count")[0]
    cols = _to_ints(src, size_tok[1:2], [size_line], "column count")[0]
    nnz = _to_ints(src, size_tok[2:], [size_line], "non-zero count")[0]
    if rows < 1 or cols < 1 or nnz < 0:
        raise src.fail(size_line, "sizes must be positive")
    if symmetric and rows != cols:
        raise src.fail(size_line, "symmetric matrices must be square")
    host = _host_f64(rows, cols, zero=True)
    dense = host.numpy()
    seen = 0
    for chunk in data:
        # a line without three fields ends the chunk early; the lines before
        # it are checked first, as the reference checks line by line
        fields, lines, short = [], [], None
        for ln, text in chunk:
            parts = text.split()
            if len(parts) != 3:
                short = src.fail(ln, f"expected 'i j value', got {text!r}")
                break
            fields.append(parts)
            lines.append(ln)
        try:
            ii = np.asarray(list(map(int, (f[0] for f in fields))), dtype=np.int64)
            jj = np.asarray(list(map(int, (f[1] for f in fields))), dtype=np.int64)
            vv = np.asarray(list(map(float, (f[2] for f in fields))), dtype=np.float64)
        except ValueError:
            # locate the first failing line and check (row index, column
            # index, value, bounds -- the reference's order)
            for ln, (ti, tj, tv) in zip(lines, fields):
                i = _to_ints(src, [ti], [ln], "row index")[0]
                j = _to_ints(src, [tj], [ln], "column index")[0]
                _to_floats(src, [tv], [ln])
                if not (1 <= i <= rows and 1 <= j <= cols):
                    raise src.fail(ln, f"index ({i}, {j}) out of bounds for {rows}x{cols}")
            raise
        bad = np.flatnonzero((ii < 1) | (ii > rows) | (jj < 1) | (jj > cols))
        if bad.size:
            b = int(bad[0])
            raise src.fail(lines[b], f"index ({ii[b]}, {jj[b]}) out of bounds for {rows}x{cols}")
        # file order decides repeated coordinates: the last write wins (the
        # symmetric mirror write follows each entry); numpy's fancy assignment
        # leaves the winner of duplicates unspecified, so keep only the last
        # write per cell explicitly
        if symmetric:
            r_ = np.stack([ii - 1, jj - 1], axis=1).ravel()
            c_ = np.stack([jj - 1, ii - 1], axis=1).ravel()
            v_ = np.repeat(vv, 2)
        else:
            r_, c_, v_ = ii - 1, jj - 1, vv
        flat_idx = r_ * cols + c_
        _, last = np.unique(flat_idx[::-1], return_index=True)
        keep = len(flat_idx) - 1 - last
        dense.reshape(-1)[flat_idx[keep]] = v_[keep]
        seen += len(fields)
        if short is not None:
            raise short
    if seen != nnz:
        raise src.fail(src.total, f"expected {nnz} entries, got {seen}")
    return host


def read_matrix_market_host(path) -> torch.Tensor:
    """The host half of read_matrix_market: parse and validate into a float64
    host tensor (pinned when a CUDA device is present)."""
    src = _MMSource(path)
    try:
        first = src.banner()
        if first is None:
            raise src.fail(1, "empty file")
        words = first.split()
        if len(words) != 5 or words[0] != "%%MatrixMarket" or words[1].lower() != "matrix":
            raise src.fail(1, f"malformed MatrixMarket header: {first.rstrip()!r}")
        layout, field, symmetry = (w.lower() for w in words[2:])
        if layout not in ("array", "coordinate"):
            raise src.fail(1, f"unsupported format {layout!r}")
        if field != "real":
            raise src.fail(1, f"unsupported field {field!r} (only real)")
        if symmetry not in ("general", "symmetric"):
            raise src.fail(1, f"unsupported symmetry {symmetry!r}")
        data = src.chunks()
        head = next(data, None)
        if head is None:
            raise src.fail(src.total, "missing size line")
        size_line, size_text = head[0]

        def rest():
            if len(head) > 1:
                yield head[1:]
            yield from data
        parse = _mm_array if layout == "array" else _mm_coordinate
        return parse(src, rest(), size_line, size_text.split(), symmetry == "symmetric")
    finally:
        src.close()


def _host_f64(rows: int, cols: int, zero: bool) -> torch.Tensor:
    pin = torch.cuda.is_available()
    if zero:
        return torch.zeros((rows, cols), dtype=F64, pin_memory=pin)
    return torch.empty((rows, cols), dtype=F64, pin_memory=pin)


def read_matrix_market(path, device=None, dtype=torch.float64) -> torch.Tensor:
    """A real MatrixMarket file (array or coordinate, general or symmetric) as a
    device tensor; symmetric storage expanded (data_io.read_matrix_market,
    data_io.py:99-206: same checks, messages and line numbers).  The file is
    streamed in chunks of lines into a pinned host matrix, uploaded once and
    checked for non-finite entries on the device."""
    dev = _ops.require_cuda(device)
    host = read_matrix_market_host(path)
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
