"""Device operations over torch CUDA tensors, each one libskp call (or a few).

torch is plumbing here: device memory, the current stream and dtype tags.
Every arithmetic step runs in libskp.so kernels; nothing falls back to torch
or the CPU.  ``CudaBackend`` is the compute backend the algorithm engine
(``_engine.py``) drives.
"""
from __future__ import annotations

import threading

import numpy as np
import torch

from . import _lib
from ._lib import call

F32, F64 = torch.float32, torch.float64
_SFX = {F32: "f32", F64: "f64"}


def require_cuda(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2605_09755_b200 needs a CUDA device (sm_100a); "
                           "there is no CPU fallback")
    _lib.load()
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    d = torch.device(device)
    if d.type != "cuda":
        raise ValueError(f"device must be a CUDA device, got {d}")
    return d if d.index is not None else torch.device("cuda", torch.cuda.current_device())


def stream_ptr(device=None) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


class _Workspace(threading.local):
    """Per-thread, per-device scratch (callers on different threads never share)."""

    def __init__(self):
        self.buf = {}

    def get(self, device: torch.device, nbytes: int) -> torch.Tensor:
        key = (device.index, torch.cuda.current_stream(device).cuda_stream)
        b = self.buf.get(key)
        if b is None or b.numel() < nbytes:
            b = torch.empty(max(int(nbytes), 1 << 20), dtype=torch.uint8, device=device)
            self.buf[key] = b
        return b


_WS = _Workspace()


_TOTAL_MEM: dict = {}


def _device_total(device) -> int:
    """Total HBM of a device (cached host-side: no driver query per call)."""
    idx = torch.device(device).index
    if idx is None:
        idx = torch.cuda.current_device()
    if idx not in _TOTAL_MEM:
        _TOTAL_MEM[idx] = torch.cuda.get_device_properties(idx).total_memory
    return _TOTAL_MEM[idx]


def workspace(device, nbytes: int) -> torch.Tensor:
    return _WS.get(device, nbytes)


def empty2d(rows: int, cols: int, dtype, device) -> torch.Tensor:
    """rows x cols view of a buffer whose rows start on 128-byte boundaries
    (leading dimension rounded up to 32 fp32 / 16 fp64): TMA needs 16-byte
    aligned rows, and the GEMM's one-box-per-stage 3-D view of an MN-major
    operand needs 32-element chunks that never cross a row."""
    per = 128 // torch.empty((), dtype=dtype).element_size()
    ld = max(per, (cols + per - 1) // per * per)
    return torch.empty((rows, ld), dtype=dtype, device=device)[:, :cols]


def aligned2d(t: torch.Tensor) -> torch.Tensor:
    """t itself if its rows are 16-byte aligned, else a padded copy."""
    es = t.element_size()
    if t.stride(1) == 1 and (t.stride(0) * es) % 16 == 0 and t.data_ptr() % 16 == 0:
        return t
    out = empty2d(t.shape[0], t.shape[1], t.dtype, t.device)
    out.copy_(t)
    return out


def _rows_ld(x: torch.Tensor):
    if x.dim() != 2:
        raise ValueError(f"expected a 2-D tensor, got shape {tuple(x.shape)}")
    if x.stride(1) != 1:
        raise ValueError("expected unit column stride (row-major)")
    return x.shape[0], x.shape[1], x.stride(0)


# --------------------------------------------------------------- sketch ----

def countsketch(state: int, inc: int, n: int, r: int, s: int, device, j0: int = 0,
                j1: int | None = None):
    """K1: rows [j0, j1) of (cols int32 (rows, s), signs int8 (rows, s))."""
    j1 = n if j1 is None else j1
    m64 = (1 << 64) - 1
    cols = torch.empty((j1 - j0, s), dtype=torch.int32, device=device)
    signs = torch.empty((j1 - j0, s), dtype=torch.int8, device=device)
    lib = _lib.load()
    wsb = lib.skp_countsketch_ws_bytes(n, r, s)
    ws = workspace(device, wsb) if wsb else None
    call("skp_countsketch_gen", (state >> 64) & m64, state & m64, (inc >> 64) & m64, inc & m64,
         n, r, s, j0, j1, ptr(cols), ptr(signs), ptr(ws), wsb, stream_ptr(device))
    return cols, signs


def csc(cols: torch.Tensor, signs: torch.Tensor, n: int, s: int, r: int):
    """CSC view of S: (colptr int32 (r+1,), entries int32 (n*s,))."""
    dev = cols.device
    colptr = torch.empty(r + 1, dtype=torch.int32, device=dev)
    entries = torch.empty(n * s, dtype=torch.int32, device=dev)
    wsb = _lib.load().skp_countsketch_csc_ws_bytes(n, s, r)
    ws = workspace(dev, wsb)
    call("skp_countsketch_csc", ptr(cols), ptr(signs), n, s, r, ptr(colptr), ptr(entries),
         ptr(ws), wsb, stream_ptr(dev))
    return colptr, entries


def sketch_right(a: torch.Tensor, colptr, entries, s: int, r: int, out=None, fro2=None,
                 nonfinite=None):
    """K2: a (m x n) @ S -> (m x r), fused ||a||_F^2 / non-finite count."""
    m, n, lda = _rows_ld(a)
    if out is None:
        out = empty2d(m, r, a.dtype, a.device)
    _, _, ldo = _rows_ld(out)
    wsb = _lib.load().skp_sketch_right_ws_bytes(n, s, r, a.element_size())
    ws = workspace(a.device, wsb)
    call(f"skp_sketch_right_{_SFX[a.dtype]}", ptr(a), lda, m, n, ptr(colptr), ptr(entries), s, r,
         ptr(out), ldo, ptr(fro2), ptr(nonfinite), ptr(ws), wsb, stream_ptr(a.device))
    return out


GATHER_PLAN_FAIL_MARK = 1 << 40   # added to the non-finite counter by a failed plan


def gather_plan(colptr, entries, n: int, r: int, device, check: bool = True):
    """K2 v2 plan (once per sketch): (plan bytes on the device, perm or None).

    None when the shape is outside the kernel (n > 98304).  With check=True the
    schedule is verified on the host (one sync; None if a column / warp needs
    more than 128 steps) and perm[v] (numpy) = the column written at position v.
    With check=False nothing is read back: a failed schedule surfaces as
    GATHER_PLAN_FAIL_MARK in the non-finite counter of sketch_gather."""
    lib = _lib.load()
    nb = int(lib.skp_sketch_gather_plan_bytes(n, r))
    plan = torch.empty(nb, dtype=torch.uint8, device=device)
    rc = lib.skp_sketch_gather_plan(ptr(colptr), ptr(entries), n, r, ptr(plan), nb,
                                    stream_ptr(device))
    if rc == _lib.SKP_ERR_UNSUPPORTED:
        return None
    _lib.check(rc, "skp_sketch_gather_plan")
    if not check:
        return plan, None
    return gather_plan_checked(plan, r)


def gather_plan_checked(plan: torch.Tensor, r: int):
    """(plan, perm) after the host check of a built plan, or None if it failed."""
    off = int(_lib.load().skp_sketch_gather_plan_fail_offset(r))
    if int(plan[off:off + 4].view(torch.int32).item()) != 0:
        return None
    # the plan starts with the perm table (P slices x kGCols int32), which
    # ends where the fail word begins
    perm = plan[:off].view(torch.int32).cpu().numpy()
    return plan, perm[perm >= 0].astype(np.int64)


def sketch_gather(a: torch.Tensor, plan: torch.Tensor, r: int, s: int, out=None, fro2=None,
                  nonfinite=None, amax=None, out_dtype=None):
    """K2 v2: (a @ S) with the plan's column permutation, fused ||a||_F^2 and
    non-finite test; fp32 a with 16-byte aligned rows (empty2d).  amax (int32
    view, 1 element, zeroed by the caller): atomicMax of max|out|'s bits.
    out_dtype=float64: fp64 accumulation and output (no amax)."""
    m, n, lda = _rows_ld(a)
    od = out_dtype or (out.dtype if out is not None else a.dtype)
    if out is None:
        out = empty2d(m, r, od, a.device)
    _, _, ldo = _rows_ld(out)
    if od == F64:
        call("skp_sketch_gather_f32_acc64", ptr(a), lda, m, n, r, ptr(plan), 1.0 / float(np.sqrt(s)),
             ptr(out), ldo, ptr(fro2), ptr(nonfinite), stream_ptr(a.device))
        return out
    call("skp_sketch_gather_f32", ptr(a), lda, m, n, r, ptr(plan), 1.0 / float(np.sqrt(s)),
         ptr(out), ldo, ptr(fro2), ptr(nonfinite), ptr(amax), stream_ptr(a.device))
    return out


OMEGA_FAIL_MARK = 1 << 50   # added to a counter by a device Gaussian draw that failed


def gaussian(st: int, inc: int, rows: int, cols: int, divisor: float, dtype, device,
             fail_counter=None, out=None) -> torch.Tensor:
    """numpy Generator(PCG64(st, inc)).standard_normal((rows, cols)) / divisor
    on the device (the reference's Gaussian Omega), fp32 or fp64."""
    if out is None:
        out = empty2d(rows, cols, dtype, device)
    _, _, ldo = _rows_ld(out)
    lib = _lib.load()
    wsb = int(lib.skp_gaussian_ws_bytes(rows * cols))
    ws = workspace(out.device, wsb) if wsb else None
    m64 = (1 << 64) - 1
    call(f"skp_gaussian_{_SFX[dtype]}", st >> 64, st & m64, inc >> 64, inc & m64, rows, cols,
         float(divisor), ptr(out), ldo, ptr(fail_counter), ptr(ws), wsb, stream_ptr(out.device))
    return out


def gesvj(a: torch.Tensor, max_sweeps: int = 40):
    """One-sided Jacobi thin SVD of a (m x n, m >= n; fp32 or fp64): fp64
    (U m x n, S n descending, V n x n) -- skp_gesvj."""
    m, n, lda = _rows_ld(a)
    dev = a.device
    s = torch.empty(n, dtype=F64, device=dev)
    u = empty2d(m, n, F64, dev)
    v = empty2d(n, n, F64, dev)
    sweeps = torch.zeros(1, dtype=torch.int32, device=dev)
    wsb = int(_lib.load().skp_gesvj_ws_bytes(m, n))
    ws = workspace(dev, wsb)
    call(f"skp_gesvj_{_SFX[a.dtype]}", ptr(a), m, n, lda, ptr(s), ptr(u), u.stride(0), ptr(v),
         v.stride(0), max_sweeps, ptr(ws), wsb, ptr(sweeps), stream_ptr(dev))
    return u, s, v


def sym_check(x: torch.Tensor) -> torch.Tensor:
    """(max |x - x^T|, max |x|) as a float64 device tensor of 2, reading the
    square matrix x once (skp_sym_check)."""
    n, _, ld = _rows_ld(x)
    out = torch.empty(2, dtype=F64, device=x.device)
    call(f"skp_sym_check_{_SFX[x.dtype]}", ptr(x), n, ld, ptr(out), stream_ptr(x.device))
    return out


UNPERMUTE_MAX_COLS = 25600   # skp_unpermute_cols_f32's shared-memory row


def unpermute_cols(x: torch.Tensor, perm_dev: torch.Tensor) -> torch.Tensor:
    """In place: x[:, perm_dev[v]] = x[:, v] (the K2 v2 output back in the
    natural column order).  Returns x."""
    rows, cols, ldx = _rows_ld(x)
    call(f"skp_unpermute_cols_{_SFX[x.dtype]}", ptr(x), rows, cols, ldx, ptr(perm_dev),
         stream_ptr(x.device))
    return x


def permute_rows(x: torch.Tensor, perm_dev: torch.Tensor, out=None) -> torch.Tensor:
    """out[v, :] = x[perm_dev[v], :] for v < x.shape[0] (perm_dev: int32 on the device)."""
    rows, cols, ldx = _rows_ld(x)
    if out is None:
        out = empty2d(rows, cols, x.dtype, x.device)
    _, _, ldy = _rows_ld(out)
    call(f"skp_permute_rows_{_SFX[x.dtype]}", ptr(x), ldx, ptr(perm_dev), ptr(out), ldy, rows,
         cols, stream_ptr(x.device))
    return out


def sketch_left_t(x: torch.Tensor, colptr, entries, s: int, r: int, out=None):
    """K3: S^T @ x (x n x c) -> (r x c)."""
    n, c, ldx = _rows_ld(x)
    if out is None:
        out = empty2d(r, c, x.dtype, x.device)
    _, _, ldo = _rows_ld(out)
    call(f"skp_sketch_left_t_{_SFX[x.dtype]}", ptr(x), ldx, n, c, ptr(colptr), ptr(entries), s, r,
         ptr(out), ldo, stream_ptr(x.device))
    return out


# ----------------------------------------------------------------- gemm ----

GEMM_MODE = {"auto": 0, "3xtf32": 1, "fp32": 2}


def gemm(a, b, ta: bool = False, tb: bool = False, alpha: float = 1.0, beta: float = 0.0,
         out=None, mode: str = "auto"):
    """K4: out = alpha * op(a) @ op(b) + beta * out."""
    if a.dtype != b.dtype:
        raise ValueError("gemm operands must share a dtype")
    ra, ca, lda = _rows_ld(a)
    rb, cb, ldb = _rows_ld(b)
    M, K = (ca, ra) if ta else (ra, ca)
    Kb, N = (cb, rb) if tb else (rb, cb)
    if K != Kb:
        raise ValueError(f"dimension mismatch: {M}x{K} @ {Kb}x{N}")
    if out is None:
        out = empty2d(M, N, a.dtype, a.device)
        if beta != 0.0:
            raise ValueError("beta != 0 needs out")
    _, _, ldc = _rows_ld(out)
    lib = _lib.load()
    eb = 4 if a.dtype == F32 else 8
    md = GEMM_MODE[mode]
    wsb = lib.skp_gemm_ws_bytes(int(ta), int(tb), M, N, K, eb, md)
    ws = workspace(a.device, wsb) if wsb else None
    call(f"skp_gemm_{_SFX[a.dtype]}", int(ta), int(tb), M, N, K, alpha, ptr(a), lda, ptr(b), ldb,
         beta, ptr(out), ldc, md, ptr(ws), wsb, stream_ptr(a.device))
    return out


def srht(x: torch.Tensor, signs: torch.Tensor, n_pad: int, subset: torch.Tensor, r: int,
         left_t: bool, out=None) -> torch.Tensor:
    """K7: x S (left_t=False; x is m x n, fibres = rows) or S^T x (left_t=True;
    x is n x c, fibres = columns) for the SRHT S (sketching.py:167-171, :185-189)."""
    rows, cols, ld = _rows_ld(x)
    if left_t:
        fibres, n, x_fs, x_es = cols, rows, 1, ld
        if out is None:
            out = empty2d(r, cols, x.dtype, x.device)
        _, _, ldo = _rows_ld(out)
        o_fs, o_es = 1, ldo
    else:
        fibres, n, x_fs, x_es = rows, cols, ld, 1
        if out is None:
            out = empty2d(rows, r, x.dtype, x.device)
        _, _, ldo = _rows_ld(out)
        o_fs, o_es = ldo, 1
    call(f"skp_srht_apply_{_SFX[x.dtype]}", ptr(x), fibres, n, x_fs, x_es, ptr(signs), n_pad,
         ptr(subset), r, 1.0 / float(np.sqrt(r)), ptr(out), o_fs, o_es, stream_ptr(x.device))
    return out


# ------------------------------------------------ 3xFP16 (pre-split) GEMM --

H3_MIN_ELEMS = 1 << 22   # prepare() splits left operands of at least this many entries


class SplitH2:
    """fp16 two-term split of an fp32 matrix with one power-of-two scale:
    x 2^e ~= hi + lo (skp_split_h2_f32).  ``t`` (rows x cols as stored in the
    planes) is the source or, with trans=True, its transpose; planes have
    128-byte rows (ld % 64 == 0) so either major-ness can be TMA-loaded."""
    __slots__ = ("hi", "lo", "e", "rows", "cols", "ld")

    def __init__(self, hi, lo, e, rows, cols, ld):
        self.hi, self.lo, self.e, self.rows, self.cols, self.ld = hi, lo, e, rows, cols, ld


def gram_pays(l: int, r2: int, q: int) -> bool:
    """The sketch-space power iteration's cost rule (CudaBackend.gram_ok)."""
    return l <= q * r2 * (4.4 + 1.5 * r2 / l)


def split_h2(x: torch.Tensor, trans: bool = False, out: "SplitH2 | None" = None,
             e_io: torch.Tensor | None = None) -> SplitH2:
    """e_io (int32[2]): e_io[1] already holds max|x|'s bits (e.g. the sketch
    kernel's amax output), so the max pass is skipped; e_io becomes out.e."""
    r, c, ld = _rows_ld(x)
    if x.dtype != F32:
        raise ValueError("split_h2 needs float32")
    rows, cols = (c, r) if trans else (r, c)
    ldh = max(64, (cols + 63) // 64 * 64)
    if out is None or out.rows != rows or out.cols != cols:
        buf = torch.empty((2, rows, ldh), dtype=torch.float16, device=x.device)
        out = SplitH2(buf[0], buf[1], torch.zeros(2, dtype=torch.int32, device=x.device),
                      rows, cols, ldh)
    if e_io is not None:
        out.e = e_io
    call("skp_split_h2_f32", ptr(x), r, c, ld, int(trans), ptr(out.hi), ptr(out.lo), out.ld,
         ptr(out.e), int(e_io is not None), stream_ptr(x.device))
    return out


def split_h2_inplace(x: torch.Tensor, e_io: torch.Tensor | None = None) -> SplitH2:
    """split_h2 of x written over x's own storage (x is consumed): planes with
    leading dimension 2 ld (see skp_split_h2_inplace_f32)."""
    r, c, ld = _rows_ld(x)
    if x.dtype != F32:
        raise ValueError("split_h2_inplace needs float32")
    have = e_io is not None
    if e_io is None:
        e_io = torch.zeros(2, dtype=torch.int32, device=x.device)
    call("skp_split_h2_inplace_f32", ptr(x), r, c, ld, ptr(e_io), int(have), stream_ptr(x.device))
    full = x.as_strided((r, ld), (ld, 1)).view(torch.float16)      # (r, 2 ld) halves
    return SplitH2(full[:, :c], full[:, ld:ld + c], e_io, r, c, 2 * ld)


def gemm_h3(a: SplitH2, b: SplitH2, ta: bool = False, alpha: float = 1.0, beta: float = 0.0,
            out=None, b_lo: bool = True) -> torch.Tensor:
    """K4h: out = alpha op(a) b^T + beta out from pre-split operands: op(a) =
    a (M x K) or a^T (a stored K x M, ta=True); b stored N x K."""
    M, K = (a.cols, a.rows) if ta else (a.rows, a.cols)
    N, Kb = b.rows, b.cols
    if K != Kb:
        raise ValueError(f"dimension mismatch: {M}x{K} @ {Kb}x{N}")
    if out is None:
        if beta != 0.0:
            raise ValueError("beta != 0 needs out")
        out = empty2d(M, N, F32, a.hi.device)
    _, _, ldc = _rows_ld(out)
    lib = _lib.load()
    wsb = lib.skp_gemm_h3_ws_bytes(int(ta), M, N, K)
    ws = workspace(a.hi.device, wsb) if wsb else None
    call("skp_gemm_h3", int(ta), M, N, K, alpha, ptr(a.hi), ptr(a.lo), a.ld, ptr(a.e), ptr(b.hi),
         ptr(b.lo) if b_lo else None, b.ld, ptr(b.e), beta, ptr(out), ldc, ptr(ws), wsb,
         stream_ptr(a.hi.device))
    return out


def gemm_h3_emit_t(a: SplitH2, b: SplitH2, ta: bool = False, shift: int | None = None,
                   e_fixed: int | None = None, out: SplitH2 | None = None, overflow=None,
                   alpha: float = 1.0, b_lo: bool = True, b_lower: bool = False) -> SplitH2:
    """K4h product written as the fp16 split of C^T (N x M planes): C =
    alpha op(a) b^T.  Exponent e_fixed, or ea + eb - shift (default shift =
    15 + ceil(log2 K): no entry can overflow).  b_lower: b (N x K) is lower
    triangular (a Cholesky inverse), so each N tile stops at its K extent."""
    M, K = (a.cols, a.rows) if ta else (a.rows, a.cols)
    N, Kb = b.rows, b.cols
    if K != Kb:
        raise ValueError(f"dimension mismatch: {M}x{K} @ {Kb}x{N}")
    if shift is None:
        shift = 15 + max(0, (K - 1).bit_length())
    ld = max(64, (M + 63) // 64 * 64)
    if out is None or out.rows != N or out.cols != M:
        buf = torch.empty((2, N, ld), dtype=torch.float16, device=a.hi.device)
        out = SplitH2(buf[0], buf[1], torch.zeros(2, dtype=torch.int32, device=a.hi.device),
                      N, M, ld)
    wsb = int(_lib.load().skp_gemm_h3_ws_bytes(int(ta), M, N, K))
    ws = workspace(a.hi.device, wsb) if wsb else None
    call("skp_gemm_h3_emit_t", int(ta), M, N, K, alpha, ptr(a.hi), ptr(a.lo), a.ld, ptr(a.e),
         ptr(b.hi), ptr(b.lo) if b_lo else None, b.ld, ptr(b.e), ptr(out.hi), ptr(out.lo), out.ld,
         int(shift),
         int(e_fixed is not None), int(e_fixed or 0), ptr(out.e), ptr(overflow), int(b_lower),
         ptr(ws), wsb, stream_ptr(a.hi.device))
    return out


def syrk_h3(a: SplitH2, alpha: float = 1.0, out=None, rows: bool = False,
            beta: float = 0.0) -> torch.Tensor:
    """K4h SYRK, exactly symmetric: alpha a^T a (+ beta out) from the planes
    of a stored K x N (a.rows = K; both operands MN-major), or with rows=True
    alpha a a^T (the Gram of a's rows, a stored N x K, both operands K-major)."""
    N, K = (a.rows, a.cols) if rows else (a.cols, a.rows)
    if out is None:
        if beta != 0.0:
            raise ValueError("beta != 0 needs out")
        out = empty2d(N, N, F32, a.hi.device)
    _, _, ldc = _rows_ld(out)
    lib = _lib.load()
    wsb = int(lib.skp_syrk_h3_ws_bytes(N, K))
    ws = workspace(a.hi.device, wsb) if wsb else None
    call("skp_syrk_h3", int(rows), N, K, alpha, ptr(a.hi), ptr(a.lo), a.ld, ptr(a.e), beta,
         ptr(out), ldc, ptr(ws), wsb, stream_ptr(a.hi.device))
    return out


def h2_exponent(x: torch.Tensor, e_io: torch.Tensor | None = None, have_amax: bool = False,
                margin_bits: int = 0) -> torch.Tensor:
    """int32[2] e_io with e_io[0] = 15 - ceil(log2 max|x|) - margin_bits (max|x|
    computed here unless have_amax: then e_io[1] holds its bits already)."""
    r, c, ld = _rows_ld(x)
    if e_io is None:
        e_io = torch.zeros(2, dtype=torch.int32, device=x.device)
    call("skp_h2_exponent_f32", ptr(x), r, c, ld, ptr(e_io), int(have_amax), int(margin_bits),
         stream_ptr(x.device))
    return e_io


def gemm_h3s_t(a: torch.Tensor, a_e: torch.Tensor, b: SplitH2, alpha: float = 1.0,
               beta: float = 0.0, out=None, overflow=None) -> torch.Tensor:
    """K4h with the in-kernel split: out = alpha a^T b_src + beta out, a
    (K x M fp32) scaled by 2^a_e[0], b pre-split (b.rows = N, b.cols = K)."""
    K, M, lda = _rows_ld(a)
    N, Kb = b.rows, b.cols
    if K != Kb:
        raise ValueError(f"dimension mismatch: {M}x{K} @ {Kb}x{N}")
    if out is None:
        if beta != 0.0:
            raise ValueError("beta != 0 needs out")
        out = empty2d(M, N, F32, a.device)
    _, _, ldc = _rows_ld(out)
    lib = _lib.load()
    wsb = lib.skp_gemm_h3s_ws_bytes(M, N, K)
    ws = workspace(a.device, wsb) if wsb else None
    call("skp_gemm_h3s", M, N, K, alpha, ptr(a), lda, ptr(a_e), ptr(b.hi), ptr(b.lo), b.ld,
         ptr(b.e), beta, ptr(out), ldc, ptr(overflow), ptr(ws), wsb, stream_ptr(a.device))
    return out


# ------------------------------------------------------------ utilities ----

def cast(x: torch.Tensor, dtype) -> torch.Tensor:
    """fp32 <-> fp64 (device kernel); 2-D results keep 16-byte rows."""
    if x.dtype == dtype:
        return x
    sfx = "f32_f64" if dtype == F64 else "f64_f32"
    if x.dim() == 2:
        r, c, ld = _rows_ld(x)
        out = empty2d(r, c, dtype, x.device)
        call(f"skp_cast2d_{sfx}", ptr(x), ld, ptr(out), out.stride(0), r, c, stream_ptr(x.device))
        return out
    x = x.contiguous()
    out = torch.empty(x.shape, dtype=dtype, device=x.device)
    call(f"skp_cast_{sfx}", ptr(x), ptr(out), x.numel(), stream_ptr(x.device))
    return out


def sumsq(x: torch.Tensor, acc=None, nonfinite=None):
    r, c, ld = _rows_ld(x)
    if acc is None:
        acc = torch.zeros(1, dtype=F64, device=x.device)
    call(f"skp_sumsq_{_SFX[x.dtype]}", ptr(x), r, c, ld, ptr(acc), ptr(nonfinite),
         stream_ptr(x.device))
    return acc


def symmetrize_(w: torch.Tensor):
    n, _, ld = _rows_ld(w)
    call(f"skp_symmetrize_{_SFX[w.dtype]}", ptr(w), n, ld, stream_ptr(w.device))
    return w


def scale_cols_(x: torch.Tensor, scale64: torch.Tensor):
    r, c, ld = _rows_ld(x)
    call(f"skp_scale_cols_{_SFX[x.dtype]}", ptr(x), r, c, ld, ptr(scale64), stream_ptr(x.device))
    return x


SIMT_MIN_K = 128          # shorter chains: the tensor core's truncation is below 1e-6
SIMT_MAX_MACS = 1 << 33   # ~1 ms of SIMT fp32


class CudaBackend:
    """Compute backend for the engine: every op is a libskp kernel launch."""

    name = "cuda"

    def __init__(self, device, dtype, gemm_mode: str = "auto"):
        self.device = device
        self.dtype = dtype
        self.gemm_mode = gemm_mode if dtype == F32 else "auto"
        self.info = torch.zeros(2, dtype=torch.int32, device=device)
        self.fail = torch.zeros(2, dtype=torch.int32, device=device)
        self._bsplit = {}
        self.overflow = torch.zeros(1, dtype=torch.int32, device=device)
        # (min, max) Cholesky pivot of the last orthonormalisation's first,
        # shifted pass: a lower bound of sigma_min(Y) / sigma_max(Y) (clipped
        # by the shift) -- the facade promotes fp32 inputs whose spectrum the
        # fp32 arithmetic cannot resolve (power._promote_range_finder)
        self.piv = torch.ones(2, dtype=F64, device=device)

    # dense products in the compute dtype
    def mm(self, a, b, ta=False, tb=False, out=None, alpha=1.0, beta=0.0):
        if isinstance(a, SplitH2):
            # pre-split left operand (prepare): 3xFP16; b split (transposed) per call
            if tb:
                raise ValueError("mm: a pre-split left operand takes a K x N right operand")
            key = tuple(b.shape)
            self._bsplit[key] = sb = split_h2(b, trans=True, out=self._bsplit.get(key))
            return gemm_h3(a, sb, ta=ta, alpha=alpha, beta=beta, out=out)
        M = a.shape[1] if ta else a.shape[0]
        K = a.shape[0] if ta else a.shape[1]
        N = b.shape[0] if tb else b.shape[1]
        return gemm(a, b, ta, tb, alpha=alpha, beta=beta, out=out, mode=self._mode_for(M, N, K))

    def _mode_for(self, M: int, N: int, K: int) -> str:
        """fp32 products below the 3xFP16 sizes: the tcgen05 3xTF32 kernel
        accumulates in the tensor core, which truncates once per MMA (measured
        r02: a K = 4000 Gram of unit columns came out 7.4e-5 low, so
        Q^T Q = (1 - 7e-5) I and sigma moved past the 1e-5 parity bar); long
        chains that small run on the SIMT kernel instead (round-to-nearest
        FMA, 2.6e-7 on the same Gram, sub-millisecond at these sizes)."""
        if (self.dtype == F32 and self.gemm_mode == "auto" and K >= SIMT_MIN_K
                and M * N * K <= SIMT_MAX_MACS):
            return "fp32"
        return self.gemm_mode

    def mm_at_big(self, a, q, amax_hint=None):
        """a^T q for the one-pass product of randsvd (a = the input, read
        once): 3xFP16 with a split in the kernel where it applies, else
        3xTF32.  amax_hint = (e_io, margin_bits): e_io[1] holds the bits of a
        value v with max|a| <= v 2^margin_bits expected (from max|A S|); a
        wrong hint is caught by the kernel's overflow flag (overflowed())."""
        K, M = a.shape
        self.overflow.zero_()
        if (self.dtype != F32 or self.gemm_mode != "auto" or a.shape[0] * a.shape[1] < H3_MIN_ELEMS
                or not _lib.load().skp_has_tcgen05()):
            return self.mm(a, self.dense(q), ta=True)
        if a.stride(1) != 1 or a.stride(0) % 32 or a.data_ptr() % 16:
            # a device operand with unaligned rows that had no room for a padded
            # copy (_convert.upload): the round-to-nearest SIMT kernel -- the
            # 3xTF32 tensor-core chain over K = rows truncates (sigma 2.3e-5
            # low at K = 65536, scripts/unaligned_probe.py)
            return gemm(a, self.dense(q), ta=True, mode="fp32")
        if amax_hint is not None:
            e_a = amax_hint[0].clone()
            h2_exponent(a, e_a, have_amax=True, margin_bits=amax_hint[1])
        else:
            e_a = h2_exponent(a)
        # q: fp32 (rows x c), or already the planes of q^T (the planes path)
        sq = q if isinstance(q, SplitH2) else split_h2(q, trans=True)
        return gemm_h3s_t(a, e_a, sq, overflow=self.overflow)

    def dense(self, q):
        """fp32 matrix of q (q itself, or Q from the planes of Q^T)."""
        return self.planes_to_compute(q) if isinstance(q, SplitH2) else q

    def overflowed(self, comm=None) -> bool:
        """Did the last mm_at_big overflow (on any rank)?  Host sync."""
        f = self.overflow.clone()
        if comm is not None:
            comm.allreduce_(f)
        return bool(f.item())

    def prepare(self, x, e_io=None, inplace: bool = False):
        """A left operand reused by several products (the power iteration's
        A~): split once into fp16 hi/lo planes for the 3xFP16 GEMM (twice the
        3xTF32 rate at 22-bit operand accuracy).  Returns x itself where that
        does not apply (fp64, explicit GEMM modes, small operands, no
        tcgen05).  e_io: see split_h2.
        inplace: the caller gives x up (the range finder's A~), so the planes
        are written over it."""
        if isinstance(x, SplitH2) or self.dtype != F32 or self.gemm_mode != "auto":
            return x
        if x.dim() != 2 or x.shape[0] * x.shape[1] < H3_MIN_ELEMS:
            return x
        if not _lib.load().skp_has_tcgen05():
            return x
        if inplace and x.stride(0) % 32 == 0 and x.data_ptr() % 16 == 0 and x.shape[1] <= 50000:
            # x is consumed: write the planes over it when a second m x l buffer
            # would not comfortably fit (C5 on one GPU); the out-of-place split
            # is ~30% faster (1.55 vs 2.15 ms at C3)
            # (free memory from the caching allocator's own counters: the
            # driver query, cudaMemGetInfo, waits for the device -- a host
            # stall here left the GPU idle for up to 19 ms per step)
            free = _device_total(x.device) - torch.cuda.memory_allocated(x.device)
            if free < 4 * x.shape[0] * x.stride(0) * 4:
                return split_h2_inplace(x, e_io)
        return split_h2(x, e_io=e_io)

    def gram64(self, y, accurate: bool = False):
        """y^T y as fp64 (computed in the compute dtype, then widened).
        accurate: the Gram that decides the final Q's orthonormality (the
        last CholeskyQR pass).  Over K = rows ~ 1e5 the tensor core's
        truncating fp32 accumulation biases a Gram's diagonal by ~1e-4
        (measured at C3: Q^T Q = (1 + 1.2e-4) I, i.e. sigma inflated by 6e-5),
        so that pass runs 3xFP16 with register-promoted accumulation."""
        if accurate and self._h3_ok(y):
            sy = split_h2(y, trans=True)            # y^T planes: (cols x rows), K-major
            return cast(gemm_h3(sy, sy), F64)
        return cast(self.mm(y, y, ta=True), F64)

    def _h3_ok(self, x) -> bool:
        return (self.dtype == F32 and self.gemm_mode == "auto" and x.dim() == 2
                and x.shape[0] * x.shape[1] >= H3_MIN_ELEMS
                and bool(_lib.load().skp_has_tcgen05()))

    def gram64_rows(self, b):
        """b b^T in fp64 arithmetic (b: c x n, widened first)."""
        bd = cast(b, F64)
        return gemm(bd, bd, False, True)

    def gram64_rows_t(self, bt):
        """(bt^T bt) in fp64 arithmetic, i.e. b b^T for b = bt^T (bt: n x c).
        fp32 bt: exact products, fp64 accumulation, no widened copy."""
        if bt.dtype == F32:
            k, c, ld = _rows_ld(bt)
            g = torch.empty((c, c), dtype=F64, device=self.device)
            wsb = int(_lib.load().skp_gram_f32_f64_ws_bytes(k, c))
            ws = workspace(self.device, wsb)
            call("skp_gram_f32_f64", ptr(bt), k, c, ld, ptr(g), c, ptr(ws), wsb,
                 stream_ptr(self.device))
            return g
        bd = cast(bt, F64)
        return gemm(bd, bd, True, False)

    def chol_inv64(self, g, rel_tol, lazy: bool = False, shift: float = 0.0):
        """L^{-1} of G + shift max_i G_ii I = L L^T (fused cooperative kernel).

        Eager: zeroes the status, then one 4-byte device->host read; returns
        None when G is not numerically full rank.  Lazy: no host sync; a failure
        is OR-ed into ``self.fail`` (checked once by the caller, see
        ``lazy_failed``) and the returned X is then meaningless."""
        n = g.shape[0]
        x = torch.empty((n, n), dtype=F64, device=self.device)
        wsb = _lib.load().skp_cholinv_ws_bytes(n)
        ws = workspace(self.device, wsb)
        st = stream_ptr(self.device)
        flag = self.fail if lazy else self.info
        if not lazy:
            self.info.zero_()
        call("skp_cholinv_f64", ptr(g), n, g.stride(0), rel_tol, shift, ptr(x), ptr(flag), ptr(ws),
             wsb, st)
        if lazy:
            return x
        if int(self.info[0].item()) != 0:
            return None
        return x

    def svd_cols(self, x):
        """Thin SVD of x (rows >= cols) by the one-sided Jacobi kernel (K8),
        fp64: (U, S, V) with x = U diag(S) V^T."""
        return gesvj(x)

    def save_pivots(self, n: int):
        """Copy the last chol_inv64's pivot range (the 2 doubles the K5 kernel
        leaves after its 4 np^2 workspace blocks, np = 32 ceil(n / 32)) into
        self.piv: a device copy, read later with the other lazy checks."""
        np_ = -(-n // 32) * 32
        off = 4 * np_ * np_ * 8
        ws = workspace(self.device, _lib.load().skp_cholinv_ws_bytes(n))
        self.piv.copy_(ws.view(torch.uint8)[off:off + 16].view(F64))

    def pivot_ratio(self) -> float:
        """min / max pivot saved by save_pivots (host sync)."""
        p = self.piv.cpu()
        return float(p[0] / p[1]) if float(p[1]) > 0 else 1.0

    def lazy_reset(self):
        self.fail.zero_()
        self.piv.fill_(1.0)

    def lazy_failed(self, comm=None) -> bool:
        """Any lazy failure (Cholesky pivot: fail[0], identical on every rank;
        an emitted fp16 split out of range: fail[1], per rank) -- all ranks
        agree (host sync)."""
        f = self.fail.clone()
        if comm is not None:
            comm.allreduce_(f)
        return bool((f != 0).any().item())

    # ---- lazy power iteration on fp16 planes (3xFP16 end to end) --------------
    def planes_ok(self, atil, omega) -> bool:
        return isinstance(atil, SplitH2) and isinstance(omega, torch.Tensor) \
            and omega.dtype == F32 and omega.dim() == 2

    def gram64_planes(self, yt: SplitH2):
        """Y^T Y (fp64) from the split planes of Y^T: the K-major SYRK (lower
        tiles only, mirrored), 3xFP16 with promoted accumulation."""
        return cast(syrk_h3(yt, rows=True), F64)

    def power_lazy_planes(self, comm, atil: SplitH2, omega, q: int, shift: float):
        """Stabilized power iteration (power.py:113-134) with every product on
        K4h and every intermediate block kept as fp16 planes of its
        TRANSPOSE, written by the producing product's epilogue:
            Y^T = (A~ Omega)^T,  q x { G = Y^T Y;  X = chol_inv(G + shift);
                                       Q^T = (Y X^T)^T (|Q| <= 1: fixed exponent 14);
                                       Z = A~^T Q;  Y^T = (A~ Z)^T }.
        The stabilisation is the shifted CholeskyQR pass alone (range kept,
        no rank test; _engine.SHIFT_REL).  Lazy: a failed factorisation or a
        Q entry out of fp16 range only sets self.fail (the caller then reruns
        eagerly in fp32).  Returns Y^T planes."""
        yt = gemm_h3_emit_t(atil, split_h2(omega, trans=True))
        qt = None
        for _ in range(q):
            x = self.chol_inv64(comm.allreduce_(self.gram64_planes(yt)), 0.0, lazy=True,
                                shift=shift)
            qt = gemm_h3_emit_t(yt, split_h2(self.to_compute(x)), ta=True, e_fixed=14, out=qt,
                                overflow=self.fail[1:], b_lower=True)
            z = comm.allreduce_(gemm_h3(atil, qt, ta=True))
            yt = gemm_h3_emit_t(atil, split_h2(z, trans=True), out=yt)
        return yt

    def gram_wanted(self, rows: int, l: int, r2: int, q: int) -> bool:
        """gram_ok's decision from the shapes alone (before A~ exists: the
        streamed upload accumulates G block by block behind the copy)."""
        return (self.dtype == F32 and self.gemm_mode == "auto" and q >= 1
                and rows * l >= H3_MIN_ELEMS and gram_pays(l, r2, q) and rows >= 2 * l
                and bool(_lib.load().skp_has_tcgen05()))

    def gram_ok(self, atil, omega, q: int) -> bool:
        """Run the power iteration in the sketch space (power_gram)?  It costs
        one SYRK (m l^2 useful MACs, tiles of the lower triangle) plus one
        product (m l r2) against the 1 + 2q products of m l r2 each and the q
        CholeskyQR passes between them (~1.5 m r2^2 each): taken when
        l <= q r2 (4.4 + 1.5 r2 / l) -- the SYRK's flops run ~10% faster than
        the products' (C5: 0.79 vs 0.72 of the pipe; the measured l x q sweep,
        profiles/r02w_c5_sweep.txt: l = 8000, q = 2 took 262 ms on the products
        against ~215 in the sketch space) -- and when the rows outnumber the
        sketch columns (the l x l work of the q steps is replicated on every
        rank)."""
        if not self.planes_ok(atil, omega) or q < 1:
            return False
        m, l, r2 = atil.rows, atil.cols, omega.shape[1]
        return gram_pays(l, r2, q) and m >= 2 * l and atil.ld % 64 == 0

    def power_gram(self, comm, atil: SplitH2, omega, q: int, shift: float, g=None):
        """The stabilized power iteration (power.py:113-134) in the sketch
        space: with Y = A~ W,
            A~ (A~^T Y) = A~ (G W),  G = A~^T A~ (l x l, summed over ranks),
            Y^T Y = W^T G W,
        so after one SYRK every step is l-dimensional:
            W = Omega;  q x { V = G W;  X = chol_inv(W^T V + shift);  W = V X^T }
        (the shifted CholeskyQR pass of power_lazy_planes, Q = Y X^T, applied
        to W), and Y = A~ W at the end -- the same block as the product path
        in exact arithmetic, with one pass over A~ for G instead of 2q.  The
        q steps are 3xFP16 products of l x l by l x r2 whose blocks stay as
        fp16 planes of their transposes.  Lazy, as power_lazy_planes: a
        failed factorisation only sets self.fail.  Returns Y^T planes.
        g: this rank's G already formed (block by block behind a streamed
        upload), else one SYRK of atil here."""
        wt = self.power_gram_steps(comm, g if g is not None else syrk_h3(atil), omega, q, shift)
        return gemm_h3_emit_t(atil, wt)                      # (A~ W)^T

    def power_gram_steps(self, comm, g, omega, q: int, shift: float) -> SplitH2:
        """power_gram's q l-dimensional steps from this rank's G (consumed):
        the planes of W^T, Y = A~ W."""
        g = comm.allreduce_(g)
        gs = split_h2(g)
        del g
        # the blocks are re-split from fp32 every step (fresh exponents): an
        # emitted split's worst-case exponent bound (ea + eb - 15 - log2 K)
        # compounds over a chain of steps and would push W into fp16's
        # subnormal range within a few steps
        wt = split_h2(omega, trans=True)                     # W^T planes (r2 x l)
        vt = None
        for _ in range(q):
            vt = split_h2(gemm_h3(gs, wt), trans=True, out=vt)   # V^T, V = G W
            mg = cast(gemm_h3(wt, vt), F64)                  # W^T G W = Y^T Y
            symmetrize_(mg)
            x = self.chol_inv64(mg, 0.0, lazy=True, shift=shift)
            wt = split_h2(gemm_h3(vt, split_h2(self.to_compute(x)), ta=True), trans=True,
                          out=wt)                            # W = V X^T
        return wt

    def orth_planes(self, comm, yt: SplitH2, t2: float, shift: float, planes_out: bool = False):
        """Lazy shifted CholeskyQR3 of Y given as Y^T planes (_engine.orthonormalize):
        pass 1 on G + shift, pass 2 with the rank test t2 on its pivots, pass 3.
        Returns Q (fp32, rows x c), or with planes_out the planes of Q^T (what
        randsvd consumes).  yt is consumed (its buffers are reused)."""
        x1 = self.chol_inv64(comm.allreduce_(self.gram64_planes(yt)), 0.0, lazy=True, shift=shift)
        self.save_pivots(yt.rows)
        q1t = gemm_h3_emit_t(yt, split_h2(self.to_compute(x1)), ta=True, e_fixed=14,
                             overflow=self.fail[1:], b_lower=True)
        x2 = self.chol_inv64(comm.allreduce_(self.gram64_planes(q1t)), t2, lazy=True)
        # (Q2 goes into Y's planes: two plane buffers in flight, not three)
        q2t = gemm_h3_emit_t(q1t, split_h2(self.to_compute(x2)), ta=True, e_fixed=14, out=yt,
                             overflow=self.fail[1:], b_lower=True)
        x3 = self.chol_inv64(comm.allreduce_(self.gram64_planes(q2t)), 0.0, lazy=True)
        if planes_out:
            return gemm_h3_emit_t(q2t, split_h2(self.to_compute(x3)), ta=True, e_fixed=14,
                                  out=q1t, overflow=self.fail[1:], b_lower=True)
        return gemm_h3(q2t, split_h2(self.to_compute(x3)), ta=True)

    def planes_to_compute(self, yt: SplitH2):
        """fp32 Y from Y^T planes (the eager fallback): Y = (Y^T)^T I."""
        eye = torch.eye(yt.rows, dtype=F32, device=self.device)
        return gemm_h3(yt, split_h2(eye), ta=True)

    def eig_desc64(self, g, max_sweeps=30):
        n = g.shape[0]
        a = g.clone()
        w = torch.empty(n, dtype=F64, device=self.device)
        v = torch.empty((n, n), dtype=F64, device=self.device)
        wsb = _lib.load().skp_syevj_ws_bytes(n)
        ws = workspace(self.device, wsb)
        call("skp_syevj_f64", ptr(a), n, ptr(w), ptr(v), max_sweeps, ptr(ws), wsb,
             ptr(self.info[1:]), stream_ptr(self.device))
        return w, v

    def eig_orth64(self, w, v, rel_tol):
        n = w.shape[0]
        t = torch.empty((n, n), dtype=F64, device=self.device)
        call("skp_eig_orth_f64", ptr(w), ptr(v), n, rel_tol, ptr(t), ptr(self.info),
             stream_ptr(self.device))
        return t, int(self.info[0].item())

    def sqrt_eigs(self, w):
        sig = torch.empty_like(w)
        inv = torch.empty_like(w)
        call("skp_sqrt_eigs_f64", ptr(w), w.shape[0], ptr(sig), ptr(inv), stream_ptr(self.device))
        return sig, inv

    def orth_dev_t(self, g64) -> torch.Tensor:
        """max |G - I| as a device scalar (no host synchronisation)."""
        out = torch.empty(1, dtype=F64, device=self.device)
        call("skp_orth_dev_f64", ptr(g64), g64.shape[0], g64.stride(0), ptr(out),
             stream_ptr(self.device))
        return out

    def proj_sq(self, gb, gq=None):
        """||A||^2 - ||A - Q Q^T A||^2 = 2 tr(BB^T) - <Q^T Q, BB^T> as a
        device scalar (tr(BB^T) alone when Q^T Q is not at hand)."""
        t = torch.diagonal(gb).sum()
        if gq is None:
            return t
        return 2.0 * t - (gq[: gb.shape[0], : gb.shape[1]] * gb).sum()

    def orth_dev(self, g64) -> float:
        return float(self.orth_dev_t(g64).item())

    def gram64_q(self, q):
        """Q^T Q (fp64) for randsvd's orthonormality check: from the planes of
        Q^T directly on the planes path, else the accurate Gram."""
        if isinstance(q, SplitH2):
            return self.gram64_planes(q)
        return self.gram64(q, accurate=True)

    def to_compute(self, x64):
        return cast(x64, self.dtype)

    def scale_cols_(self, x, s64):
        return scale_cols_(x, s64)

    def symmetrize_(self, w):
        return symmetrize_(w)

    def cols(self, x, k):
        return x[:, :k].contiguous() if k < x.shape[1] else x

    def sumsq(self, x):
        return sumsq(x)

    def scalar(self, x) -> float:
        return float(x.reshape(-1)[0].item())

    def zeros(self, shape, dtype=None):
        return torch.zeros(shape, dtype=dtype or self.dtype, device=self.device)


def np_dtype(t: torch.dtype):
    return np.float32 if t == F32 else np.float64
