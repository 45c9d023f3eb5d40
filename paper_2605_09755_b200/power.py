"""Sketched power method on the B200 (drop-in for skpower.power).

Mirrors /root/reference/pkg/src/skpower/power.py: ``RangeFinderSpec`` (:49),
``power_iterate`` (:113), ``range_finder_sketched`` (:141),
``range_finder_classical`` (:157), ``randsvd`` (:181), ``lowrank_factorize``
(:202), ``nystrom_psd`` (:258), ``choose_q`` (:34) and the result records.

Seeds follow the reference: S from substream(seed, 0) (regenerated on the
device by K1), Omega from substream(seed, 1) (host numpy, bit-identical),
S2 from substream(seed, 2).

Precision: float32 operands run the FP32 path (3xTF32 tcgen05 GEMMs, fp64
small cores); anything else runs FP64 like the reference.  Optional keyword
``timings`` (a dict) receives per-phase device times in milliseconds (CUDA
events on the launching stream).
"""
from __future__ import annotations

import math
import threading
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _convert, _engine, _ops
from ._ops import F32, F64
from .linalg import SvdResult, _pinv_dev
from .sketching import OmegaDraw, make_sketch, omega_device, omega_tensor, substream


def choose_q(eps: float, m_hat: int) -> int:
    """ceil(ln(2 m_hat) / (2 eps)) -- power.py:34-46."""
    if not 0.0 < eps <= 0.5:
        raise ValueError(f"eps must be in (0, 1/2], got {eps}")
    if m_hat < 1:
        raise ValueError(f"m_hat must be >= 1, got {m_hat}")
    return math.ceil(math.log(2.0 * m_hat) / (2.0 * eps))


@dataclass(frozen=True)
class RangeFinderSpec:
    """Parameter record of the sketched power method (power.py:49-92)."""

    k: int
    l: int
    r1: int
    r2: int
    q: int
    eps: float
    sketch_kind: str = "countsketch"
    seed: int = 0
    stabilized: bool = True
    s: int = 1
    s2_kind: str | None = None
    s2_r: int | None = None
    omega_kind: str = "gaussian"

    def validate(self, m: int, n: int) -> None:
        if not 1 <= self.k <= self.l <= min(m, n):
            raise ValueError(
                f"need 1 <= k <= l <= min(m, n); got k={self.k}, l={self.l}, "
                f"min(m, n)={min(m, n)}"
            )
        if self.r2 < self.k:
            raise ValueError(f"r2 must be >= k, got r2={self.r2}, k={self.k}")
        if self.q < 0:
            raise ValueError(f"q must be >= 0, got {self.q}")
        if not 0.0 < self.eps <= 0.5:
            raise ValueError(f"eps must be in (0, 1/2], got {self.eps}")
        if self.r1 < 1:
            raise ValueError(f"r1 must be >= 1, got {self.r1}")


@dataclass
class FactorizationResult:
    """Low-rank factors Y (m x r2) and X (r2 x n) plus stage times (power.py:95-101)."""
    Y: object
    X: object
    elapsed: dict = field(default_factory=dict)


@dataclass
class NystromResult:
    """Nystrom factors C (n x r2) and psd core W (r2 x r2) plus stage times (power.py:104-110)."""
    C: object
    W: object
    elapsed: dict = field(default_factory=dict)


class _Phases:
    """CUDA-event phase timer on the current stream (events only when
    enabled) and NVTX ranges (always: skp.<phase> in nsys / ncu --nvtx).
    mark(name, nxt) ends phase ``name`` and begins phase ``nxt``."""

    def __init__(self, enabled: bool):
        self.enabled = enabled
        self.ev = []
        self.open = False

    def begin(self, nxt: str):
        if self.open:
            torch.cuda.nvtx.range_pop()
        torch.cuda.nvtx.range_push("skp." + nxt)
        self.open = True

    def mark(self, name: str, nxt: str | None = None):
        if self.enabled:
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            self.ev.append((name, e))
        if nxt is not None:
            self.begin(nxt)
        elif self.open:
            torch.cuda.nvtx.range_pop()
            self.open = False

    def result(self, out: dict | None, scale: float = 1.0):
        if not self.enabled or out is None:
            return
        self.ev[-1][1].synchronize()
        for (_, a), (name, b) in zip(self.ev, self.ev[1:]):
            out[name] = out.get(name, 0.0) + a.elapsed_time(b) * scale


def _be(dtype, device):
    return _ops.CudaBackend(device, dtype)


def power_iterate(atil, omega, q: int, stabilized: bool = True):
    """Block with the column span of (A~ A~^T)^q A~ Omega (power.py:113-134)."""
    oa = _convert.upload(atil, "atil")
    oo = _convert.upload(omega, "omega", oa.t.device)
    if oa.t.shape[1] != oo.t.shape[0]:
        raise ValueError(f"dimension mismatch: {tuple(oa.t.shape)} vs omega {tuple(oo.t.shape)}")
    if q < 0:
        raise ValueError(f"q must be >= 0, got {q}")
    dt = _convert.common_dtype(oa, oo)
    y = _engine.power_iterate(_be(dt, oa.t.device), _engine.LOCAL, _convert.as_dtype(oa, dt),
                              _convert.as_dtype(oo, dt), q, stabilized)
    return _convert.download(y, oa.kind)


class _SideStreams(threading.local):
    """One side stream per (thread, device): concurrent callers never share."""

    def __init__(self):
        self.s = {}

    def get(self, dev) -> torch.cuda.Stream:
        if dev.index not in self.s:
            self.s[dev.index] = torch.cuda.Stream(dev)
        return self.s[dev.index]


_SIDE = _SideStreams()


def _omega_side(spec, seed, dtype, dev, fail_counter):
    """(Omega, ready event): the device Gaussian draw (numpy's ziggurat, draw
    for draw) queued on a side stream after everything already on the
    caller's stream (fail_counter's zeroing included)."""
    if spec.omega_kind != "gaussian":
        return None
    main = torch.cuda.current_stream(dev)
    side = _SIDE.get(dev)
    side.wait_stream(main)
    with torch.cuda.stream(side):
        om = omega_device("gaussian", spec.r1, spec.r2, seed, dtype, dev, None, fail_counter)
        ev = torch.cuda.Event()
        ev.record(side)
    om.record_stream(main)        # freed by the caller's stream, not the side one
    fail_counter.record_stream(side)
    return om, ev


def _range_finder_dev(a: torch.Tensor, spec: RangeFinderSpec, comm=_engine.LOCAL,
                      rows_total: int | None = None, phases: _Phases | None = None,
                      fro2: torch.Tensor | None = None, name: str = "a",
                      streamed: "_convert.Streamed | None" = None, hint_out: dict | None = None,
                      planes_out: bool = False):
    """Alg. 1 on a device row slab; returns Q (rows x <= r2).  Raises on
    non-finite entries of a (counted inside the sketch kernel).  streamed: a
    still arrives from the host block by block -- each block is sketched as
    soon as it lands, behind the copy of the next (A S is row-separable)."""
    ph = phases or _Phases(False)
    dev = a.device
    m_loc, n = a.shape
    be = _be(a.dtype, dev)
    ph.mark("start", "make_sketch")
    # Omega: the Gaussian kind is drawn on the device (omega_device, queued
    # after K2); the other kinds on a host thread while the device runs K1 + K2
    om_seed = substream(spec.seed, 1)
    om_job = None if spec.omega_kind == "gaussian" else \
        OmegaDraw(spec.omega_kind, spec.r1, spec.r2, om_seed, a.dtype)
    nonfinite = torch.zeros(1, dtype=torch.int64, device=dev)
    sk = make_sketch(spec.sketch_kind, n, spec.r1, substream(spec.seed, 0), s=spec.s, device=dev)
    # the Gaussian Omega is drawn on a side stream, concurrently with the K2
    # plan (one warp per SM; K1 before it fills the GPU) and K2's first rows;
    # only P^T waits for the plan (in line instead, alternating A/B at C3,
    # scripts/ab_omega.sh: 63.5 vs 63.1 ms per step)
    om_side = _omega_side(spec, om_seed, a.dtype, dev, nonfinite) if om_job is None else None
    if _atil_blocked(a, spec, be, sk):
        return _range_finder_blocked(a, spec, comm, rows_total, ph, fro2, name, streamed,
                                     hint_out, planes_out, be, sk, nonfinite, om_side, om_job,
                                     om_seed)
    ph.mark("make_sketch", "apply_right")
    # K2 v2 writes A~ with its columns permuted (A S P); the power iteration
    # then uses P^T Omega, so Y = (A S P)(P^T Omega) = A S Omega exactly as in
    # the reference.  K2 v1 (natural column order) where v2 does not apply.
    # (deferred: no host sync for the plan check; a failed plan shows up as a
    # marker in the non-finite count checked at the end)
    # (e_io[1]: max|A~|, accumulated by K2 v2 for the fp16 split below)
    e_io = torch.zeros(2, dtype=torch.int32, device=dev)
    if streamed is None:
        got = sk.right_permuted(a, fro2=fro2, nonfinite=nonfinite, deferred=True, amax=e_io[1:])
        if got is not None:
            atil, perm = got
        else:
            atil, perm, e_io = sk.right(a, fro2=fro2, nonfinite=nonfinite), None, None
        del got
    else:
        atil = _ops.empty2d(m_loc, spec.r1, a.dtype, dev)
        v2, perm = None, None
        # the sketch-space power iteration needs G = A~^T A~: formed here block
        # by block (each block's own fp16 split, the SYRK accumulating into G)
        # while the next blocks are still on the PCIe link
        gram = None
        if spec.stabilized and be.gram_wanted(m_loc, spec.r1, spec.r2, spec.q):
            gram = _ops.empty2d(spec.r1, spec.r1, a.dtype, dev)
        for r0, r1 in streamed.blocks():
            if v2 is not False:
                got = sk.right_permuted(a[r0:r1], out=atil[r0:r1], fro2=fro2, nonfinite=nonfinite,
                                        deferred=True, amax=e_io[1:])
                if got is None and v2:   # v2 applies by dtype/layout: all blocks or none
                    raise RuntimeError("internal: K2 v2 declined mid-stream")
                v2 = got is not None
                perm = got[1] if v2 else None
                del got
            if not v2:
                sk.right(a[r0:r1], out=atil[r0:r1], fro2=fro2, nonfinite=nonfinite)
                e_io = None
                gram = None
            if gram is not None:
                _ops.syrk_h3(_ops.split_h2(atil[r0:r1]), out=gram, beta=0.0 if r0 == 0 else 1.0)
    ph.mark("apply_right", "split")
    # the power iteration's operand: A~ split once into fp16 hi/lo planes (the
    # fp32 A~ is released here; the footprint stays m x l x 4 bytes)
    atil = be.prepare(atil, e_io, inplace=True)
    ph.mark("split", "omega")

    def omega_for(perm_dev, host: bool = False):
        if om_side is not None and not host:
            torch.cuda.current_stream(dev).wait_event(om_side[1])
            return _ops.permute_rows(om_side[0], perm_dev) if perm_dev is not None else om_side[0]
        if om_job is None and not host:
            return omega_device(spec.omega_kind, spec.r1, spec.r2, om_seed, a.dtype, dev,
                                perm_dev, nonfinite)
        job = om_job or OmegaDraw(spec.omega_kind, spec.r1, spec.r2, om_seed, a.dtype)
        return job.to_device(dev, perm_dev)

    omega = omega_for(perm)
    ph.mark("omega", "power")
    bad = comm.allreduce_(nonfinite)
    # Fast path: no host synchronisation until the end -- CholeskyQR failures
    # (numerical rank deficiency) are flagged on the device and checked once,
    # together with the non-finite count; only then is the eager,
    # rank-truncating path run.
    be.lazy_reset()
    y = _engine.power_iterate(be, comm, atil, omega, spec.q, spec.stabilized, rows_total,
                              lazy=True, gram=gram if streamed is not None else None)
    # A~ is released before the final orthonormalisation (C5 on one GPU: A
    # 128 GiB + A~ 31 GiB leave no room for Q); the rare eager rerun below
    # sketches again
    atil = None
    ph.mark("power", "orth")
    qb = _engine.orthonormalize(be, comm, y, rows_total=rows_total, lazy=True,
                                planes_out=planes_out)
    if (a.dtype == F64 and getattr(comm, "world", 1) == 1 and isinstance(y, torch.Tensor)
            and hasattr(be, "svd_cols") and y.shape[0] >= y.shape[1]
            and be.pivot_ratio() < _engine.RESOLVE["float64"]):
        # cond(Y) beyond what the shifted Gram keeps accurate (its pivots fell
        # under 1e-6 of the largest; Y = A~ A~^T Q squares A's spectrum): the
        # basis from Y's own SVD, as the reference's Householder QR would
        # resolve it (host sync: fp64 only)
        qb = _engine._svd_rank_basis(be, y, _engine.rank_floor(be, rows_total or y.shape[0],
                                                                y.shape[1]))
    del y
    ph.mark("orth")
    nbad = int(bad.item())
    omega_failed = nbad >= _ops.OMEGA_FAIL_MARK
    plan_failed = nbad % _ops.OMEGA_FAIL_MARK >= _ops.GATHER_PLAN_FAIL_MARK
    nbad %= _ops.GATHER_PLAN_FAIL_MARK
    if plan_failed:
        # K2 v2's schedule overflowed (very uneven sketch columns): K2 v1 in
        # the natural column order, with Omega unpermuted
        nonfinite.zero_()
        if fro2 is not None:
            fro2.zero_()
        atil = sk.right(a, fro2=fro2, nonfinite=nonfinite)
        nbad = int(comm.allreduce_(nonfinite).item()) % _ops.GATHER_PLAN_FAIL_MARK
        perm = None
    if nbad != 0:
        raise ValueError(f"{name} contains non-finite entries")
    if plan_failed or omega_failed:
        # (a device Omega that could not complete is redrawn by numpy itself)
        omega = omega_for(perm, host=omega_failed)
    if plan_failed or omega_failed or be.lazy_failed(comm):
        if atil is None:
            qb = None
            scratch = torch.zeros(1, dtype=torch.int64, device=dev)
            got = sk.right_permuted(a, nonfinite=scratch) if perm is not None else None
            atil = got[0] if got is not None else sk.right(a, nonfinite=scratch)
        y = _engine.power_iterate(be, comm, atil, omega, spec.q, spec.stabilized, rows_total)
        qb = _engine.orthonormalize(be, comm, y, rows_total=rows_total)
    if hint_out is not None and e_io is not None and not plan_failed:
        # for randsvd's in-kernel fp16 split of a: max|a| <~ sqrt(s) max|a S|
        # (a lone large entry lands in s outputs scaled 1/sqrt(s)); 2x slack
        hint_out["amax"] = (e_io, int(math.ceil(math.log2(2.0 * math.sqrt(spec.s or 1)))) + 1)
    if hint_out is not None and hasattr(be, "pivot_ratio"):
        hint_out["pivot_ratio"] = be.pivot_ratio() ** (1.0 / getattr(be, "y_power", 1))
    return qb


def _atil_blocked(a: torch.Tensor, spec: RangeFinderSpec, be, sk) -> bool:
    """Does A~ (rows x l fp32) fail to fit next to A?  Then the range finder
    runs blocked (_range_finder_blocked): C5 at l = 16000 on one B200 (A 128
    GiB + A~ 62.5 GiB > 178 GiB).  The estimate is the resident path's peak
    beyond A: A~ (split in place), Y^T planes and Y, the l x l Gram and its
    planes, 2 GiB of slack -- from the caching allocator's own counters (no
    device sync)."""
    if (a.dtype != F32 or sk.kind != "countsketch" or not spec.stabilized or spec.q < 1
            or not hasattr(be, "power_gram_steps") or a.stride(1) != 1
            or (a.stride(0) * 4) % 16 or a.data_ptr() % 16):
        return False
    m, ld, ldr = a.shape[0], -(-spec.r1 // 32) * 32, -(-spec.r2 // 32) * 32
    need = m * ld * 4 + 2 * m * ldr * 4 + 3 * ld * ld * 4 + (2 << 30)
    free = _ops._device_total(a.device) - torch.cuda.memory_allocated(a.device)
    return need > free


_BLOCK_BYTES = 2 << 30   # A~ row block of the blocked range finder (fp32)


def _range_finder_blocked(a, spec, comm, rows_total, ph, fro2, name, streamed, hint_out,
                          planes_out, be, sk, nonfinite, om_side, om_job, om_seed, host=None):
    """Alg. 1 when A~ does not fit beside A: the sketch-space power iteration
    with A~ formed in row blocks twice -- pass 1 sketches each block (K2 v2),
    splits it and accumulates G = A~^T A~ (SYRK, beta = 1; behind a streamed
    upload, block by block as it lands); the q steps run in the l-dimensional
    space as in the resident path; pass 2 sketches each block again and forms
    its rows of Y = A~ W.  Only an A~ block, G (l x l) and Y (rows x r2) are
    ever resident.  host (_HostBlocks): A itself does not fit either -- both
    passes stream its row blocks from host memory (out of core).  The rare
    eager fallbacks (a sketch plan or device Omega that failed, a
    rank-deficient CholeskyQR) need A~ resident and raise."""
    dev = host.dev if host is not None else a.device
    m_loc = host.m if host is not None else a.shape[0]
    l, r2 = spec.r1, spec.r2
    ld = -(-l // 32) * 32
    blk = host.rows if host is not None else int(max(1024, min(m_loc, _BLOCK_BYTES // (ld * 4))))
    e_io = torch.zeros(2, dtype=torch.int32, device=dev)
    buf = _ops.empty2d(blk, l, F32, dev)
    gram = _ops.empty2d(l, l, F32, dev)

    def ranges(src_blocks):
        for r0, r1 in src_blocks:
            for s0 in range(r0, r1, blk):
                yield s0, min(r1, s0 + blk)

    def blocks(first: bool):
        """(r0, r1, the device rows of A) for one pass."""
        if host is not None:
            yield from host.blocks()
            return
        src = streamed.blocks() if (first and streamed is not None) else [(0, m_loc)]
        for r0, r1 in ranges(src):
            yield r0, r1, a[r0:r1]

    ph.mark("make_sketch", "apply_right")
    perm, first = None, True
    for r0, r1, ab in blocks(True):
        got = sk.right_permuted(ab, out=buf[:r1 - r0], fro2=fro2, nonfinite=nonfinite,
                                deferred=True, amax=e_io[1:])
        if got is None:
            raise RuntimeError("internal: the blocked range finder needs the row gather (K2 v2)")
        perm = got[1]
        _ops.syrk_h3(_ops.split_h2(buf[:r1 - r0]), out=gram, beta=0.0 if first else 1.0)
        first = False
    ph.mark("apply_right", "omega")
    if om_side is not None:
        torch.cuda.current_stream(dev).wait_event(om_side[1])
        omega = _ops.permute_rows(om_side[0], perm)
    elif om_job is None:
        omega = omega_device(spec.omega_kind, l, r2, om_seed, F32, dev, perm, nonfinite)
    else:
        omega = om_job.to_device(dev, perm)
    ph.mark("omega", "power")
    bad = comm.allreduce_(nonfinite)
    be.lazy_reset()
    wt = be.power_gram_steps(comm, gram, omega, spec.q, _engine.SHIFT_REL[_engine._dtype_key(be)])
    del gram, omega
    y = _ops.empty2d(m_loc, r2, F32, dev)
    scratch = torch.zeros(1, dtype=torch.int64, device=dev)
    for r0, r1, ab in blocks(False):
        sk.right_permuted(ab, out=buf[:r1 - r0], nonfinite=scratch, deferred=True)
        _ops.gemm_h3(_ops.split_h2(buf[:r1 - r0]), wt, out=y[r0:r1])     # A~_b W
    del buf, wt
    yt = _ops.split_h2(y, trans=True)
    del y
    ph.mark("power", "orth")
    qb = _engine.orthonormalize(be, comm, yt, rows_total=rows_total, lazy=True,
                                planes_out=planes_out)
    del yt
    ph.mark("orth")
    nbad = int(bad.item())
    if nbad % _ops.GATHER_PLAN_FAIL_MARK:
        raise ValueError(f"{name} contains non-finite entries")
    if nbad >= _ops.GATHER_PLAN_FAIL_MARK or be.lazy_failed(comm):
        raise RuntimeError(
            "the blocked range finder (A~ does not fit beside A on this device) has no eager "
            "fallback: the sketch plan or device Omega failed, or Y is numerically rank-deficient; "
            "shard A over more GPUs so that A~ stays resident")
    if hint_out is not None:
        hint_out["amax"] = (e_io, int(math.ceil(math.log2(2.0 * math.sqrt(spec.s or 1)))) + 1)
        hint_out["pivot_ratio"] = be.pivot_ratio() ** 0.5   # (Y = A~ A~^T Q_prev: power 2)
    return qb


_OOC_BLOCK_BYTES = 2 << 30   # host row block of an out-of-core A (fp32)


class _HostBlocks:
    """Row blocks of a host fp32 matrix staged into two device buffers: the
    copy of block b + 1 runs on a side stream while the caller's stream works
    on block b (each buffer is refilled only after the work queued on it)."""

    def __init__(self, src: torch.Tensor, dev, rows: int | None = None):
        self.src, self.dev = src, dev
        self.m, n = src.shape
        per = -(-n // 32) * 32 * 4
        self.rows = int(rows or max(8, min(self.m, _OOC_BLOCK_BYTES // per) // 8 * 8))
        self.bufs = [_ops.empty2d(min(self.rows, self.m), n, F32, dev) for _ in range(2)]

    def blocks(self):
        cur = torch.cuda.current_stream(self.dev)
        side = _SIDE.get(self.dev)
        free = [None, None]   # event: the caller's work on the buffer is queued before it
        for bi, r0 in enumerate(range(0, self.m, self.rows)):
            r1 = min(self.m, r0 + self.rows)
            b = bi & 1
            if free[b] is not None:
                side.wait_event(free[b])
            else:
                side.wait_stream(cur)
            with torch.cuda.stream(side):
                self.bufs[b][:r1 - r0].copy_(self.src[r0:r1], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(side)
            cur.wait_event(ev)
            yield r0, r1, self.bufs[b][:r1 - r0]
            free[b] = torch.cuda.Event()
            free[b].record(cur)
        for buf in self.bufs:
            buf.record_stream(side)


def _host_f32(a):
    """A host 2-D float32 operand as a CPU tensor (else None)."""
    if isinstance(a, _convert.DeviceMatrix):
        return None
    if isinstance(a, torch.Tensor):
        return a if (not a.is_cuda and a.dim() == 2 and a.dtype == F32) else None
    arr = np.asarray(a) if not isinstance(a, np.ndarray) else a
    if arr.ndim != 2 or arr.dtype != np.float32 or not arr.size:
        return None
    return torch.from_numpy(np.ascontiguousarray(arr))


def _needs_out_of_core(shape, spec_r2: int, spec_l: int, dev) -> bool:
    """Does A (fp32) plus the range finder's least working set -- Y, Q and
    their planes, the l x l Gram and its planes, an A~ block -- fail to fit?"""
    m, n = shape
    ld, ldr, ldl = (-(-x // 32) * 32 for x in (n, spec_r2, spec_l))
    need = m * ld * 4 + 3 * m * ldr * 4 + 3 * ldl * ldl * 4 + (4 << 30)
    return need > _ops._device_total(dev) - torch.cuda.memory_allocated(dev)


def _range_finder_ooc(src: torch.Tensor, spec: RangeFinderSpec, dev, fro2=None,
                      hint_out: dict | None = None, planes_out: bool = False, name: str = "a",
                      rows: int | None = None):
    """Alg. 1 for a host fp32 A that does not fit on the device: the blocked
    sketch-space range finder with both passes streaming A's row blocks from
    host memory (two trips over the link); Y, Q and G stay resident."""
    if spec.sketch_kind != "countsketch" or not spec.stabilized or spec.q < 1:
        raise ValueError("unsupported: a matrix larger than the device needs the stabilised "
                         "countsketch range finder with q >= 1 (out of core)")
    m, n = src.shape
    be = _be(F32, dev)
    ph = _Phases(False)
    om_seed = substream(spec.seed, 1)
    om_job = None if spec.omega_kind == "gaussian" else \
        OmegaDraw(spec.omega_kind, spec.r1, spec.r2, om_seed, F32)
    nonfinite = torch.zeros(1, dtype=torch.int64, device=dev)
    sk = make_sketch(spec.sketch_kind, n, spec.r1, substream(spec.seed, 0), s=spec.s, device=dev)
    om_side = _omega_side(spec, om_seed, F32, dev, nonfinite) if om_job is None else None
    host = _HostBlocks(src, dev, rows)
    return _range_finder_blocked(None, spec, _engine.LOCAL, m, ph, fro2, name, None, hint_out,
                                 planes_out, be, sk, nonfinite, om_side, om_job, om_seed,
                                 host=host)


def _randsvd_ooc(src: torch.Tensor, qb, dev, stats: dict | None = None, rows: int | None = None):
    """randsvd (power.py:181-199) for a host fp32 A that does not fit:
    B^T = sum_b A_b^T Q_b over A's row blocks streamed from host memory
    (3xFP16, each block split in the kernel with its own exponent), the rest
    on the resident Q as usual; the reference's orthonormality check first."""
    be = _be(F32, dev)
    comm = _engine.LOCAL
    gq = be.gram64_q(qb)
    devn = be.orth_dev_t(gq)
    sq = qb if isinstance(qb, _ops.SplitH2) else _ops.split_h2(qb, trans=True)
    m, n = src.shape
    bt = _ops.empty2d(n, sq.rows, F32, dev)
    host = _HostBlocks(src, dev, rows)
    first = True
    for r0, r1, ab in host.blocks():
        qs = _ops.SplitH2(sq.hi[:, r0:r1], sq.lo[:, r0:r1], sq.e, sq.rows, r1 - r0, sq.ld)
        _ops.gemm_h3s_t(ab, _ops.h2_exponent(ab), qs, beta=0.0 if first else 1.0, out=bt)
        first = False
    out = _engine._randsvd_core(be, comm, bt, qb, gq, stats)
    _engine._raise_if_not_orthonormal(be, be.scalar(devn))
    return out


# fp32 operands whose spectrum the fp32 arithmetic cannot resolve are
# recomputed in fp64 -- the reference computes in fp64 for every input
# (as_matrix, linalg.py:30-39).  The fp32 path keeps sigma within 1e-5 of it
# while the returned sigma stay above ~1e-2 sigma_1 (3xFP16 products carry
# ~2^-22 ||A|| ||Q||), and its CholeskyQR resolves Y's directions down to the
# shift (~3e-3 sigma_1 after q >= 1 steps); below that the reference's
# pivoted QR still keeps columns (tests/test_gpu_sweep.py found both).
_PROMOTE_SIGMA_RATIO = 1e-2


def _fp64_fits(a: torch.Tensor) -> bool:
    """Room for an fp64 copy of a (plus the fp64 range finder's blocks)?"""
    need = 2 * a.shape[0] * (a.shape[1] + 16) * 8 + (2 << 30)
    return _ops._device_total(a.device) - torch.cuda.memory_allocated(a.device) >= need


def _promote_range_finder(a: torch.Tensor, spec: RangeFinderSpec, qb, hint: dict,
                          name: str = "a"):
    """(a64, Q64) when the fp32 range finder met a spectrum it cannot resolve
    -- its CholeskyQR truncated columns, or Y's first (shifted) pass saw pivots
    below _PROMOTE_SIGMA_RATIO of the largest -- and an fp64 copy fits, else
    None."""
    if a.dtype != F32:
        return None
    ncols = qb.rows if isinstance(qb, _ops.SplitH2) else qb.shape[1]
    wide = hint.get("pivot_ratio", 1.0) < _PROMOTE_SIGMA_RATIO
    if (ncols >= min(spec.r2, a.shape[0], a.shape[1]) and not wide) or not _fp64_fits(a):
        return None
    a64 = _ops.cast(a, F64)
    return a64, _range_finder_dev(a64, spec, name=name)


def _sigma_too_wide(s: torch.Tensor) -> bool:
    return s.numel() > 1 and float(s[-1]) < _PROMOTE_SIGMA_RATIO * float(s[0])


def range_finder_sketched(a, spec: RangeFinderSpec, *, timings: dict | None = None, device=None):
    """Orthonormal range finder from power iteration on the sketch A S (power.py:141-154)."""
    src = _host_f32(a)
    if src is not None:
        dev = _ops.require_cuda(device)
        if _needs_out_of_core(tuple(src.shape), spec.r2, spec.r1, dev):
            spec.validate(*src.shape)
            qb = _range_finder_ooc(src, spec, dev)
            return _convert.download(qb, "cpu" if isinstance(a, torch.Tensor) else "numpy")
    op, streamed = _convert.upload_streamed(a, "a", device)
    m, n = op.t.shape
    spec.validate(m, n)
    ph = _Phases(timings is not None)
    hint = {}
    qb = _range_finder_dev(op.t, spec, phases=ph, streamed=streamed, hint_out=hint)
    promoted = _promote_range_finder(op.t, spec, qb, hint)
    if promoted is not None:
        qb = promoted[1]
    if isinstance(a, _convert.DeviceMatrix):
        a.finite = True           # K2 counted every entry (none non-finite)
    ph.result(timings)
    return _convert.download(qb, op.kind)


def range_finder_classical(a, k: int, r2: int, q: int, seed: int, stabilized: bool = True):
    """Power iteration on a itself: the identity-sketch case (power.py:157-178)."""
    op = _convert.upload(a, "a", check_finite=False)
    m, n = op.t.shape
    spec = RangeFinderSpec(k=k, l=min(m, n), r1=n, r2=r2, q=q, eps=0.5, sketch_kind="identity",
                           seed=seed, stabilized=stabilized)
    spec.validate(m, n)
    return _convert.download(_range_finder_dev(op.t, spec), op.kind)


def _randsvd_dev(a: torch.Tensor, qb: torch.Tensor, comm=_engine.LOCAL, check: bool = True,
                 amax_hint=None, stats: dict | None = None):
    be = _be(a.dtype, a.device)
    return _engine.randsvd(be, comm, a, qb, check, amax_hint, stats)


def randsvd(a, q_basis, *, timings: dict | None = None) -> SvdResult:
    """U diag(sigma) V^T == Q Q^T a (power.py:181-199)."""
    src = _host_f32(a)
    if src is not None:
        dev = _ops.require_cuda(None)
        oq0 = np.asarray(q_basis) if not isinstance(q_basis, torch.Tensor) else q_basis
        r2 = int(oq0.shape[1]) if getattr(oq0, "ndim", 2) == 2 else 1
        if _needs_out_of_core(tuple(src.shape), r2, r2, dev):
            oq = _convert.upload(q_basis, "q_basis", dev, dtype=F32)
            if oq.t.shape[0] != src.shape[0]:
                raise ValueError(f"dimension mismatch: Q has {oq.t.shape[0]} rows, "
                                 f"a has {src.shape[0]}")
            u, s, v = _randsvd_ooc(src, oq.t, dev)
            kind = "cpu" if isinstance(a, torch.Tensor) else "numpy"
            return SvdResult(_convert.download(u, kind), _convert.download(s, kind),
                             _convert.download(v, kind))
    oa = _convert.upload(a, "a")
    oq = _convert.upload(q_basis, "q_basis", oa.t.device)
    if oq.t.shape[0] != oa.t.shape[0]:
        raise ValueError(f"dimension mismatch: Q has {oq.t.shape[0]} rows, a has {oa.t.shape[0]}")
    dt = _convert.common_dtype(oa, oq)
    if dt == F64 and oa.t.dtype == F32 and not _fp64_fits(oa.t):
        # an fp64 Q (e.g. a promoted range finder's) with an fp32 A too large
        # for an fp64 copy: the fp32 product on Q rounded to fp32
        dt = F32
    ph = _Phases(timings is not None)
    ph.mark("start", "randsvd")
    at = _convert.as_dtype(oa, dt)
    qt = _convert.as_dtype(oq, dt)
    u, s, v = _randsvd_dev(at, qt)
    if dt == F32 and _sigma_too_wide(s) and _fp64_fits(at):
        # (Q passed the fp32 run's orthonormality check, at the fp32 tolerance)
        u, s, v = _randsvd_dev(_ops.cast(at, F64), _ops.cast(qt, F64), check=False)
    ph.mark("randsvd")
    ph.result(timings)
    return SvdResult(_convert.download(u, oa.kind), _convert.download(s, oa.kind),
                     _convert.download(v, oa.kind))


def rsvd(a, spec: RangeFinderSpec, *, timings: dict | None = None, with_error: bool = False):
    """range_finder_sketched + randsvd with ONE upload of ``a`` (convenience
    entry, not in the reference: the two reference calls each re-read a).

    Returns SvdResult, or (SvdResult, rel_err) with ``with_error`` where
    rel_err = ||a - QQ^T a||_F / ||a||_F from ||a||_F^2 - sum(sigma^2)
    (Pythagorean identity, in the form that holds for any Q:
    _engine.randsvd's stats; ||a||_F^2 is fused into the sketch)."""
    src = _host_f32(a)
    if src is not None:
        dev = _ops.require_cuda(None)
        if _needs_out_of_core(tuple(src.shape), spec.r2, spec.r1, dev):
            return _rsvd_ooc(src, spec, dev, with_error,
                             "cpu" if isinstance(a, torch.Tensor) else "numpy")
    op, streamed = _convert.upload_streamed(a, "a")
    m, n = op.t.shape
    spec.validate(m, n)
    ph = _Phases(timings is not None)
    fro2 = torch.zeros(1, dtype=torch.float64, device=op.t.device) if with_error else None
    hint = {}
    qb = _range_finder_dev(op.t, spec, phases=ph, fro2=fro2, streamed=streamed, hint_out=hint,
                           planes_out=True)
    if isinstance(a, _convert.DeviceMatrix):
        a.finite = True
    a_rs = op.t
    promoted = _promote_range_finder(op.t, spec, qb, hint)
    if promoted is not None:
        a_rs, qb = promoted
        hint = {}
    st = {}
    ph.begin("randsvd")
    u, s, v = _randsvd_dev(a_rs, qb, check=True, amax_hint=hint.get("amax"), stats=st)
    if a_rs.dtype == F32 and _sigma_too_wide(s) and _fp64_fits(a_rs):
        q32 = _ops.CudaBackend(a_rs.device, F32).dense(qb)
        a_rs = _ops.cast(a_rs, F64)
        u, s, v = _randsvd_dev(a_rs, _ops.cast(q32, F64), check=False, stats=st)
    ph.mark("randsvd")
    res = SvdResult(_convert.download(u, op.kind), _convert.download(s, op.kind),
                    _convert.download(v, op.kind))
    ph.result(timings)
    if not with_error:
        return res
    a2 = float(fro2.item())
    rel = math.sqrt(max(a2 - float(st["qa2"]), 0.0) / a2) if a2 > 0 else 0.0
    return res, rel


def _rsvd_ooc(src: torch.Tensor, spec: RangeFinderSpec, dev, with_error: bool, kind: str):
    """rsvd for a host fp32 A larger than the device: three trips of A's row
    blocks over the link (G, then Y = A~ W, then B^T = A^T Q)."""
    m, n = src.shape
    spec.validate(m, n)
    fro2 = torch.zeros(1, dtype=torch.float64, device=dev) if with_error else None
    qb = _range_finder_ooc(src, spec, dev, fro2=fro2, planes_out=True)
    st = {}
    u, s, v = _randsvd_ooc(src, qb, dev, stats=st)
    res = SvdResult(_convert.download(u, kind), _convert.download(s, kind),
                    _convert.download(v, kind))
    if not with_error:
        return res
    a2 = float(fro2.item())
    return res, (math.sqrt(max(a2 - float(st["qa2"]), 0.0) / a2) if a2 > 0 else 0.0)


def lowrank_factorize(a, spec: RangeFinderSpec) -> FactorizationResult:
    """Generalized Nystrom a ~= Y X with X = (S2^T Y)^+ (S2^T a) (power.py:202-239)."""
    op = _convert.upload(a, "a", check_finite=False)
    t = op.t
    m, n = t.shape
    spec.validate(m, n)
    s2_kind = spec.s2_kind or spec.sketch_kind
    s2_r = spec.s2_r or spec.r1
    dev = t.device
    be = _be(t.dtype, dev)
    ph = _Phases(True)
    ph.mark("t0", "sketch")
    s1 = make_sketch(spec.sketch_kind, n, spec.r1, substream(spec.seed, 0), s=spec.s, device=dev)
    nonfinite = torch.zeros(1, dtype=torch.int64, device=dev)
    atil = s1.right(t, nonfinite=nonfinite)
    ph.mark("sketch", "power")
    if int(nonfinite.item()):
        raise ValueError("a contains non-finite entries")
    omega = omega_tensor(spec.omega_kind, spec.r1, spec.r2, substream(spec.seed, 1), t.dtype, dev)
    y = _engine.power_iterate(be, _engine.LOCAL, atil, omega, spec.q, spec.stabilized)
    ph.mark("power", "regression")
    s2 = make_sketch(s2_kind, m, s2_r, substream(spec.seed, 2), s=spec.s, device=dev)
    s2y = s2.left_t(y)
    if float(_ops.sumsq(s2y).item()) == 0.0:
        raise ValueError("S2.T Y is numerically rank-zero; regression is undefined")
    x = be.mm(_pinv_dev(be, s2y), s2.left_t(t))
    ph.mark("regression")
    el = {}
    ph.result(el, 1e-3)
    return FactorizationResult(Y=_convert.download(y, op.kind), X=_convert.download(x, op.kind),
                               elapsed=el)


# psd checks (power.py:242-255).  The symmetry test runs on the device at any
# size; the O(n^3) eigenvalue test only up to PSD_EIG_MAX (documented gap).
PSD_EIG_MAX = 1024


def _check_psd_dev(t: torch.Tensor, tol: float = 1e-8) -> None:
    n = t.shape[0]
    if t.shape[0] != t.shape[1]:
        raise ValueError(f"psd input must be square, got {tuple(t.shape)}")
    asym, scale = _ops.sym_check(t).tolist()      # one tiled pass over t, one sync
    if scale == 0.0:
        return
    if asym > tol * scale:
        raise ValueError("matrix is not symmetric within tolerance")
    if n <= PSD_EIG_MAX:
        be = _be(F64, t.device)
        g = _ops.cast(t, F64).clone()
        _ops.symmetrize_(g)
        w, _ = be.eig_desc64(g)
        lo, hi = float(w[-1].item()), float(w.abs().max().item())
        if hi > 0.0 and lo < -tol * hi:
            raise ValueError(f"matrix is not psd: min eigenvalue {lo:.3e} < {-tol * hi:.3e}")


def _nystrom_dev(t: torch.Tensor, spec: RangeFinderSpec, comm=_engine.LOCAL, row0: int = 0,
                 n_total: int | None = None, stabilized: bool | None = None,
                 phases: _Phases | None = None):
    """Alg. 3 on a row slab t = K[row0:row0+rows, :] (power.py:272-287).

    The sketch C~ = K S runs in the input's precision (K2); everything after
    it -- W~ = S^T C~, the power on W~, C = C~ Y and W = Y^T W~ Y -- runs in
    fp64, as in the reference (as_matrix casts to float64): the core W is
    ill-conditioned (C4: the Nystrom error came out 4x the reference's with
    an fp32 core), and C, W are returned as float64 like the reference's.
    FP64 follows the reference literally (Y = W~^q Omega) unless
    ``stabilized`` asks for the orthonormalised power (same span)."""
    ph = phases or _Phases(False)
    dev = t.device
    n = t.shape[1] if n_total is None else n_total
    be = _be(F64, dev)
    if stabilized is None:
        stabilized = False
    ph.mark("t0", "sketch")
    sk = make_sketch(spec.sketch_kind, n, spec.r1, substream(spec.seed, 0), s=spec.s, device=dev)
    nonfinite = torch.zeros(1, dtype=torch.int64, device=dev)
    # K2 v2 (row gather) writes C~ P -- columns permuted by the plan; the
    # whole core then runs in permuted sketch coordinates: W~_P = P^T W~ P
    # (rows of S^T C~ P permuted), Omega_P = P^T Omega, so C = (C~ P)(P^T Y)
    # and W = Y^T W~ Y are the reference's (power.py:276-287).  K2 v1
    # (natural order) where v2 does not apply or its plan fails.
    # (fp32 K: the gather accumulates in fp64 and writes C~ in fp64 -- the
    # literal core amplifies the rounding of an fp32 sketch)
    got = sk.right_permuted(t, nonfinite=nonfinite, deferred=True, out_dtype=F64)
    ctil, perm = got if got is not None else (None, None)
    bad = int(comm.allreduce_(nonfinite).item())
    if bad >= _ops.GATHER_PLAN_FAIL_MARK:
        nonfinite.zero_()
        ctil, perm = None, None
    if ctil is None:
        ctil = sk.right(t, nonfinite=nonfinite)
        bad = int(comm.allreduce_(nonfinite).item())
    if bad % _ops.GATHER_PLAN_FAIL_MARK:
        raise ValueError("a contains non-finite entries")
    ctil = _ops.cast(ctil, F64)          # exact widening; the core is fp64
    rows = t.shape[0]
    if rows == n:
        wtil = sk.left_t(ctil)
    else:  # S rows of this shard: W~ = sum_p S[I_p]^T C~_p
        shard = _shard_sketch(sk, row0, rows)
        wtil = shard.left_t(ctil)
    wtil = comm.allreduce_(wtil)
    if perm is not None:
        wtil = _ops.permute_rows(wtil, perm)
    be.symmetrize_(wtil)
    ph.mark("sketch", "contract")
    omega = omega_tensor(spec.omega_kind, spec.r1, spec.r2, substream(spec.seed, 1), F64, dev)
    if perm is not None:
        omega = _ops.permute_rows(omega, perm)
    cmat, w = _engine.nystrom(be, comm, ctil, wtil, omega, spec.q, stabilized)
    ph.mark("contract")
    return cmat, w


class _ShardSketch:
    """Rows [row0, row0+rows) of a countsketch / dense sketch, for S[I_p]^T X."""

    def __init__(self, sk, row0, rows):
        self.sk, self.row0, self.rows = sk, row0, rows
        if sk.kind == "countsketch":
            c = sk.d_cols[row0:row0 + rows].contiguous()
            g = sk.d_signs[row0:row0 + rows].contiguous()
            self.colptr, self.entries = _ops.csc(c, g, rows, sk.s, sk.r)

    def left_t(self, x):
        sk = self.sk
        if sk.kind == "countsketch":
            return _ops.sketch_left_t(x, self.colptr, self.entries, sk.s, sk.r)
        if sk.kind == "identity":
            out = torch.zeros((sk.n, x.shape[1]), dtype=x.dtype, device=x.device)
            out[self.row0:self.row0 + self.rows] = x
            return out
        d = sk._dense(x.dtype)[self.row0:self.row0 + self.rows].contiguous()
        return _ops.gemm(d, x, ta=True)


def _shard_sketch(sk, row0, rows):
    return _ShardSketch(sk, row0, rows)


def nystrom_psd(a, spec: RangeFinderSpec, *, stabilized: bool | None = None) -> NystromResult:
    """Psd Nystrom a ~= C pinv(W) C^T (power.py:258-298).

    The sketch C~ = a S runs in a's precision (fp32: K2 v2); the core after
    it in fp64, literally as the reference (Y = W~^q Omega; ``stabilized=True``
    orthonormalises between the W~ products instead -- same span).
    C and W are float64, as the reference returns them."""
    op = _convert.upload(a, "a", check_finite=False)
    t = op.t
    n = t.shape[0]
    if t.shape[0] != t.shape[1]:
        raise ValueError(f"psd Nystrom needs a square matrix, got {tuple(t.shape)}")
    _convert.ensure_finite(op)
    _check_psd_dev(t)
    spec.validate(n, n)
    ph = _Phases(True)
    cmat, w = _nystrom_dev(t, spec, stabilized=stabilized, phases=ph)
    el = {}
    ph.mark("end")
    ph.result(el, 1e-3)
    el.pop("end", None)
    el["power"] = 0.0
    return NystromResult(C=_convert.download(cmat, op.kind), W=_convert.download(w, op.kind),
                         elapsed=el)
