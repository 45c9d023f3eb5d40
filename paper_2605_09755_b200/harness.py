"""Error-versus-time harness on the B200 (reference bench.py, data_io.py:263-320).

SURVEY.md §8(f) row 2: the reference's benchmark protocol -- every method x
sketch size l x trial, the power iteration advanced one step at a time up to
q_max with a TrialRecord after each iterate -- run on the device, with
``time_ms`` the cumulative CUDA-event time of the work the iteration performs
(reference bench.py:7-18 for what is timed):

* q = 0: sketch construction, the sketched product, the start-block draw and
  the first product (sketched / classical randSVD, low-rank factorisation),
  or C~ = A S, W~ = S^T C~ and the start block (Nystrom);
* each q: one power-iteration pair (and the stabilisation QR when enabled).

The per-point factorisation assembly and the error evaluation are untimed,
as in the reference.  Errors follow skpower.diagnostics: the spectral residual
is estimated by seeded block power iteration (relative tolerance 1e-6, start
block drawn by numpy exactly as the reference draws it), the Frobenius
residual is exact (formed in row blocks), and rel_err = spec / sigma_(k+1) - 1
against the dataset's singular-value profile (computed once, untimed: the
eigenvalues of the fp64 Gram matrix on the device).

Same seeds as the reference (substream(root_seed, method, l, trial), start
blocks substream(seed, 1), error starts substream(seed, 100, q)); same CSV
schema (write_records_csv / read_records_csv).  Arithmetic follows the data:
float64 data runs the fp64 kernels (errors reproduce the reference's to the
estimator's tolerance), float32 data the fp32 tensor-core path.
"""
from __future__ import annotations

import argparse
import csv
from dataclasses import dataclass, field, fields

import numpy as np
import torch

from . import _engine, _ops, datagen
from ._ops import F32, F64
from .linalg import _pinv_dev
from .sketching import make_sketch, omega_device, substream

METHODS = (
    "classical-randsvd",
    "sketched-randsvd",
    "lowrank-factorize",
    "lowrank-factorize-unsketched",
    "nystrom",
)
_CLASSICAL = {"classical-randsvd", "lowrank-factorize-unsketched"}
DEFAULT_QMAX_SKETCHED = 15
DEFAULT_QMAX_CLASSICAL = 5
_ERR_STREAM = 100  # substream tag of the residual estimator's start block


# ------------------------------------------------------------- records ----

@dataclass
class TrialRecord:
    """One benchmark row (reference data_io.py:263-287); ``time_ms`` is the
    cumulative algorithm time up to this iterate (non-decreasing in q_iter)."""

    method: str
    dataset: str
    m: int
    n: int
    k: int
    l: int
    r1: int
    r2: int
    s: int
    q_iter: int
    eps: float
    seed: int
    trial: int
    time_ms: float
    spec_err: float
    frob_err: float
    rel_err: float


RECORD_FIELDS = [f.name for f in fields(TrialRecord)]
_INT_FIELDS = {"m", "n", "k", "l", "r1", "r2", "s", "q_iter", "seed", "trial"}


def _format_record(rec: TrialRecord) -> list[str]:
    row = []
    for name in RECORD_FIELDS:
        value = getattr(rec, name)
        if name in ("method", "dataset"):
            row.append(str(value))
        elif name in _INT_FIELDS:
            row.append(str(int(value)))
        else:
            row.append(repr(float(value)))
    return row


def write_records_csv(records, path) -> None:
    """Canonical column order, lossless floats (reference data_io.py:296-304)."""
    with open(path, "w", newline="", encoding="ascii") as fh:
        writer = csv.writer(fh)
        writer.writerow(RECORD_FIELDS)
        for rec in records:
            writer.writerow(_format_record(rec))


def read_records_csv(path) -> list[TrialRecord]:
    """Read records; validates the header and time_ms monotonicity per series."""
    with open(path, "r", newline="", encoding="ascii") as fh:
        rows = list(csv.reader(fh))
    if not rows or rows[0] != RECORD_FIELDS:
        raise ValueError(f"{path}: unexpected header {rows[0] if rows else None}")
    out, last = [], {}
    for row in rows[1:]:
        kw = {}
        for name, val in zip(RECORD_FIELDS, row):
            kw[name] = val if name in ("method", "dataset") else (
                int(val) if name in _INT_FIELDS else float(val))
        rec = TrialRecord(**kw)
        key = (rec.method, rec.dataset, rec.l, rec.seed, rec.trial)
        if key in last and rec.time_ms < last[key]:
            raise ValueError(f"{path}: time_ms decreases within a series")
        last[key] = rec.time_ms
        out.append(rec)
    return out


# ------------------------------------------------------------- datasets ----

def _rotate_spectrum(m: int, n: int, spectrum: np.ndarray, seed: int) -> np.ndarray:
    return datagen.rotate_spectrum(m, n, spectrum, seed)


_RECIPES = ("polydecay", "expdecay", "lowrank")


def _leading_digits(s: str, i: int) -> int:
    """End of the run of decimal digits starting at s[i]."""
    while i < len(s) and s[i].isdecimal():
        i += 1
    return i


def _recipe(text: str):
    """(name, m, n, options) of a synthetic dataset spec, or None.

    Grammar (the reference's pattern, bench.py:88-107): NAME ":" DIGITS "x"
    DIGITS REST, where REST is ``:key=value`` fields and holds no newline
    (one trailing newline on the whole text is tolerated)."""
    body = text[:-1] if text.endswith("\n") else text
    name, colon, tail = body.partition(":")
    if not colon or name not in _RECIPES or "\n" in tail:
        return None
    i = _leading_digits(tail, 0)
    if i == 0 or tail[i:i + 1] != "x":
        return None
    j = _leading_digits(tail, i + 1)
    if j == i + 1:
        return None
    fields = (f.partition("=") for f in tail[j:].split(":") if f)
    return name, int(tail[:i]), int(tail[i + 1:j]), {k: v for k, _, v in fields}


def synthetic(text: str) -> np.ndarray | None:
    """The reference's synthetic recipes (bench.py:88-107, data_io.py:49-81):
    ``polydecay:MxN:seed=S``, ``expdecay:MxN:rate=R:seed=S``,
    ``lowrank:MxN:rank=R:noise=E:seed=S``; None for anything else."""
    parsed = _recipe(text)
    if parsed is None:
        return None
    name, m, n, opts = parsed
    seed = int(opts.get("seed", 0))
    p = min(m, n)
    if name == "polydecay":
        return _rotate_spectrum(m, n, max(m, n) / np.arange(1.0, p + 1.0), seed)
    if name == "expdecay":
        return _rotate_spectrum(m, n, np.exp(-float(opts.get("rate", 0.1)) * np.arange(p, dtype=np.float64)), seed)
    r, noise = int(opts.get("rank", 10)), float(opts.get("noise", 0.0))
    if not 1 <= r <= p:
        raise ValueError(f"need 1 <= r <= min(m, n), got r={r}")
    base = _rotate_spectrum(m, n, np.ones(r), seed)
    if noise > 0.0:
        rng = np.random.default_rng(np.random.SeedSequence(entropy=[substream(seed, 2)]))
        base = base + noise * rng.standard_normal((m, n))
    return base


@dataclass
class BenchConfig:
    """Everything one run needs (reference bench.py:115-154)."""

    dataset: str
    methods: list[str]
    k: int
    l_values: list[int]
    label: str | None = None
    eps: float = 0.5
    q_max: int | None = None  # None: 15 for sketched methods, 5 for classical
    trials: int = 20
    root_seed: int = 0
    sketch_kind: str = "countsketch"
    s: int = 1
    stabilized: bool = True
    dtype: str = "float64"
    extra: dict = field(default_factory=dict)

    def validate(self) -> None:
        if self.trials < 1:
            raise ValueError("trials must be >= 1")
        if self.q_max is not None and self.q_max < 0:
            raise ValueError("q_max must be >= 0")
        if not self.methods:
            raise ValueError("at least one method required")
        for method in self.methods:
            if method not in METHODS:
                raise ValueError(f"unknown method {method!r}; expected one of {METHODS}")
        for l in self.l_values:
            if l < self.k:
                raise ValueError(f"every l must be >= k, got l={l} < k={self.k}")
        if self.dtype not in ("float64", "float32"):
            raise ValueError("dtype must be float64 or float32")

    def q_max_for(self, method: str) -> int:
        if self.q_max is not None:
            return self.q_max
        return DEFAULT_QMAX_CLASSICAL if method in _CLASSICAL else DEFAULT_QMAX_SKETCHED


# ---------------------------------------------------------- error terms ----

class _Errors:
    """skpower.diagnostics on the device (diagnostics.py:169-231)."""

    def __init__(self, be, a: torch.Tensor):
        self.be, self.a = be, a

    def _sigma_max(self, u: torch.Tensor) -> float:
        g = self.be.gram64(u)
        w, _ = self.be.eig_desc64(g)
        return float(np.sqrt(max(float(w[0].item()), 0.0)))

    def spectral_norm(self, apply, apply_t, n: int, tol: float = 1e-6, block: int = 8,
                      max_iter: int = 1000, seed: int = 0) -> float:
        """Seeded block power iteration on R^T R (diagnostics.py:169-194): the
        start block is numpy's draw, so the iterates follow the reference's."""
        be = self.be
        block = min(block, n, self.a.shape[0])
        rng = np.random.default_rng(np.random.SeedSequence([int(seed) & ((1 << 64) - 1)]))
        v0 = rng.standard_normal((n, block)).astype(np.float64)
        v = _orth(be, torch.from_numpy(v0).to(self.a.device, self.a.dtype))
        estimate = 0.0
        for _ in range(max_iter):
            u = apply(v)
            s = self._sigma_max(u)
            if s == 0.0:
                return 0.0
            v = _orth(be, apply_t(u))
            if abs(s - estimate) <= tol * s:
                return s
            estimate = s
        return float(estimate)

    def frobenius(self, resid_rows) -> float:
        """||R||_F with R formed in row blocks (exact, no cancellation)."""
        acc = torch.zeros(1, dtype=F64, device=self.a.device)
        for blk in resid_rows():
            _ops.sumsq(blk, acc)
        return float(np.sqrt(acc.item()))


def _orth(be, y):
    return _engine.orthonormalize(be, _engine.LOCAL, _ops.aligned2d(y))


def _rows(m: int, step: int = 8192):
    for r0 in range(0, m, step):
        yield r0, min(m, r0 + step)


class _Runner:
    """One (method, l, seed) series, advanced one iterate at a time
    (reference bench.py:219-290)."""

    def __init__(self, a, be, *, method, k, l, sketch_kind, s, seed, stabilized):
        self.a, self.be, self.method, self.k, self.l = a, be, method, k, l
        self.stabilized, self.seed = stabilized, seed
        m, n = a.shape
        dt, dev = a.dtype, a.device
        self.q_done = 0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if method == "nystrom":
            self.sketch = make_sketch(sketch_kind, n, l, substream(seed, 0), s=s, device=dev)
            self.ctil = self.sketch.right(a)
            w = self.sketch.left_t(_ops.aligned2d(self.ctil))
            be.symmetrize_(w)
            self.wtil = w
            self.y = omega_device("gaussian", l, k, substream(seed, 1), dt, dev)
            self.r1 = l
        elif method in _CLASSICAL:
            self.atil = a
            self.y = be.mm(a, omega_device("gaussian", n, k, substream(seed, 1), dt, dev))
            self.r1 = n
        else:
            self.sketch = make_sketch(sketch_kind, n, l, substream(seed, 0), s=s, device=dev)
            self.atil = self.sketch.right(a)
            self.y = be.mm(self.atil, omega_device("gaussian", l, k, substream(seed, 1), dt, dev))
            self.r1 = l
        e1.record()
        e1.synchronize()
        self.cumulative = e0.elapsed_time(e1)
        if method in ("lowrank-factorize", "lowrank-factorize-unsketched"):
            # regression-stage inputs; untimed (identical across methods)
            self.s2 = make_sketch(sketch_kind, m, l, substream(seed, 2), s=s, device=dev)
            self.s2a = self.s2.left_t(a)

    def advance(self) -> None:
        be = self.be
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if self.method == "nystrom":
            self.y = be.mm(self.wtil, self.y)
        else:
            y = _orth(be, self.y) if self.stabilized else self.y
            self.y = be.mm(self.atil, be.mm(self.atil, y, ta=True))
        e1.record()
        e1.synchronize()
        self.cumulative += e0.elapsed_time(e1)
        self.q_done += 1

    def errors(self, sigma_k1: float) -> tuple[float, float, float]:
        be, a = self.be, self.a
        m, n = a.shape
        err = _Errors(be, a)
        err_seed = substream(self.seed, _ERR_STREAM, self.q_done)
        if self.method in ("classical-randsvd", "sketched-randsvd"):
            q = _orth(be, self.y)
            qta = be.mm(q, a, ta=True)                        # c x n
            left, right = q, qta                             # Q (Q^T A)
        else:
            if self.method == "nystrom":
                c = be.mm(self.ctil, self.y)
                w = be.mm(self.y, be.mm(self.wtil, self.y), ta=True)
                be.symmetrize_(w)
                left, right = c, be.mm(_pinv_dev(be, w), c, tb=True)     # C W^+ C^T
            else:
                s2y = self.s2.left_t(_ops.aligned2d(self.y))
                left, right = self.y, be.mm(_pinv_dev(be, s2y), self.s2a)  # Y X

        # R = A - left right, applied as an operator (libskp GEMMs with beta)
        def apply(v):
            out = be.mm(a, v)
            return be.mm(left, be.mm(right, v), out=out, alpha=-1.0, beta=1.0)

        def apply_t(u):
            out = be.mm(a, u, ta=True)
            return be.mm(right, be.mm(left, u, ta=True), ta=True, out=out, alpha=-1.0, beta=1.0)

        def resid_rows():
            for r0, r1 in _rows(m):
                blk = _ops.empty2d(r1 - r0, n, a.dtype, a.device)
                blk.copy_(a[r0:r1])
                yield be.mm(_ops.aligned2d(left[r0:r1]), right, out=blk, alpha=-1.0, beta=1.0)
        spec = err.spectral_norm(apply, apply_t, n, seed=err_seed)
        frob = err.frobenius(resid_rows)
        return spec, frob, spec / sigma_k1 - 1.0


def singular_values(a: torch.Tensor, be) -> np.ndarray:
    """Descending singular values from the fp64 Gram of the short side (untimed)."""
    m, n = a.shape
    a64 = _ops.cast(a, F64) if a.dtype != F64 else a
    bd = _ops.CudaBackend(a.device, F64)
    g = bd.gram64(a64) if m >= n else bd.gram64_rows(a64)
    w, _ = bd.eig_desc64(g)
    return np.sqrt(np.clip(w.cpu().numpy(), 0.0, None))


def run_series(a, sigma, cfg: BenchConfig, method: str, l: int, trial: int, seed: int,
               label: str, be) -> list[TrialRecord]:
    runner = _Runner(a, be, method=method, k=cfg.k, l=l, sketch_kind=cfg.sketch_kind, s=cfg.s,
                     seed=seed, stabilized=cfg.stabilized)
    rows = []
    for q in range(cfg.q_max_for(method) + 1):
        if q > 0:
            runner.advance()
        spec, frob, rel = runner.errors(float(sigma[cfg.k]))
        rows.append(TrialRecord(
            method=method, dataset=label, m=a.shape[0], n=a.shape[1], k=cfg.k, l=l,
            r1=runner.r1, r2=cfg.k,
            s=cfg.s if method != "classical-randsvd" and cfg.sketch_kind == "countsketch" else 0,
            q_iter=q, eps=cfg.eps, seed=seed, trial=trial, time_ms=runner.cumulative,
            spec_err=spec, frob_err=frob, rel_err=rel))
    return rows


def run_benchmark(cfg: BenchConfig, csv_path: str | None = None, a=None,
                  progress=None) -> list[TrialRecord]:
    """The configured benchmark on the device (reference bench.py:333-384);
    rows stream to ``csv_path`` when given.  ``a`` overrides the dataset
    recipe (a numpy array or CUDA tensor)."""
    cfg.validate()
    if a is None:
        a = synthetic(cfg.dataset)
        if a is None:
            # files go straight to the device (io.py: .skpw streamed, MatrixMarket parsed)
            from . import io as skio
            a = (skio.read_skpw(cfg.dataset) if cfg.dataset.endswith(".skpw")
                 else skio.read_matrix_market(cfg.dataset))
    label = cfg.label or cfg.dataset
    dt = F64 if cfg.dtype == "float64" else F32
    dev = _ops.require_cuda()
    t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a))
    at = _ops.empty2d(t.shape[0], t.shape[1], dt, dev)
    at.copy_(t.to(dev, dt))
    be = _ops.CudaBackend(dev, dt)
    if "nystrom" in cfg.methods:
        from .power import _check_psd_dev
        _check_psd_dev(at)
    sigma = singular_values(at, be)
    if sigma[cfg.k] <= 0.0:
        raise ValueError(f"sigma_(k+1) vanishes for k={cfg.k}; relative error undefined")
    records: list[TrialRecord] = []
    fh = open(csv_path, "w", newline="", encoding="ascii") if csv_path else None
    try:
        writer = csv.writer(fh) if fh else None
        if writer:
            writer.writerow(RECORD_FIELDS)
        for mi, method in enumerate(cfg.methods):
            for li, l in enumerate(cfg.l_values):
                for trial in range(cfg.trials):
                    seed = substream(cfg.root_seed, mi, li, trial)
                    rows = run_series(at, sigma, cfg, method, l, trial, seed, label, be)
                    if writer:
                        for rec in rows:
                            writer.writerow(_format_record(rec))
                        fh.flush()
                    records.extend(rows)
                    if progress is not None:
                        progress(rows[-1])
    finally:
        if fh:
            fh.close()
    return records


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description="error-versus-time curves on the B200")
    ap.add_argument("--dataset", required=True, help="synthetic recipe, e.g. polydecay:2000x1000:seed=7")
    ap.add_argument("--methods", default="sketched-randsvd,classical-randsvd")
    ap.add_argument("--k", type=int, default=40)
    ap.add_argument("--l-values", required=True, help="comma-separated sketch sizes")
    ap.add_argument("--trials", type=int, default=20)
    ap.add_argument("--q-max", type=int, default=None)
    ap.add_argument("--root-seed", type=int, default=0)
    ap.add_argument("--sketch-kind", default="countsketch")
    ap.add_argument("--s", type=int, default=1)
    ap.add_argument("--unstabilized", action="store_true")
    ap.add_argument("--dtype", default="float64", choices=["float64", "float32"])
    ap.add_argument("--output", default="bench.csv")
    args = ap.parse_args(argv)
    cfg = BenchConfig(dataset=args.dataset, methods=[m for m in args.methods.split(",") if m],
                      k=args.k, l_values=[int(x) for x in args.l_values.split(",") if x],
                      q_max=args.q_max, trials=args.trials, root_seed=args.root_seed,
                      sketch_kind=args.sketch_kind, s=args.s, stabilized=not args.unstabilized,
                      dtype=args.dtype)
    recs = run_benchmark(cfg, args.output)
    print(f"{len(recs)} records -> {args.output}")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
