"""Seeded synthetic inputs for the BASELINE.json configurations (C1-C5).

Input construction only -- not part of the accelerated path.  C1/C2 restate
the reference generator (``_haar_columns`` / ``_rotate_spectrum``,
/root/reference/pkg/src/skpower/data_io.py:38-52) in numpy so the oracle and
the device see identical bytes.  C3-C5 are too large for a CPU Haar QR and are
built on the GPU with torch (cuSOLVER QR + cuBLAS), row block by row block,
from a fixed seed; the same bytes are copied to the host for the oracle.

Noise conventions (BASELINE.json configs):
  C2  "E i.i.d. N(0, (1e-4)^2/n)"  -> variance notation, std = 1e-4/sqrt(n).
  C3  "N(0, 1e-6) noise"            -> read as std 1e-6 (variance 1e-6 would be
                                       std 1e-3, 20x the signal RMS of 4.5e-5 and
                                       would turn the polydecay matrix into noise).
  C5  "N(0, 1e-8)"                  -> std 1e-8, same reading.
"""
from __future__ import annotations

import math

import numpy as np

_M64 = (1 << 64) - 1


def _substream(seed: int, *idx: int) -> int:
    # same derivation as sketching.substream (reference sketching.py:46-54)
    ent = [int(seed) & _M64] + [int(i) & _M64 for i in idx]
    return int(np.random.SeedSequence(entropy=ent).generate_state(1, np.uint64)[0])


def haar_columns(rows: int, cols: int, seed: int) -> np.ndarray:
    """data_io.py:38-46: QR of a seeded Gaussian, R-diagonal sign-fixed."""
    g = np.random.default_rng(np.random.SeedSequence(entropy=[seed])).standard_normal((rows, cols))
    q, r = np.linalg.qr(g)
    sg = np.sign(np.diag(r))
    sg[sg == 0.0] = 1.0
    return q * sg


def rotate_spectrum(m: int, n: int, spectrum: np.ndarray, seed: int) -> np.ndarray:
    """data_io.py:49-52."""
    u = haar_columns(m, len(spectrum), _substream(seed, 0))
    v = haar_columns(n, len(spectrum), _substream(seed, 1))
    return (u * spectrum) @ v.T


def c1_matrix(seed: int = 1, m: int = 2000, n: int = 1000) -> np.ndarray:
    """C1: float64, sigma_i = 1/i (i = 1..1000)."""
    p = min(m, n)
    return rotate_spectrum(m, n, 1.0 / np.arange(1.0, p + 1.0), seed)


def c2_matrix(seed: int = 2, m: int = 20000, n: int = 10000, r: int = 1000) -> np.ndarray:
    """C2: fp32, sigma_i = 10^(-i/100), i <= r, plus E ~ N(0, (1e-4)^2/n)."""
    a = rotate_spectrum(m, n, 10.0 ** (-np.arange(1.0, r + 1.0) / 100.0), seed)
    rng = np.random.default_rng(np.random.SeedSequence(entropy=[_substream(seed, 2)]))
    a += (1e-4 / math.sqrt(n)) * rng.standard_normal((m, n))
    return a.astype(np.float32)


# ---------------------------------------------------------------------------
# GPU-built inputs (C3-C5): torch is input-construction plumbing here.
# ---------------------------------------------------------------------------

def _torch_orth(rows: int, cols: int, gen, device):
    import torch
    g = torch.randn(rows, cols, generator=gen, device=device, dtype=torch.float32)
    q, _ = torch.linalg.qr(g)
    return q


def lowrank_plus_noise_gpu(m: int, n: int, spectrum: np.ndarray, noise_std: float, seed: int,
                           device="cuda", row0: int = 0, rows: int | None = None, block: int = 65536):
    """A = G diag(spectrum) H^T + noise, G (m x r), H (n x r) orthonormalised
    seeded Gaussians, fp32, built on ``device``.  Returns rows [row0, row0+rows)
    of A; the full-matrix factors are seeded so any row slab is reproducible
    (used by row-sharded multi-GPU runs)."""
    import torch
    rows = m - row0 if rows is None else rows
    r = len(spectrum)
    gen = torch.Generator(device=device)
    gen.manual_seed(int(_substream(seed, 1)) & 0x7FFFFFFFFFFFFFFF)
    h = _torch_orth(n, r, gen, device)
    sig = torch.as_tensor(np.asarray(spectrum, dtype=np.float32), device=device)
    hs = (h * sig).T.contiguous()                       # r x n
    # G: orthonormal columns of an m x r Gaussian.  Built blockwise by
    # Cholesky-QR in fp64 so any row slab can be regenerated independently.
    gram = torch.zeros(r, r, dtype=torch.float64, device=device)
    for b0 in range(0, m, block):
        gb = _g_block(seed, b0, min(block, m - b0), r, device)
        gram += gb.double().T @ gb.double()
    lchol = torch.linalg.cholesky(gram)
    linv_t = torch.linalg.solve_triangular(lchol, torch.eye(r, dtype=torch.float64, device=device),
                                           upper=False).T.contiguous()
    out = torch.empty(rows, n, dtype=torch.float32, device=device)
    for b0 in range(row0 - row0 % block, row0 + rows, block):
        bl = min(block, m - b0)
        gb = (_g_block(seed, b0, bl, r, device).double() @ linv_t).float()
        lo, hi = max(b0, row0), min(b0 + bl, row0 + rows)
        if lo >= hi:
            continue
        blk = gb[lo - b0:hi - b0] @ hs
        if noise_std > 0:
            ng = torch.Generator(device=device)
            ng.manual_seed((int(_substream(seed, 3, b0)) & 0x7FFFFFFFFFFFFFFF))
            nz = torch.randn(bl, n, generator=ng, device=device, dtype=torch.float32)
            blk += noise_std * nz[lo - b0:hi - b0]
        out[lo - row0:hi - row0] = blk
    return out


def _g_block(seed: int, b0: int, bl: int, r: int, device):
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(int(_substream(seed, 2, b0)) & 0x7FFFFFFFFFFFFFFF)
    return torch.randn(bl, r, generator=g, device=device, dtype=torch.float32)


def c3_matrix_gpu(seed: int = 3, m: int = 262144, n: int = 16384, rank: int = 4096,
                  noise_std: float = 1e-6, device="cuda", row0: int = 0, rows: int | None = None):
    """C3: sigma_i = i^-0.5 (i <= 4096), fp32, plus N(0, std=1e-6)."""
    spec = np.arange(1.0, rank + 1.0) ** -0.5
    return lowrank_plus_noise_gpu(m, n, spec, noise_std, seed, device, row0, rows)


def c5_matrix_gpu(seed: int = 5, m: int = 1048576, n: int = 32768, rank: int = 8192,
                  noise_std: float = 1e-8, device="cuda", row0: int = 0, rows: int | None = None):
    """C5: sigma_i = exp(-i/1000) (i <= 8192), fp32, plus N(0, std=1e-8)."""
    spec = np.exp(-np.arange(1.0, rank + 1.0) / 1000.0)
    return lowrank_plus_noise_gpu(m, n, spec, noise_std, seed, device, row0, rows)


def rbf_points(n: int, d: int = 16, seed: int = 4) -> np.ndarray:
    return np.random.default_rng(np.random.SeedSequence(entropy=[seed])).standard_normal((n, d))


def rbf_bandwidth(x: np.ndarray, sub: int = 4096, seed: int = 4) -> float:
    """Median pairwise distance over a seeded ``sub``-point subsample."""
    rng = np.random.default_rng(np.random.SeedSequence(entropy=[_substream(seed, 1)]))
    idx = rng.choice(x.shape[0], size=min(sub, x.shape[0]), replace=False)
    p = x[idx]
    sq = (p * p).sum(1)
    d2 = np.maximum(sq[:, None] + sq[None, :] - 2.0 * p @ p.T, 0.0)
    iu = np.triu_indices(len(p), 1)
    return float(np.median(np.sqrt(d2[iu])))


def rbf_kernel_gpu(x: np.ndarray, h: float, device="cuda", row0: int = 0, rows: int | None = None):
    """K_ij = exp(-||x_i - x_j||^2 / (2 h^2)), fp32, exactly symmetric
    (entries computed in fp64 from the unordered pair, then rounded)."""
    import torch
    n = x.shape[0]
    rows = n - row0 if rows is None else rows
    xt = torch.as_tensor(x, dtype=torch.float64, device=device)
    sq = (xt * xt).sum(1)
    out = torch.empty(rows, n, dtype=torch.float32, device=device)
    blk = 4096
    for b0 in range(row0, row0 + rows, blk):
        b1 = min(b0 + blk, row0 + rows)
        d2 = (sq[b0:b1, None] + sq[None, :] - 2.0 * xt[b0:b1] @ xt.T).clamp_min_(0.0)
        out[b0 - row0:b1 - row0] = torch.exp(-d2 / (2.0 * h * h)).float()
    # symmetric by construction up to the fp64 rounding of d2; force exact
    # symmetry when the whole matrix is resident
    if row0 == 0 and rows == n:
        out = torch.minimum(out, out.T.contiguous())
    return out
