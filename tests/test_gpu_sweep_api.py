"""Seeded sweeps of the rest of the reference surface against the CPU oracle
on the same bytes: orthonormalize (column count, span), thin_svd / pinv on
graded and rank-deficient matrices, lowrank_factorize (the regression's
error) and power_iterate (span).  fp32 and fp64, ragged shapes."""
import numpy as np
import pytest

from oracle import skp_oracle as o

pytestmark = pytest.mark.gpu


def _graded(m, n, decades, rank, seed, dtype):
    rng = np.random.default_rng(seed)
    u, _ = np.linalg.qr(rng.standard_normal((m, rank)))
    v, _ = np.linalg.qr(rng.standard_normal((n, rank)))
    return ((u * np.logspace(0, -decades, rank)) @ v.T).astype(dtype)


def _proj_dist(q1, q2):
    """|| Q1 Q1^T - Q2 Q2^T ||_2 (same-size orthonormal bases)."""
    return float(np.linalg.norm(q1 @ (q1.T @ q2) - q2, 2)) if q1.shape == q2.shape else np.inf


@pytest.mark.parametrize("i", range(16))
def test_orthonormalize_sweep(i):
    import paper_2605_09755_b200 as skp
    rng = np.random.default_rng(2000 + i)
    m, c = int(rng.integers(50, 3000)), int(rng.integers(1, 120))
    c = min(c, m)
    rank = int(rng.integers(1, c + 1))
    dtype = np.float64 if i % 2 else np.float32
    decades = float(rng.uniform(0, 6 if dtype == np.float32 else 10))
    y = _graded(m, c, decades, rank, i, dtype)
    qo = o.orthonormalize(y)
    qb = skp.orthonormalize(y)
    assert np.abs(qb.T.astype(np.float64) @ qb - np.eye(qb.shape[1])).max() <= (
        1e-5 if dtype == np.float32 else 1e-12)
    # the reference's rank decision (fp32 inputs are decided in fp64, as the
    # reference computes: their rounding noise counts as rank there too)
    assert qb.shape[1] == qo.shape[1], (qb.shape, qo.shape, rank, decades)
    if qb.shape[1] == rank or dtype == np.float64:
        # same span, to the conditioning of y's kept part
        tol = (1e-4 if dtype == np.float32 else 1e-13) * 10 ** decades
        assert _proj_dist(qb.astype(np.float64), qo) <= tol


@pytest.mark.parametrize("i", range(16))
def test_thin_svd_and_pinv_sweep(i):
    import paper_2605_09755_b200 as skp
    rng = np.random.default_rng(3000 + i)
    m, n = int(rng.integers(2, 400)), int(rng.integers(2, 400))
    rank = int(rng.integers(1, min(m, n) + 1))
    a = _graded(m, n, float(rng.uniform(0, 12)), rank, i, np.float64)
    uo, so, vo = o.thin_svd(a)
    res = skp.thin_svd(a)
    np.testing.assert_allclose(res.sigma, so, rtol=0, atol=1e-12 * so[0])
    np.testing.assert_allclose((res.U * res.sigma) @ res.V.T, a, atol=1e-12 * so[0])
    po, pg = o.pinv(a), skp.pinv(a)
    # Moore-Penrose conditions to the accuracy of the kept singular values
    # (entrywise the two pseudo-inverses agree only to eps sigma_1 / sigma_min,
    # the accuracy of either SVD), and entrywise where that is tight
    cut = so > max(m, n) * np.finfo(np.float64).eps * so[0]
    kappa = so[0] / so[cut][-1]
    assert np.linalg.norm(a @ pg @ a - a) <= 1e-12 * kappa * np.linalg.norm(a)
    assert np.linalg.norm(pg @ a @ pg - pg) <= 1e-12 * kappa * np.linalg.norm(pg)
    if kappa < 1e6:
        assert np.abs(pg - po).max() <= 1e-13 * kappa ** 2 * max(1.0, np.abs(po).max())


@pytest.mark.parametrize("i", range(12))
def test_lowrank_factorize_sweep(i):
    import paper_2605_09755_b200 as skp
    rng = np.random.default_rng(4000 + i)
    m, n = int(rng.integers(300, 3000)), int(rng.integers(200, 2000))
    l = int(rng.integers(40, min(n, 500)))
    r2 = int(rng.integers(8, min(l, 80)))
    q = int(rng.integers(0, 3))
    dtype = np.float64 if i % 2 else np.float32
    a = _graded(m, n, float(rng.uniform(0.5, 2.0)), min(m, n, 300), i, dtype)
    spec = skp.RangeFinderSpec(k=max(1, r2 - 5), l=l, r1=l, r2=r2, q=q, eps=0.5, seed=i, s=8)
    yo, xo = o.lowrank_factorize(a, o.Spec(k=max(1, r2 - 5), l=l, r1=l, r2=r2, q=q, seed=i, s=8))
    res = skp.lowrank_factorize(a, spec)
    a64 = a.astype(np.float64)
    eo = np.linalg.norm(yo @ xo - a64) / np.linalg.norm(a64)
    e = np.linalg.norm(res.Y.astype(np.float64) @ res.X - a64) / np.linalg.norm(a64)
    assert abs(e - eo) <= 1e-3 * eo + (1e-6 if dtype == np.float32 else 1e-12), (e, eo)


@pytest.mark.parametrize("i", range(16))
def test_power_iterate_span_sweep(i):
    import paper_2605_09755_b200 as skp
    rng = np.random.default_rng(5000 + i)
    m, l = int(rng.integers(200, 3000)), int(rng.integers(20, 300))
    r2 = int(rng.integers(2, min(l, 60)))
    q = int(rng.integers(0, 4))
    dtype = np.float64 if i < 12 else np.float32
    stab = i % 3 != 2
    atil = _graded(m, l, float(rng.uniform(0.2, 1.5)), min(m, l), i, dtype)
    omega = np.random.default_rng(i).standard_normal((l, r2)).astype(dtype)
    yo = o.power_iterate(atil, omega, q, stabilized=stab)
    y = skp.power_iterate(atil, omega, q, stabilized=stab)
    assert y.shape == yo.shape
    d = _proj_dist(o.orthonormalize(y), o.orthonormalize(yo))
    assert d <= (1e-6 if dtype == np.float64 else 1e-3), (d, stab, q)


@pytest.mark.parametrize("i", range(12))
def test_nystrom_sweep(i):
    """nystrom_psd (power.py:258-298) on seeded PSD matrices against the
    oracle's core on the same bytes: the orthonormalised power at the 1e-3
    bar; the literal core (cond(W) up to ~1e15) at the documented 5e-3."""
    import paper_2605_09755_b200 as skp
    rng = np.random.default_rng(6000 + i)
    n = int(rng.integers(300, 3000))
    l = int(rng.integers(40, min(n, 500)))
    r2 = int(rng.integers(8, min(l, 80)))
    q = int(rng.integers(1, 3))
    dtype = np.float64 if i % 2 else np.float32
    rank = int(rng.integers(r2, min(n, 400)))
    u, _ = np.linalg.qr(rng.standard_normal((n, rank)))
    kmat = ((u * np.exp(-np.arange(rank) * float(rng.uniform(0.01, 0.1)))) @ u.T)
    kmat = ((kmat + kmat.T) / 2).astype(dtype)
    spec = skp.RangeFinderSpec(k=max(1, r2 - 4), l=l, r1=l, r2=r2, q=q, eps=0.5, seed=i, s=8)
    ospec = o.Spec(k=max(1, r2 - 4), l=l, r1=l, r2=r2, q=q, seed=i, s=8)
    for stab, tol in ((True, 1e-3), (False, 5e-3)):
        res = skp.nystrom_psd(kmat, spec, stabilized=stab)
        c = np.asarray(res.C.cpu() if hasattr(res.C, "cpu") else res.C, dtype=np.float64)
        w = np.asarray(res.W.cpu() if hasattr(res.W, "cpu") else res.W, dtype=np.float64)
        e = o.nystrom_rel_error(kmat, c, w)
        co, wo = o.nystrom_core(kmat, ospec, stabilized=stab)
        eo = o.nystrom_rel_error(kmat, co, wo)
        assert abs(e - eo) <= tol * eo + 1e-12, (stab, e, eo, n, l, r2, q, dtype)


@pytest.mark.parametrize("i", range(24))
def test_sketch_apply_sweep(i):
    """SketchOperator.apply_right / apply_left_transpose (sketching.py:158-192)
    for every kind against the oracle (whose draws are pinned to the live
    reference): ragged n, r, s; fp32 and fp64; numpy and CUDA operands."""
    import torch
    import paper_2605_09755_b200 as skp
    rng = np.random.default_rng(9000 + i)
    kind = ("countsketch", "srht", "gaussian", "sign")[i % 4]
    n = int(rng.integers(1, 3000))
    r = int(rng.integers(1, min(n, 600) + 1)) if kind != "srht" else \
        int(rng.integers(1, min(1 << (n - 1).bit_length(), 600) + 1))
    s = int(rng.integers(1, min(r, 12) + 1)) if kind == "countsketch" else None
    dtype = np.float64 if (i // 4) % 2 else np.float32
    cuda = (i // 8) % 2 == 1
    op = skp.make_sketch(kind, n, r, seed=i, s=s)
    ref = o.CountSketch(kind, n, r, i, s=s)
    a = rng.standard_normal((int(rng.integers(1, 300)), n)).astype(dtype)
    x = rng.standard_normal((n, int(rng.integers(1, 40)))).astype(dtype)
    ar = torch.from_numpy(a).cuda() if cuda else a
    xr = torch.from_numpy(x).cuda() if cuda else x
    got_r = op.apply_right(ar)
    got_l = op.apply_left_transpose(xr)
    got_r = got_r.cpu().numpy() if cuda else got_r
    got_l = got_l.cpu().numpy() if cuda else got_l
    tol = 1e-12 if dtype == np.float64 else 2e-6
    want_r = ref.apply_right(a)
    want_l = ref.apply_left_transpose(x)
    assert np.abs(got_r - want_r).max() <= tol * max(1.0, np.abs(want_r).max()) * np.sqrt(n)
    assert np.abs(got_l - want_l).max() <= tol * max(1.0, np.abs(want_l).max()) * np.sqrt(n)


@pytest.mark.parametrize("i", range(12))
def test_lowrank_factorize_kinds_sweep(i):
    """lowrank_factorize (power.py:202-239) with the secondary sketch's own
    family and size (s2_kind, s2_r) and other primary families, vs the oracle."""
    import paper_2605_09755_b200 as skp
    rng = np.random.default_rng(9700 + i)
    kind = ("countsketch", "srht", "gaussian", "sign")[i % 4]
    s2_kind = ("srht", "countsketch", "sign", "gaussian")[(i // 4) % 4]
    m, n = int(rng.integers(300, 2500)), int(rng.integers(200, 1500))
    l = int(rng.integers(40, min(n, 300)))
    r2 = int(rng.integers(8, min(l, 60)))
    s2_r = int(rng.integers(r2 + 2, min(m, 4 * l) + 1))
    q = int(rng.integers(0, 3))
    dtype = np.float64 if i % 2 else np.float32
    a = _graded(m, n, float(rng.uniform(0.5, 2.0)), min(m, n, 300), i + 50, dtype)
    spec = skp.RangeFinderSpec(k=max(1, r2 - 5), l=l, r1=l, r2=r2, q=q, eps=0.5, seed=i, s=4,
                               sketch_kind=kind, s2_kind=s2_kind, s2_r=s2_r)
    yo, xo = o.lowrank_factorize(a, o.Spec(k=max(1, r2 - 5), l=l, r1=l, r2=r2, q=q, seed=i, s=4,
                                           sketch_kind=kind, s2_kind=s2_kind, s2_r=s2_r))
    res = skp.lowrank_factorize(a, spec)
    a64 = a.astype(np.float64)
    eo = np.linalg.norm(yo @ xo - a64) / np.linalg.norm(a64)
    e = np.linalg.norm(res.Y.astype(np.float64) @ res.X - a64) / np.linalg.norm(a64)
    assert abs(e - eo) <= 1e-3 * eo + (1e-6 if dtype == np.float32 else 1e-12), (kind, s2_kind, e, eo)


@pytest.mark.parametrize("i", range(8))
def test_nystrom_kinds_sweep(i):
    """nystrom_psd with the other sketch families and start-block families
    (orthonormalised core, the 1e-3 bar) vs the oracle."""
    import paper_2605_09755_b200 as skp
    rng = np.random.default_rng(9900 + i)
    kind = ("srht", "gaussian", "sign", "countsketch")[i % 4]
    omega_kind = ("gaussian", "sign")[(i // 4) % 2]
    n = int(rng.integers(300, 2000))
    l = int(rng.integers(40, min(n, 400)))
    r2 = int(rng.integers(8, min(l, 60)))
    dtype = np.float64 if i % 2 else np.float32
    rank = int(rng.integers(r2, min(n, 300)))
    u, _ = np.linalg.qr(rng.standard_normal((n, rank)))
    kmat = (u * np.exp(-np.arange(rank) * float(rng.uniform(0.02, 0.1)))) @ u.T
    kmat = ((kmat + kmat.T) / 2).astype(dtype)
    spec = skp.RangeFinderSpec(k=max(1, r2 - 4), l=l, r1=l, r2=r2, q=2, eps=0.5, seed=i, s=4,
                               sketch_kind=kind, omega_kind=omega_kind)
    ospec = o.Spec(k=max(1, r2 - 4), l=l, r1=l, r2=r2, q=2, seed=i, s=4, sketch_kind=kind,
                   omega_kind=omega_kind)
    res = skp.nystrom_psd(kmat, spec, stabilized=True)
    c = np.asarray(res.C.cpu() if hasattr(res.C, "cpu") else res.C, dtype=np.float64)
    w = np.asarray(res.W.cpu() if hasattr(res.W, "cpu") else res.W, dtype=np.float64)
    e = o.nystrom_rel_error(kmat, c, w)
    co, wo = o.nystrom_core(kmat, ospec, stabilized=True)
    eo = o.nystrom_rel_error(kmat, co, wo)
    assert abs(e - eo) <= 1e-3 * eo + 1e-12, (kind, omega_kind, e, eo)
