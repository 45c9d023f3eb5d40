"""Per-kernel parity on the B200, through the C-ABI (libskp.so via ctypes).

K1 (CountSketch draw) must be bit-exact with the live-reference golden
fixtures and the C oracle; K2/K3 sketch application, the GEMMs and the small
fp64 kernels are compared with numpy/torch fp64 references at stated
tolerances.
"""
import hashlib

import numpy as np
import pytest
import torch

from conftest import small_cs_cases
from oracle import skp_oracle as o

pytestmark = pytest.mark.gpu


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def skp():
    import paper_2605_09755_b200 as m
    return m


@pytest.fixture(scope="module")
def ops():
    from paper_2605_09755_b200 import _ops
    return _ops


# ------------------------------------------------------------------ K1 ----

def test_countsketch_small_golden(skp, golden_cs):
    for i, n, r, s, seed in small_cs_cases(golden_cs):
        if s > 32 or r >= 2**31:
            with pytest.raises(ValueError, match="unsupported"):
                skp.make_sketch("countsketch", n, r, seed, s=s)
            continue
        op = skp.make_sketch("countsketch", n, r, seed, s=s)
        np.testing.assert_array_equal(op._cols, golden_cs[f"cs{i}_cols"], err_msg=f"case {i}")
        np.testing.assert_array_equal(op._signs.astype(np.int8), golden_cs[f"cs{i}_signs"])


@pytest.mark.parametrize("name", ["C2", "C3", "C4", "C5_l4000", "C5_l8000", "C5_l16000"])
def test_countsketch_config_shapes_golden(skp, golden, name):
    b = golden["countsketch_big"][name]
    op = skp.make_sketch("countsketch", b["n"], b["r"], int(b["seed"]), s=b["s"])
    assert sha(op._cols) == b["cols_sha256"]
    assert sha(op._signs.astype(np.int8)) == b["signs_sha256"]


@pytest.mark.parametrize("n,r,s,seed", [
    (1, 1, 1, 0), (1, 5, 5, 3), (37, 1, 1, 4), (100, 3, 2, 5), (513, 1000, 7, 6),
    (64, 1025, 32, 7), (333, 31, 31, 8), (1000, 1_500_000_000, 1, 9), (2049, 2, 1, 10),
    (3000, 129, 1, 11), (40, 33, 9, 12), (513, 64, 1, 13), (1025, 4000, 1, 5),
    (16385, 4000, 1, 2), (999, 37, 1, 77)])
def test_countsketch_random_vs_c_oracle(skp, n, r, s, seed):
    op = skp.make_sketch("countsketch", n, r, seed, s=s)
    cols, signs = o.countsketch_c(seed, n, r, s)
    np.testing.assert_array_equal(op._cols, cols)
    np.testing.assert_array_equal(op._signs, signs)
    if r < 10**6 and n * r < 10**7:   # and numpy itself (the reference's generator)
        cn, sn = o.countsketch_numpy(seed, n, r, s)
        np.testing.assert_array_equal(op._cols, cn)
        np.testing.assert_array_equal(op._signs, sn)


@pytest.mark.parametrize("s", [1, 3, 8])
def test_countsketch_row_ranges_compose(ops, s):
    n, r, seed = 1001, 257, 42
    st, inc = o.pcg64_state(seed)
    full_c, full_s = ops.countsketch(st, inc, n, r, s, "cuda")
    for j0, j1 in [(0, 1), (0, 500), (500, 1001), (999, 1001), (333, 334)]:
        c, g = ops.countsketch(st, inc, n, r, s, "cuda", j0, j1)
        assert torch.equal(c, full_c[j0:j1]) and torch.equal(g, full_s[j0:j1])


def test_countsketch_bad_arguments(skp):
    with pytest.raises(ValueError):
        skp.make_sketch("countsketch", 10, 4, seed=0, s=5)
    with pytest.raises(ValueError):
        skp.make_sketch("gaussian", 10, 0, seed=0)
    with pytest.raises(ValueError):
        skp.make_sketch("nope", 10, 4, seed=0)
    with pytest.raises(ValueError):
        skp.make_sketch("identity", 10, 4, seed=0)
    with pytest.raises(ValueError, match="padded dimension"):
        skp.make_sketch("srht", 16, 17, seed=0)


# ------------------------------------------------------------------- K7 ---

@pytest.mark.parametrize("case", ["50_12_9", "64_64_3", "1000_37_21", "3000_300_77"])
@pytest.mark.parametrize("dtype,tol", [(np.float64, 1e-12), (np.float32, 3e-6)])
def test_srht_matches_live_reference(skp, case, dtype, tol):
    """Signs / subset bit-exact (numpy draw); A S, S^T X and densify vs the
    reference's own outputs (tests/golden/make_srht_golden.py)."""
    import os
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "srht_golden.npz"))
    n, r, seed = (int(v) for v in case.split("_"))
    op = skp.make_sketch("srht", n, r, seed=seed)
    assert np.array_equal(op._signs, g[f"signs_{case}"])
    assert np.array_equal(op._subset, g[f"subset_{case}"])
    a, x = g[f"a_{case}"].astype(dtype), g[f"x_{case}"].astype(dtype)
    ra, rx = g[f"right_{case}"], g[f"left_{case}"]
    got_a, got_x = op.apply_right(a), op.apply_left_transpose(x)
    assert got_a.dtype == dtype and got_x.dtype == dtype
    scale_a = np.abs(a).max() * np.sqrt(n) + 1e-300
    scale_x = np.abs(x).max() * np.sqrt(n) + 1e-300
    assert np.abs(got_a - ra).max() <= tol * scale_a
    assert np.abs(got_x - rx).max() <= tol * scale_x
    if f"dense_{case}" in g.files:
        assert np.abs(op.densify() - g[f"dense_{case}"]).max() <= 1e-12


# ---------------------------------------------------------------- K2/K3 ---

@pytest.mark.parametrize("dtype,tol", [(np.float64, 1e-12), (np.float32, 2e-6)])
@pytest.mark.parametrize("m,n,r,s", [(50, 200, 40, 4), (1, 7, 3, 2), (257, 1000, 200, 8),
                                     (3, 60000, 100, 8), (130, 513, 64, 1)])
def test_sketch_apply_matches_dense(skp, dtype, tol, m, n, r, s):
    rng = np.random.default_rng(m + n)
    op = skp.make_sketch("countsketch", n, r, seed=21, s=s)
    dense = op.densify() if n * r <= 10**7 else None
    a = rng.standard_normal((m, n)).astype(dtype)
    fast = op.apply_right(a)
    assert fast.dtype == dtype and fast.shape == (m, r)
    ref = a.astype(np.float64) @ dense if dense is not None else o.CountSketch(
        "countsketch", n, r, 21, s=s).apply_right(a)
    assert np.abs(fast - ref).max() <= tol * np.linalg.norm(a.astype(np.float64)) + 1e-300
    b = rng.standard_normal((n, 30)).astype(dtype)
    fast_t = op.apply_left_transpose(b)
    ref_t = (dense.T @ b.astype(np.float64)) if dense is not None else o.CountSketch(
        "countsketch", n, r, 21, s=s).apply_left_transpose(b)
    assert np.abs(fast_t - ref_t).max() <= tol * np.linalg.norm(b.astype(np.float64))


def test_sketch_identity_input_and_zero(skp):
    op = skp.make_sketch("countsketch", 20, 7, seed=11, s=3)
    np.testing.assert_array_equal(op.apply_right(np.eye(20)), op.densify())
    np.testing.assert_array_equal(op.apply_left_transpose(np.eye(20)), op.densify().T)
    np.testing.assert_array_equal(op.apply_right(np.zeros((5, 20))), np.zeros((5, 7)))


def test_sketch_fused_norm_and_nonfinite(skp, ops):
    rng = np.random.default_rng(3)
    for n in (500, 60000):
        a = rng.standard_normal((9, n)).astype(np.float32)
        a[4, n // 3] = np.nan
        a[7, 1] = np.inf
        op = skp.make_sketch("countsketch", n, 50, seed=1, s=4)
        t = torch.from_numpy(a).cuda()
        fro2 = torch.zeros(1, dtype=torch.float64, device="cuda")
        bad = torch.zeros(1, dtype=torch.int64, device="cuda")
        op.right(t, fro2=fro2, nonfinite=bad)
        # K2 v1 counts the 2 non-finite inputs, the row gather (fp32, aligned
        # rows) the s outputs each of them reaches: a counter read as a flag
        assert int(bad.item()) >= 2
        bad.zero_()
        ops.sketch_right(t, op.colptr, op.entries, op.s, op.r, nonfinite=bad)
        assert int(bad.item()) == 2
        with pytest.raises(ValueError, match="non-finite"):
            op.apply_right(a)
        a[4, n // 3] = 0
        a[7, 1] = 0
        fro2.zero_()
        op.right(torch.from_numpy(a).cuda(), fro2=fro2)
        assert abs(fro2.item() - float((a.astype(np.float64) ** 2).sum())) <= 1e-9 * fro2.item()


@pytest.mark.parametrize("m,n,r,s", [(67, 16384, 4000, 8), (5, 1000, 300, 8), (130, 513, 64, 1),
                                     (40, 2050, 1600, 3), (1, 24576, 4000, 8),
                                     (9, 32768, 4000, 8), (3, 70001, 6000, 4),
                                     # the three-buffer ring wrapping several times
                                     (300, 4096, 2000, 8), (1000, 8192, 768, 8),
                                     # K2 v3 lanes with > 2 entries on the row's first
                                     # 32 words (the re-read path), and an odd pass width
                                     (50, 2000, 900, 32), (7, 16383, 1700, 5)])
def test_sketch_gather_permuted(skp, ops, m, n, r, s):
    """K2 v2: (A S) P from the row-gather kernel == the oracle's A S with its
    columns taken in plan order; fused fp64 ||A||_F^2 and the non-finite test."""
    rng = np.random.default_rng(n + r)
    op = skp.make_sketch("countsketch", n, r, seed=13, s=s)
    plan = op.gather_plan()
    assert plan is not None
    g, perm = plan
    assert sorted(perm.tolist()) == list(range(r))      # a permutation of the columns
    a = rng.standard_normal((m, n)).astype(np.float32)
    t = ops.empty2d(m, n, torch.float32, "cuda")
    t.copy_(torch.from_numpy(a))
    fro2 = torch.zeros(1, dtype=torch.float64, device="cuda")
    bad = torch.zeros(1, dtype=torch.int64, device="cuda")
    amax = torch.zeros(1, dtype=torch.int32, device="cuda")
    out, perm2 = op.right_permuted(t, fro2=fro2, nonfinite=bad, amax=amax)
    assert (perm2.cpu().numpy() == perm).all()
    # the fused max|A S| (input of the 3xFP16 split) is exact
    assert amax.view(torch.float32).item() == out.abs().max().item()
    ref = o.CountSketch("countsketch", n, r, 13, s=s).apply_right(a.astype(np.float64))
    got = out.cpu().numpy().astype(np.float64)
    scale = np.abs(ref).max()
    assert np.abs(got - ref[:, perm]).max() <= 4e-7 * np.sqrt(n * s / r) * scale + 1e-30
    assert int(bad.item()) == 0
    want = float((a.astype(np.float64) ** 2).sum())
    assert abs(fro2.item() - want) <= 1e-12 * want
    # a single non-finite entry is reported
    a[m // 2, n // 3] = np.nan
    t.copy_(torch.from_numpy(a))
    bad.zero_()
    op.right_permuted(t, nonfinite=bad)
    assert int(bad.item()) >= 1


def test_sketch_gather_variant(skp):
    """The BASELINE sketch shapes run K2 v3 (two slices per CTA, 16-bit
    schedule): C2 (n 10000, l 2000), C3 (16384, 4000), C5 (32768, 8000 in two
    column passes); one slice per CTA where the slice count is one or a pass
    is wider than 16384 words."""
    from paper_2605_09755_b200 import _lib
    v = _lib.load().skp_sketch_gather_variant
    for n, r in [(10000, 2000), (16384, 4000), (32768, 8000), (32768, 16000)]:
        assert v(n, r) == 3, (n, r)
    # passes wider than 16384 words (C4's n = 65536: 3 x 21856) or one slice
    assert v(24576, 4000) == 2 and v(65536, 4096) == 2 and v(16384, 700) == 2


@pytest.mark.parametrize("m,n,r,s", [(67, 16384, 4000, 8), (9, 32768, 4000, 8), (3, 70001, 6000, 4),
                                     (130, 512, 64, 1), (1000, 8192, 768, 8)])
def test_right_natural_order_on_the_gather(skp, ops, m, n, r, s):
    """SketchOperator.right (apply_right's device op) in the reference's column
    order through K2 v2 + the in-place column un-permutation -- fused checks
    kept, a caller-provided out honoured -- against the oracle."""
    rng = np.random.default_rng(m * 7 + n)
    op = skp.make_sketch("countsketch", n, r, seed=23, s=s)
    a = rng.standard_normal((m, n)).astype(np.float32)
    t = ops.empty2d(m, n, torch.float32, "cuda")
    t.copy_(torch.from_numpy(a))
    fro2 = torch.zeros(1, dtype=torch.float64, device="cuda")
    bad = torch.zeros(1, dtype=torch.int64, device="cuda")
    out = ops.empty2d(m, r, torch.float32, "cuda")
    got = op.right(t, out=out, fro2=fro2, nonfinite=bad)
    assert got.data_ptr() == out.data_ptr()
    assert op.gather_plan() is not None          # the row gather ran (v1 has no plan)
    ref = o.CountSketch("countsketch", n, r, 23, s=s).apply_right(a.astype(np.float64))
    scale = np.abs(ref).max()
    assert np.abs(got.cpu().numpy() - ref).max() <= 4e-7 * np.sqrt(n * s / r) * scale + 1e-30
    assert int(bad.item()) == 0
    want = float((a.astype(np.float64) ** 2).sum())
    assert abs(fro2.item() - want) <= 1e-12 * want
    # the reference API on top of it
    assert np.abs(op.apply_right(a) - ref).max() <= 4e-7 * np.sqrt(n * s / r) * scale + 1e-30


@pytest.mark.parametrize("m,n,r,s", [(67, 16384, 4000, 8), (9, 32768, 4000, 8), (5, 65536, 4096, 8)])
def test_sketch_gather_acc64(skp, ops, m, n, r, s):
    """K2 v2 with fp64 accumulation (the psd Nystrom sketch): (A S) P in fp64
    equal to the oracle's fp64 product to fp64 rounding."""
    rng = np.random.default_rng(n + r + 1)
    op = skp.make_sketch("countsketch", n, r, seed=17, s=s)
    g, perm = op.gather_plan()
    a = rng.standard_normal((m, n)).astype(np.float32)
    t = ops.empty2d(m, n, torch.float32, "cuda")
    t.copy_(torch.from_numpy(a))
    bad = torch.zeros(1, dtype=torch.int64, device="cuda")
    out, _ = op.right_permuted(t, nonfinite=bad, out_dtype=torch.float64)
    assert out.dtype == torch.float64 and int(bad.item()) == 0
    ref = o.CountSketch("countsketch", n, r, 17, s=s).apply_right(a.astype(np.float64))
    assert np.abs(out.cpu().numpy() - ref[:, perm]).max() <= 1e-13 * np.abs(ref).max()


@pytest.mark.parametrize("n", [1, 63, 64, 65, 300, 4097])
@pytest.mark.parametrize("dt", [torch.float32, torch.float64])
def test_sym_check(ops, n, dt):
    """_check_psd's tiled symmetry test: max |a - a^T| and max |a| in one pass,
    exact against torch (ragged tiles and unaligned rows included)."""
    g = torch.Generator(device="cuda").manual_seed(n)
    x = torch.randn(n, n, generator=g, device="cuda", dtype=torch.float64)
    a = ((x + x.T) / 2).to(dt)
    i, j = (n * 2) // 3, n // 5
    a[i, j] += 0.125
    ref_d = (a.double() - a.double().T).abs().max().item()
    ref_a = a.double().abs().max().item()
    got = ops.sym_check(a).tolist()
    assert got == [ref_d, ref_a]
    if n > 8:   # a view with an odd leading dimension (scalar loads)
        big = torch.zeros(n, n + 3, device="cuda", dtype=dt)
        big[:, :n] = a
        got2 = ops.sym_check(big[:, :n]).tolist()
        assert got2 == [ref_d, ref_a]


def test_sketch_gather_declines_outside_its_envelope(skp, ops):
    """No plan (and right_permuted -> None, the caller keeps K2 v1) when rows do
    not fit the smem row buffer or a column needs more than 128 steps."""
    assert skp.make_sketch("countsketch", 98305, 4000, seed=1, s=8).gather_plan() is None
    op = skp.make_sketch("countsketch", 4096, 64, seed=1, s=8)     # ~512 entries per column
    assert op.gather_plan() is None
    t = ops.empty2d(3, 4096, torch.float32, "cuda").zero_()
    assert op.right_permuted(t) is None
    assert op.right_permuted(t.double()) is None


def test_sketch_gather_deferred_failure_falls_back(skp, ops):
    """A plan whose schedule overflows (here ~512 entries per column) is not
    checked on the host in the range finder: the kernel flags it through the
    non-finite counter and the range finder re-runs on K2 v1 -- same result as
    the oracle, and a genuinely non-finite input still raises."""
    rng = np.random.default_rng(8)
    m, n = 300, 4096
    a = (rng.standard_normal((m, 30)) @ rng.standard_normal((30, n))).astype(np.float32)
    spec = skp.RangeFinderSpec(k=10, l=64, r1=64, r2=20, q=1, eps=0.5, s=8, seed=4)
    op = skp.make_sketch("countsketch", n, 64, seed=0, s=8)
    t = ops.empty2d(m, n, torch.float32, "cuda")
    t.copy_(torch.from_numpy(a))
    bad = torch.zeros(1, dtype=torch.int64, device="cuda")
    got = op.right_permuted(t, nonfinite=bad, deferred=True)
    assert got is not None and int(bad.item()) >= ops.GATHER_PLAN_FAIL_MARK
    q = skp.range_finder_sketched(a, spec)
    ref = o.range_finder_sketched(a, o.Spec(k=10, l=64, r1=64, r2=20, q=1, s=8, seed=4))
    a64 = a.astype(np.float64)
    assert abs(o.proj_rel_error(a64, q.astype(np.float64)) - o.proj_rel_error(a64, ref)) \
        <= 1e-3 * o.proj_rel_error(a64, ref) + 1e-6
    a[5, 7] = np.inf
    with pytest.raises(ValueError, match="non-finite"):
        skp.range_finder_sketched(a, spec)


def test_sketch_gather_range_finder_matches_v1(skp, ops, monkeypatch):
    """The range finder on (A S P, P^T Omega) (K2 v2) gives the same sigma and
    projection error as on (A S, Omega) (K2 v1): both fp32 on the device, they
    differ only in the sketch's summation order."""
    from paper_2605_09755_b200 import sketching
    rng = np.random.default_rng(5)
    m, n = 600, 3000
    u = np.linalg.qr(rng.standard_normal((m, 40)))[0]
    v = np.linalg.qr(rng.standard_normal((n, 40)))[0]
    # noise floor ~8% of sigma_1: inside the fp32 CholeskyQR envelope
    a = ((u * np.logspace(0, -1, 40)) @ v.T + 1e-3 * rng.standard_normal((m, n))).astype(np.float32)
    spec = skp.RangeFinderSpec(k=20, l=400, r1=400, r2=60, q=2, eps=0.5, s=8, seed=9)
    assert skp.make_sketch("countsketch", n, 400, seed=0, s=8).gather_plan() is not None
    q2 = skp.range_finder_sketched(a, spec)                       # K2 v2
    monkeypatch.setattr(sketching.SketchOperator, "right_permuted", lambda *x, **k: None)
    q1 = skp.range_finder_sketched(a, spec)                       # K2 v1
    a64 = a.astype(np.float64)
    s1 = np.linalg.svd(q1.T.astype(np.float64) @ a64, compute_uv=False)
    s2 = np.linalg.svd(q2.T.astype(np.float64) @ a64, compute_uv=False)
    assert np.abs(s1[:20] - s2[:20]).max() <= 2e-6 * s1[0]
    e1, e2 = o.proj_rel_error(a64, q1.astype(np.float64)), o.proj_rel_error(a64, q2.astype(np.float64))
    ref = o.range_finder_sketched(a, o.Spec(k=20, l=400, r1=400, r2=60, q=2, s=8, seed=9))
    e0 = o.proj_rel_error(a64, ref)
    assert abs(e2 - e1) <= 1e-4 * e1 and abs(e2 - e0) <= 1e-3 * e0


def test_sketch_dimension_mismatch(skp):
    op = skp.make_sketch("countsketch", 20, 7, seed=11, s=3)
    with pytest.raises(ValueError, match="mismatch"):
        op.apply_right(np.ones((3, 19)))
    with pytest.raises(ValueError, match="mismatch"):
        op.apply_left_transpose(np.ones((19, 3)))


# ------------------------------------------------------------------ K4 ----

@pytest.mark.parametrize("ta,tb", [(0, 0), (1, 0), (0, 1), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (67, 45, 131), (256, 130, 4097), (30, 40, 200000),
                                   (1000, 110, 2000)])
@pytest.mark.parametrize("dt", [torch.float32, torch.float64])
def test_gemm_vs_torch(ops, ta, tb, M, N, K, dt):
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N + K)
    a = torch.randn((K, M) if ta else (M, K), generator=g, device="cuda", dtype=dt)
    b = torch.randn((N, K) if tb else (K, N), generator=g, device="cuda", dtype=dt)
    ref = (a.double().T if ta else a.double()) @ (b.double().T if tb else b.double())
    c0 = torch.randn(M, N, generator=g, device="cuda", dtype=dt)
    out = c0.clone()
    ops.gemm(a, b, bool(ta), bool(tb), alpha=0.5, beta=2.0, out=out)
    expect = 0.5 * ref + 2.0 * c0.double()
    scale = (a.double().abs().max() * b.double().abs().max() * np.sqrt(K)).item() + 1.0
    tol = 1e-13 if dt == torch.float64 else 2e-6
    assert (out.double() - expect).abs().max().item() <= tol * scale


def test_gemm_modes_agree(ops):
    g = torch.Generator(device="cuda").manual_seed(5)
    a = torch.randn(2048, 520, generator=g, device="cuda")
    b = torch.randn(2048, 110, generator=g, device="cuda")
    ref = a.double().T @ b.double()
    for mode in ("auto", "fp32"):
        c = ops.gemm(a, b, True, False, mode=mode)
        assert (c.double() - ref).abs().max().item() <= 1e-5 * ref.abs().max().item()


# ------------------------------------------------ K4h (3xFP16, pre-split) --

@pytest.mark.parametrize("scale", [1.0, 3e-19, 7e17])
@pytest.mark.parametrize("trans", [False, True])
def test_split_h2_roundtrip(ops, scale, trans):
    g = torch.Generator(device="cuda").manual_seed(11)
    x = torch.randn(300, 197, generator=g, device="cuda") * scale
    x[3, 5] = 0.0
    sp = ops.split_h2(x, trans=trans)
    e = int(sp.e[0].item())
    amax = x.abs().max().item()
    assert 2.0 ** 14 <= amax * 2.0 ** e < 2.0 ** 15
    rec = (sp.hi[:, :sp.cols].double() + sp.lo[:, :sp.cols].double()) * 2.0 ** -e
    src = x.double().T if trans else x.double()
    assert rec.shape == src.shape
    # per element: |x - rec| <= 2^-22 |x| + the fp16 subnormal floor (2^-25 of 2^15)
    err = (rec - src).abs()
    assert (err <= 2.0 ** -22 * src.abs() + 2.0 ** (-25 - e)).all()


def test_split_h2_inplace_matches(ops):
    g = torch.Generator(device="cuda").manual_seed(12)
    x = ops.empty2d(301, 133, torch.float32, "cuda")
    x.copy_(torch.randn(301, 133, generator=g, device="cuda") * 5e3)
    ref = ops.split_h2(x)
    sp = ops.split_h2_inplace(x)
    assert int(sp.e[0].item()) == int(ref.e[0].item())
    assert torch.equal(sp.hi, ref.hi[:, :133]) and torch.equal(sp.lo, ref.lo[:, :133])
    assert sp.hi.data_ptr() == x.data_ptr() and sp.ld == 2 * x.stride(0)


def test_split_h2_zero(ops):
    sp = ops.split_h2(torch.zeros(5, 9, device="cuda"))
    assert int(sp.e[0].item()) == 0
    assert sp.hi[:, :9].abs().max().item() == 0 and sp.lo[:, :9].abs().max().item() == 0


@pytest.mark.parametrize("ta", [0, 1])
@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (67, 45, 131), (128, 16, 64), (300, 520, 4000),
                                   (1000, 110, 2000), (4000, 520, 65536), (257, 176, 1000)])
def test_gemm_h3_vs_torch(ops, ta, M, N, K):
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N + K)
    a = torch.randn((K, M) if ta else (M, K), generator=g, device="cuda") * 3.0
    b = torch.randn(K, N, generator=g, device="cuda") * 1e-3
    sa = ops.split_h2(a)
    sb = ops.split_h2(b, trans=True)   # B^T (N x K, K-major)
    ref = (a.double().T if ta else a.double()) @ b.double()
    c0 = torch.randn(M, N, generator=g, device="cuda")
    out = c0.clone()
    ops.gemm_h3(sa, sb, ta=bool(ta), alpha=0.5, beta=2.0, out=out)
    expect = 0.5 * ref + 2.0 * c0.double()
    scale = (a.double().abs().max() * b.double().abs().max() * np.sqrt(K)).item()
    # 2^-22 per product, fp32 accumulation: the same bound as the 3xTF32 test
    assert (out.double() - expect).abs().max().item() <= 2e-6 * scale + 1e-6


@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (67, 45, 131), (300, 520, 4000), (16384, 520, 20000),
                                   (257, 176, 1000)])
def test_gemm_h3s_vs_torch(ops, M, N, K):
    """In-kernel split of an fp32 A^T operand (randsvd's B^T = A^T Q)."""
    g = torch.Generator(device="cuda").manual_seed(M + 3 * N + K)
    a = ops.empty2d(K, M, torch.float32, "cuda")
    a.copy_(torch.randn(K, M, generator=g, device="cuda") * 7.0)
    b = torch.randn(K, N, generator=g, device="cuda") * 1e-2
    e_a = ops.h2_exponent(a)
    assert 2.0 ** 14 <= a.abs().max().item() * 2.0 ** int(e_a[0].item()) < 2.0 ** 15
    ovf = torch.zeros(1, dtype=torch.int32, device="cuda")
    c0 = torch.randn(M, N, generator=g, device="cuda")
    out = c0.clone()
    ops.gemm_h3s_t(a, e_a, ops.split_h2(b, trans=True), alpha=0.5, beta=2.0, out=out, overflow=ovf)
    assert int(ovf.item()) == 0
    expect = 0.5 * (a.double().T @ b.double()) + 2.0 * c0.double()
    scale = (a.double().abs().max() * b.double().abs().max() * np.sqrt(K)).item()
    assert (out.double() - expect).abs().max().item() <= 2e-6 * scale + 1e-6


def test_gemm_h3s_overflow_flag_and_fallback(ops):
    g = torch.Generator(device="cuda").manual_seed(1)
    a = ops.empty2d(4096, 2048, torch.float32, "cuda")
    a.copy_(torch.randn(4096, 2048, generator=g, device="cuda"))
    q = torch.randn(4096, 64, generator=g, device="cuda")
    be = ops.CudaBackend("cuda", torch.float32)
    # a hint far below the true max: the kernel flags it ...
    e_io = torch.zeros(2, dtype=torch.int32, device="cuda")
    e_io[1] = torch.tensor([1e-6], dtype=torch.float32).view(torch.int32).item()
    be.mm_at_big(a, q, (e_io, 0))
    assert be.overflowed()
    # ... and the engine recomputes with 3xTF32
    from paper_2605_09755_b200 import _engine
    u, s, v = _engine.randsvd(be, _engine.LOCAL, a, torch.linalg.qr(q)[0].contiguous(), False,
                              (e_io, 0))
    ref = torch.linalg.svdvals((torch.linalg.qr(q.double())[0].T @ a.double()))
    assert (s.cpu() - ref.cpu()).abs().max().item() <= 1e-5 * ref.max().item()


def test_h3_long_k_accumulation_is_unbiased(ops):
    """The tensor core's fp32 accumulation truncates: one 262144-deep chain of
    positive products comes out ~3e-5 low (3xTF32 in one chain: ~8e-5).  The
    3xFP16 kernels sum 1024-deep chunks in registers (round to nearest)."""
    K, M, N = 262144, 256, 64
    g = torch.Generator(device="cuda").manual_seed(0)
    a = ops.empty2d(K, M, torch.float32, "cuda")
    a.copy_(torch.rand(K, M, generator=g, device="cuda") + 0.5)
    q = torch.rand(K, N, generator=g, device="cuda") + 0.5
    ref = a.double().T @ q.double()
    sq = ops.split_h2(q, trans=True)
    for out in (ops.gemm_h3s_t(a, ops.h2_exponent(a), sq), ops.gemm_h3(ops.split_h2(a), sq, ta=True)):
        rel = (out.double() - ref) / ref
        assert abs(rel.mean().item()) < 1e-5 and rel.abs().max().item() < 2e-5


def test_accurate_gram_orthonormal_basis(ops):
    """The Gram of the last CholeskyQR pass (accurate=True) is unbiased at
    K = 262144, so the final basis is orthonormal to ~1e-5."""
    g = torch.Generator(device="cuda").manual_seed(2)
    y = ops.empty2d(262144, 96, torch.float32, "cuda")
    y.copy_(torch.randn(262144, 96, generator=g, device="cuda") + 0.3)
    be = ops.CudaBackend("cuda", torch.float32)
    ref = y.double().T @ y.double()
    g64 = be.gram64(y, accurate=True)
    rel = (torch.diagonal(g64) - torch.diagonal(ref)) / torch.diagonal(ref)
    assert rel.abs().max().item() < 1e-5


@pytest.mark.parametrize("N,K", [(1, 1), (45, 131), (128, 64), (300, 5000), (520, 4000),
                                 (1000, 20000), (1111, 3000), (4000, 8192)])
def test_syrk_h3_vs_torch(ops, N, K):
    """K4h SYRK (the sketch-space power iteration's G = A~^T A~): both
    operands MN-major from one set of planes, lower-triangle tiles only,
    mirrored -- exactly symmetric, 3xFP16 accuracy against fp64."""
    g = torch.Generator(device="cuda").manual_seed(N + 7 * K)
    a = torch.randn(K, N, generator=g, device="cuda") * 2.0 + 0.1
    out = ops.syrk_h3(ops.split_h2(a), alpha=0.5)
    ref = 0.5 * (a.double().T @ a.double())
    assert torch.equal(out, out.T)
    # 2^-22 per product plus the fp32 accumulation of 1024-deep chunks, whose
    # truncation on the positive diagonal (sums of squares) is ~1e-5 of
    # sum |a_ki a_kj| (test_h3_long_k_accumulation_is_unbiased)
    ab = a.double().abs()
    bound = 0.5 * (2e-5 * (ab.T @ ab) + 2e-6 * ab.max().item() ** 2 * np.sqrt(K))
    assert bool(((out.double() - ref).abs() <= bound + 1e-6).all())


@pytest.mark.parametrize("N,K", [(45, 1000), (130, 5000), (520, 262144), (1050, 65536)])
def test_syrk_h3_rows_vs_torch(ops, N, K):
    """The K-major SYRK (Y^T Y from the planes of Y^T: the CholeskyQR Grams),
    with split-K when the lower-triangle tiles are fewer than the CTA pairs."""
    g = torch.Generator(device="cuda").manual_seed(N * 3 + K)
    y = torch.randn(K, N, generator=g, device="cuda") + 0.2
    out = ops.syrk_h3(ops.split_h2(y, trans=True), rows=True)
    ref = y.double().T @ y.double()
    assert torch.equal(out, out.T)
    ab = y.double().abs()
    bound = 2e-5 * (ab.T @ ab) + 2e-6 * ab.max().item() ** 2 * np.sqrt(K)
    assert bool(((out.double() - ref).abs() <= bound + 1e-6).all())


@pytest.mark.parametrize("M,N,K", [(3000, 520, 520), (70000, 1050, 1050), (300, 130, 130)])
def test_gemm_h3_emit_lower_triangular_b(ops, M, N, K):
    """Q^T = (Y X^T)^T with X lower triangular (b_lower): the N tiles stop at
    their K extent; same result as the dense product."""
    g = torch.Generator(device="cuda").manual_seed(M + N)
    y = torch.randn(M, K, generator=g, device="cuda")
    x = torch.tril(torch.randn(N, K, generator=g, device="cuda"))
    yt = ops.split_h2(y, trans=True)
    xs = ops.split_h2(x)
    dense = ops.gemm_h3_emit_t(yt, xs, ta=True)
    tri = ops.gemm_h3_emit_t(yt, xs, ta=True, b_lower=True)
    def val(p):
        return ((p.hi.float() + p.lo.float())[:, :p.cols] * 2.0 ** -int(p.e[0].item())).double()
    ref = (y.double() @ x.double().T).T
    scale = (y.abs().max() * x.abs().max()).item() * np.sqrt(K)
    assert (val(tri) - ref).abs().max().item() <= 4e-6 * scale
    assert torch.equal(val(tri), val(dense))


def test_syrk_h3_inplace_planes_long_k(ops):
    """The power iteration's operand: A~ split in place (planes with leading
    dimension 2 ld) and K = 262144 rows (register-promoted accumulation:
    the diagonal of G = sums of squares is unbiased)."""
    K, N = 262144, 640
    g = torch.Generator(device="cuda").manual_seed(5)
    x = ops.empty2d(K, N, torch.float32, "cuda")
    x.copy_(torch.randn(K, N, generator=g, device="cuda"))
    ref = x.double().T @ x.double()
    out = ops.syrk_h3(ops.split_h2_inplace(x))
    rel = (torch.diagonal(out).double() - torch.diagonal(ref)) / torch.diagonal(ref)
    assert abs(rel.mean().item()) < 1e-5 and rel.abs().max().item() < 2e-5
    assert (out.double() - ref).abs().max().item() <= 2e-5 * torch.diagonal(ref).max().item()


# ----------------------------------------------------------- K5 / K6 ------

def _spd(n, cond=1e4, seed=0):
    rng = np.random.default_rng(seed)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    w = np.logspace(0, -np.log10(cond), n)
    return (q * w) @ q.T


@pytest.mark.parametrize("n", [1, 2, 63, 64, 65, 130, 520, 1050])
def test_cholesky_and_trinv(n):
    from paper_2605_09755_b200 import _lib
    from paper_2605_09755_b200._ops import ptr
    g = _spd(n, seed=n)
    t = torch.from_numpy(g).cuda()
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    _lib.call("skp_cholesky_f64", ptr(t), n, n, ptr(info), st)
    assert int(info.item()) == 0
    lmat = np.tril(t.cpu().numpy())
    np.testing.assert_allclose(lmat, np.linalg.cholesky(g), rtol=0, atol=1e-10)
    x = torch.empty_like(t)
    _lib.call("skp_trinv_lower_f64", ptr(t), n, n, ptr(x), st)
    np.testing.assert_allclose(x.cpu().numpy() @ lmat, np.eye(n), atol=1e-8)


def test_cholesky_reports_indefinite():
    from paper_2605_09755_b200 import _lib
    from paper_2605_09755_b200._ops import ptr
    g = _spd(100)
    g[70, 70] = -1.0
    t = torch.from_numpy(g).cuda()
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    _lib.call("skp_cholesky_f64", ptr(t), 100, 100, ptr(info), torch.cuda.current_stream().cuda_stream)
    assert int(info.item()) > 0


@pytest.mark.parametrize("n", [1, 2, 3, 30, 111, 112, 113, 300, 520, 641, 700, 1050, 1500])
def test_jacobi_eigensolver(n):
    from paper_2605_09755_b200._ops import CudaBackend
    rng = np.random.default_rng(n)
    b = rng.standard_normal((n, 3 * n + 1))
    g = b @ b.T
    be = CudaBackend(torch.device("cuda", 0), torch.float64)
    w, v = be.eig_desc64(torch.from_numpy(g).cuda())
    w, v = w.cpu().numpy(), v.cpu().numpy()
    ref = np.sort(np.linalg.eigvalsh(g))[::-1]
    np.testing.assert_allclose(w, ref, rtol=1e-11, atol=1e-11 * ref[0])
    np.testing.assert_allclose(v.T @ v, np.eye(n), atol=1e-11)
    np.testing.assert_allclose(g @ v, v * w, atol=1e-9 * ref[0])


@pytest.mark.parametrize("n", [1, 5, 32, 33, 64, 110, 520, 1050])
def test_fused_cholinv(n):
    from paper_2605_09755_b200 import _lib
    from paper_2605_09755_b200._ops import ptr, workspace
    g = _spd(n, cond=1e6, seed=n)
    t = torch.from_numpy(g).cuda()
    x = torch.empty_like(t)
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    wsb = _lib.load().skp_cholinv_ws_bytes(n)
    ws = workspace(t.device, wsb)
    _lib.call("skp_cholinv_f64", ptr(t), n, n, 1e-9, 0.0, ptr(x), ptr(info), ptr(ws), wsb,
              torch.cuda.current_stream().cuda_stream)
    assert int(info.item()) == 0
    xi = x.cpu().numpy()
    lmat = np.linalg.cholesky(g)
    np.testing.assert_allclose(xi @ lmat, np.eye(n), atol=1e-7)
    assert np.all(np.triu(xi, 1) == 0)
    # shifted factorisation (first pass of shifted CholeskyQR3): G + 1e-3 max G_ii I
    _lib.call("skp_cholinv_f64", ptr(t), n, n, 0.0, 1e-3, ptr(x), ptr(info), ptr(ws), wsb,
              torch.cuda.current_stream().cuda_stream)
    assert int(info.item()) == 0
    ls = np.linalg.cholesky(g + 1e-3 * np.diag(g).max() * np.eye(n))
    np.testing.assert_allclose(x.cpu().numpy() @ ls, np.eye(n), atol=1e-9)
    # rank check and indefinite detection
    g2 = g.copy()
    g2[n // 2, n // 2] = -1.0 if n > 1 else -1.0
    t2 = torch.from_numpy(g2).cuda()
    _lib.call("skp_cholinv_f64", ptr(t2), n, n, 1e-9, 0.0, ptr(x), ptr(info), ptr(ws), wsb,
              torch.cuda.current_stream().cuda_stream)
    assert int(info.item()) != 0


# ---------------------------------------------------------------- Omega ----

@pytest.mark.parametrize("rows,cols,seed", [(4000, 520, 1), (2000, 110, 2), (13, 7, 5),
                                            (8000, 1050, 3), (1, 1, 9)])
def test_gaussian_omega_matches_numpy(ops, rows, cols, seed):
    """Device Omega == numpy's standard_normal((rows, cols)) / sqrt(cols): the
    fp32 matrix bit for bit; fp64 to 1 ulp (CUDA's log1p in a few tail values)."""
    import math
    from paper_2605_09755_b200.sketching import _host_rng, pcg64_state
    st, inc = pcg64_state(seed)
    fail = torch.zeros(1, dtype=torch.int64, device="cuda")
    g32 = ops.gaussian(st, inc, rows, cols, math.sqrt(cols), torch.float32, "cuda", fail)
    g64 = ops.gaussian(st, inc, rows, cols, math.sqrt(cols), torch.float64, "cuda", fail)
    ref = _host_rng(seed).standard_normal((rows, cols)) / math.sqrt(cols)
    assert int(fail.item()) == 0
    np.testing.assert_array_equal(g32.cpu().numpy(), ref.astype(np.float32))
    d64 = g64.cpu().numpy()
    ulp = np.spacing(np.abs(ref))
    assert (np.abs(d64 - ref) <= ulp).all()
    assert np.count_nonzero(d64 != ref) <= max(3, rows * cols // 100000)


@pytest.mark.parametrize("k,c", [(16384, 520), (1000, 130), (37, 5), (262144, 64)])
def test_gram_f32_f64(ops, k, c):
    """G = X^T X in fp64 from fp32 X: exact products, fp64 sums (randsvd's B B^T)."""
    rng = np.random.default_rng(k + c)
    x = rng.standard_normal((k, c)).astype(np.float32)
    t = ops.empty2d(k, c, torch.float32, "cuda")
    t.copy_(torch.from_numpy(x))
    be = ops.CudaBackend(torch.device("cuda", 0), torch.float32)
    g = be.gram64_rows_t(t).cpu().numpy()
    ref = x.astype(np.float64).T @ x.astype(np.float64)
    assert np.abs(g - ref).max() <= 1e-13 * np.abs(ref).max()
    np.testing.assert_array_equal(g, g.T)


def test_srht_range_finder_exact_rank(skp):
    """The SRHT sketch inside the range finder: an exactly rank-8 matrix is
    recovered (sigma to 1e-10 in fp64), as with the other sketch kinds."""
    rng = np.random.default_rng(3)
    u = np.linalg.qr(rng.standard_normal((300, 8)))[0]
    v = np.linalg.qr(rng.standard_normal((200, 8)))[0]
    s = np.linspace(3.0, 1.0, 8)
    a = (u * s) @ v.T
    spec = skp.RangeFinderSpec(k=8, l=40, r1=40, r2=12, q=1, eps=0.5, sketch_kind="srht", seed=4)
    q = skp.range_finder_sketched(a, spec)
    res = skp.randsvd(a, q)
    np.testing.assert_allclose(np.asarray(res.sigma)[:8], s, rtol=0, atol=1e-10)
