"""Pin the CPU oracle (oracle/) against the live-reference golden fixtures.

tests/golden/make_golden.py recorded these from /root/reference itself; here
both restatements (plain C and numpy) must reproduce them bit for bit
(integer/index work) or to fp64 rounding (end-to-end C1).
"""
import hashlib
import os

import numpy as np
import pytest

from conftest import GOLDEN, small_cs_cases
from oracle import skp_oracle as o
from paper_2605_09755_b200 import datagen


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_substream(golden):
    for s in golden["substream"]:
        assert o.substream(s["seed"], *s["idx"]) == int(s["value"])


def test_pcg64_state_and_raw_draws(golden):
    for st in golden["pcg64"]:
        S, I = o.pcg64_state(int(st["seed"]))
        assert (S, I) == (int(st["state"]), int(st["inc"]))
        raw = o.pcg64_raw_c(S, I, 16)
        assert [str(int(x)) for x in raw] == st["raw16"]


def test_pcg64_jump_ahead_composes(golden):
    S, I = o.pcg64_state(17)
    assert o.pcg64_advance_c(S, I, 1000) == o.pcg64_advance_c(o.pcg64_advance_c(S, I, 333), I, 667)
    raw = o.pcg64_raw_c(o.pcg64_advance_c(S, I, 5), I, 1)
    assert raw[0] == o.pcg64_raw_c(S, I, 6)[5]


def test_countsketch_small_c_and_numpy(golden_cs):
    for i, n, r, s, seed in small_cs_cases(golden_cs):
        cols, signs = o.countsketch_c(seed, n, r, s)
        np.testing.assert_array_equal(cols, golden_cs[f"cs{i}_cols"])
        np.testing.assert_array_equal(signs.astype(np.int8), golden_cs[f"cs{i}_signs"])
        if r < 10**6:
            c2, s2 = o.countsketch_numpy(seed, n, r, s)
            np.testing.assert_array_equal(c2, golden_cs[f"cs{i}_cols"])


@pytest.mark.parametrize("name", ["C2", "C3", "C5_l4000", "C5_l8000"])
def test_countsketch_config_shapes_c(golden, name):
    b = golden["countsketch_big"][name]
    cols, signs = o.countsketch_c(int(b["seed"]), b["n"], b["r"], b["s"])
    assert sha(cols) == b["cols_sha256"]
    assert sha(signs.astype(np.int8)) == b["signs_sha256"]


def test_c1_generator_matches_reference(golden):
    a = datagen.c1_matrix(1)
    assert sha(a) == golden["C1"]["sha256_A"]


def test_c1_oracle_end_to_end(golden):
    g = golden["C1"]
    a = datagen.c1_matrix(1)
    spec = o.Spec(k=20, l=200, r1=200, r2=30, q=2, seed=1, s=8)
    qb = o.range_finder_sketched(a, spec)
    _, s, _ = o.randsvd(a, qb)
    np.testing.assert_allclose(s, g["sigma"], rtol=1e-12)
    assert abs(o.proj_rel_error(a, qb) - g["rel_err"]) <= 1e-12


def test_nystrom_literal_oracle(golden):
    g = golden["nystrom_small"]
    x = datagen.rbf_points(g["n"], 16, seed=4)
    h = datagen.rbf_bandwidth(x, g["n"], seed=4)
    assert abs(h - g["h"]) < 1e-12
    sq = (x * x).sum(1)
    k = np.exp(-np.maximum(sq[:, None] + sq[None, :] - 2 * x @ x.T, 0) / (2 * h * h))
    k = (k + k.T) / 2
    sp = g["spec"]
    spec = o.Spec(k=sp["k"], l=sp["l"], r1=sp["r1"], r2=sp["r2"], q=sp["q"], seed=sp["seed"], s=sp["s"])
    c, w = o.nystrom_core(k, spec, stabilized=False)
    np.testing.assert_allclose(np.linalg.eigvalsh(w), g["W_eigs"], rtol=1e-8,
                               atol=1e-10 * max(abs(x) for x in g["W_eigs"]))
    assert abs(o.nystrom_rel_error(k, c, w) - g["rel_err_literal"]) <= 1e-6


@pytest.mark.parametrize("seed", [0, 7, 2**40 + 3])
def test_ziggurat_restatement_matches_numpy(seed):
    """The ziggurat constants compiled into csrc/omega.cu reproduce numpy's
    standard_normal draw for draw (rectangles, wedges and the tail)."""
    from oracle import ziggurat
    n = 120_000
    ref = np.random.Generator(np.random.PCG64(seed)).standard_normal(n)
    raw = np.random.PCG64(seed).random_raw(n + n // 16 + 64)
    np.testing.assert_array_equal(ziggurat.standard_normal_from_raw(raw, n), ref)


def test_oracle_srht_matches_live_reference():
    """The oracle's SRHT (sketching.py:65-90, :125-130, :165-171, :183-189)
    against values recorded from the live reference."""
    g = np.load(os.path.join(GOLDEN, "srht_golden.npz"))
    for key in sorted({k.split("_", 1)[1] for k in g.files if k.startswith("signs_")}):
        n, r, seed = (int(v) for v in key.split("_"))
        op = o.CountSketch("srht", n, r, seed)
        np.testing.assert_array_equal(op.srht_signs, g[f"signs_{key}"])
        np.testing.assert_array_equal(op.subset, g[f"subset_{key}"])
        np.testing.assert_allclose(op.apply_right(g[f"a_{key}"]), g[f"right_{key}"], rtol=0, atol=1e-12)
        np.testing.assert_allclose(op.apply_left_transpose(g[f"x_{key}"]), g[f"left_{key}"], rtol=0,
                                   atol=1e-12)


def test_oracle_dense_sketches_match_live_reference():
    """gaussian / sign S (sketching.py:131-136) drawn bit for bit as the reference."""
    g = np.load(os.path.join(GOLDEN, "dense_sketch_golden.npz"))
    for key in g.files:
        kind, n, r, seed = key.split("_")
        op = o.CountSketch(kind, int(n), int(r), int(seed))
        np.testing.assert_array_equal(op.dense, g[key])
