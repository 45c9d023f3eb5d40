"""Device harness against the reference's own benchmark
records (tests/golden/make_harness_golden.py ran skpower.bench here)."""
import os

import numpy as np
import pytest

from paper_2605_09755_b200 import harness as H

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_records_csv_roundtrip(tmp_path):
    recs = H.read_records_csv(os.path.join(GOLD, "harness_poly.csv"))
    assert len(recs) == 64 and recs[0].method == "classical-randsvd"
    out = tmp_path / "r.csv"
    H.write_records_csv(recs, out)
    assert out.read_bytes() == open(os.path.join(GOLD, "harness_poly.csv"), "rb").read()


def test_records_csv_rejects_bad_header(tmp_path):
    p = tmp_path / "bad.csv"
    p.write_text("method,dataset\nx,y\n")
    with pytest.raises(ValueError, match="header"):
        H.read_records_csv(p)


def test_config_validation():
    with pytest.raises(ValueError, match="unknown method"):
        H.BenchConfig(dataset="polydecay:10x10", methods=["nope"], k=2, l_values=[4]).validate()
    with pytest.raises(ValueError, match="l must be >= k"):
        H.BenchConfig(dataset="polydecay:10x10", methods=["nystrom"], k=5, l_values=[4]).validate()
    cfg = H.BenchConfig(dataset="x", methods=["nystrom", "classical-randsvd"], k=2, l_values=[4])
    assert cfg.q_max_for("nystrom") == 15 and cfg.q_max_for("classical-randsvd") == 5


def _compare(ours, ref):
    assert len(ours) == len(ref)
    for a, b in zip(ours, ref):
        for f in ("method", "m", "n", "k", "l", "r1", "r2", "s", "q_iter", "seed", "trial"):
            assert getattr(a, f) == getattr(b, f), (f, a, b)
        for f in ("spec_err", "frob_err"):
            assert abs(getattr(a, f) - getattr(b, f)) <= 1e-5 * abs(getattr(b, f)) + 1e-9, (f, a, b)
        assert abs(a.rel_err - b.rel_err) <= 1e-5 * (1.0 + abs(b.rel_err)), (a, b)
    series = {}
    for r in ours:
        key = (r.method, r.l, r.trial)
        assert r.time_ms >= series.get(key, 0.0)
        series[key] = r.time_ms


@pytest.mark.gpu
def test_harness_matches_reference_records(tmp_path):
    cfg = H.BenchConfig(dataset="polydecay:300x200:seed=7", label="poly",
                        methods=["classical-randsvd", "sketched-randsvd", "lowrank-factorize",
                                 "lowrank-factorize-unsketched"],
                        k=5, l_values=[10, 20], trials=2, q_max=3, root_seed=3, s=2)
    out = tmp_path / "ours.csv"
    ours = H.run_benchmark(cfg, str(out))
    assert H.read_records_csv(out) == ours
    _compare(ours, H.read_records_csv(os.path.join(GOLD, "harness_poly.csv")))


@pytest.mark.gpu
def test_harness_nystrom_matches_reference_records():
    a = np.load(os.path.join(GOLD, "harness_psd_matrix.npy"))
    cfg = H.BenchConfig(dataset="psd", label="psd", methods=["nystrom"], k=4, l_values=[12],
                        trials=2, q_max=2, root_seed=5, s=2)
    _compare(H.run_benchmark(cfg, a=a), H.read_records_csv(os.path.join(GOLD, "harness_psd.csv")))
