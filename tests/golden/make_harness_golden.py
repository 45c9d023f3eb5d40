"""Golden records for the device harness (paper_2605_09755_b200.harness):
the reference's own benchmark protocol (skpower.bench.run_benchmark) run in
this container on two small configs.  Writes tests/golden/harness_*.csv.

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \\
        python tests/golden/make_harness_golden.py
"""
import os
import sys
import tempfile

import numpy as np

import skpower.bench as rb
from skpower import data_io

HERE = os.path.dirname(os.path.abspath(__file__))


def psd_matrix(n: int = 120, seed: int = 11) -> np.ndarray:
    rng = np.random.default_rng(seed)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    w = 1.0 / np.arange(1.0, n + 1.0) ** 1.5
    a = (q * w) @ q.T
    return (a + a.T) / 2.0


def main():
    cfg = rb.config_from_mapping({
        "dataset": "polydecay:300x200:seed=7", "label": "poly",
        "methods": "classical-randsvd,sketched-randsvd,lowrank-factorize,lowrank-factorize-unsketched",
        "k": "5", "l_values": "10 20", "trials": "2", "q_max": "3", "root_seed": "3",
        "sketch_kind": "countsketch", "s": "2", "workers": "1"})
    rb.run_benchmark(cfg, os.path.join(HERE, "harness_poly.csv"))
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "psd.skpw")
        a = psd_matrix()
        data_io.write_binary(a, path)
        np.save(os.path.join(HERE, "harness_psd_matrix.npy"), a)
        cfg = rb.config_from_mapping({
            "dataset": path, "label": "psd", "methods": "nystrom", "k": "4",
            "l_values": "12", "trials": "2", "q_max": "2", "root_seed": "5",
            "sketch_kind": "countsketch", "s": "2", "workers": "1"})
        rb.run_benchmark(cfg, os.path.join(HERE, "harness_psd.csv"))
    print("ok")


if __name__ == "__main__":
    sys.exit(main())
