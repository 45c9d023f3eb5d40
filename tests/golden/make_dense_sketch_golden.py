"""Gaussian / sign sketch matrices from the live reference (this container
only): tests/golden/dense_sketch_golden.npz.

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \\
        python tests/golden/make_dense_sketch_golden.py
"""
import os

import numpy as np

from skpower.sketching import make_sketch

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = [("gaussian", 40, 7, 3), ("gaussian", 129, 33, 11), ("sign", 40, 7, 3), ("sign", 129, 33, 11)]


def main():
    out = {}
    for kind, n, r, seed in CASES:
        out[f"{kind}_{n}_{r}_{seed}"] = make_sketch(kind, n, r, seed).densify()
    np.savez_compressed(os.path.join(HERE, "dense_sketch_golden.npz"), **out)
    print("ok")


if __name__ == "__main__":
    main()
