"""SRHT golden values from the live reference (this container only):
tests/golden/srht_golden.npz.

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \\
        python tests/golden/make_srht_golden.py
"""
import os

import numpy as np

from skpower.sketching import make_sketch

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = [(50, 12, 9), (64, 64, 3), (1000, 37, 21), (3000, 300, 77)]


def main():
    out = {}
    rng = np.random.default_rng(5)
    for n, r, seed in CASES:
        op = make_sketch("srht", n, r, seed)
        key = f"{n}_{r}_{seed}"
        out[f"signs_{key}"] = op._signs
        out[f"subset_{key}"] = op._subset
        a = rng.standard_normal((3, n))
        x = rng.standard_normal((n, 3))
        out[f"a_{key}"] = a
        out[f"x_{key}"] = x
        out[f"right_{key}"] = op.apply_right(a)
        out[f"left_{key}"] = op.apply_left_transpose(x)
        if n * r <= 10**5:
            out[f"dense_{key}"] = op.densify()
    np.savez_compressed(os.path.join(HERE, "srht_golden.npz"), **out)
    print("ok")


if __name__ == "__main__":
    main()
