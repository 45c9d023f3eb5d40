"""TEST INFRASTRUCTURE ONLY -- a plain restatement of numpy's
Generator.standard_normal (the 256-layer ziggurat, Marsaglia & Tsang 2000, as
numpy 2.3.5 lays it out) over an explicit array of raw PCG64 draws, using the
constants in tests/golden/ziggurat_tables.npz (recovered from numpy by
scripts/gen_ziggurat.py, the same constants compiled into csrc/omega.cu).
Pinning this against numpy itself pins those constants.

Only tests/ may import this module.
"""
import math
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_TABLES = os.path.join(_HERE, "..", "tests", "golden", "ziggurat_tables.npz")


def tables():
    z = np.load(_TABLES)
    return z["w"], z["k"].astype(np.uint64), z["f"], float(z["r"]), float(z["inv_r"])


def standard_normal_from_raw(raw: np.ndarray, count: int) -> np.ndarray:
    """The first `count` normals numpy draws from the 64-bit outputs `raw`."""
    w, k, f, r, inv_r = tables()
    out = np.empty(count)
    p, n = 0, 0
    while n < count:
        d = int(raw[p])
        p += 1
        idx = d & 0xFF
        d >>= 8
        sign = d & 1
        rabs = (d >> 1) & 0x000FFFFFFFFFFFFF
        x = rabs * w[idx]
        if sign:
            x = -x
        if rabs < int(k[idx]):
            out[n] = x
            n += 1
            continue
        if idx == 0:
            while True:
                xx = -inv_r * math.log1p(-((int(raw[p]) >> 11) * 2.0 ** -53))
                yy = -math.log1p(-((int(raw[p + 1]) >> 11) * 2.0 ** -53))
                p += 2
                if yy + yy > xx * xx:
                    out[n] = -(r + xx) if ((rabs >> 8) & 1) else (r + xx)
                    n += 1
                    break
        else:
            u = (int(raw[p]) >> 11) * 2.0 ** -53
            p += 1
            if (f[idx - 1] - f[idx]) * u + f[idx] < math.exp(-0.5 * x * x):
                out[n] = x
                n += 1
    return out
