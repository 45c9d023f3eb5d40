"""Generate the golden fixtures under tests/golden/ from the LIVE reference.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``skpower`` from /root/reference/pkg/src (read-only; no bytecode is
written there) and records its outputs:

* ``substream`` values and the PCG64 (state, inc) that ``_rng`` seeds;
* CountSketch ``_cols`` / ``_signs`` of ``make_sketch("countsketch", ...)``:
  full arrays for small cases, sha256 digests for the BASELINE config shapes;
* end-to-end C1 (fp64) and C2 (fp32 input, q = 1, 2, 3) ``range_finder_sketched``
  + ``randsvd`` singular values and relative projection errors;
* a small literal ``nystrom_psd`` run (RBF kernel, n = 2048).

Nothing here runs on the GPU box; the fixtures travel, the reference does not.
"""
from __future__ import annotations

import hashlib
import json
import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import skpower  # noqa: E402  (the reference)
from skpower import data_io as ref_io  # noqa: E402
from skpower.power import RangeFinderSpec, nystrom_psd, randsvd, range_finder_sketched  # noqa: E402
from skpower.sketching import _rng, make_sketch, substream  # noqa: E402

from paper_2605_09755_b200 import datagen  # noqa: E402

SMALL_CS = [  # (n, r, s, seed)
    (4, 2, 1, 5), (40, 12, 4, 6), (200, 40, 4, 21), (60, 16, 2, 31), (20, 7, 3, 11),
    (500, 97, 3, 7), (300, 64, 1, 9), (1000, 37, 1, 123), (257, 33, 8, 77),
    (1000, 200, 8, None),  # C1 primary sketch: seed = substream(1, 0)
    (1000, 3_000_000_000, 1, 17),  # s=1 with frequent Lemire rejections
    (64, 64, 64, 3), (50, 40, 33, 8), (33, 1000, 17, 12),
    # s=1 with an odd number of 32-bit column draws: the first sign is the
    # high half PCG64 kept buffered from the column phase
    (513, 64, 1, 13), (1025, 64, 1, 5), (7, 3, 1, 1), (999, 37, 1, 77), (2049, 2, 1, 10),
]
# BASELINE config shapes; seed = substream(config spec seed, 0)
BIG_CS = {
    "C2": (10000, 2000, 8, 2), "C3": (16384, 4000, 8, 3), "C4": (65536, 4096, 8, 4),
    "C5_l4000": (32768, 4000, 8, 5), "C5_l8000": (32768, 8000, 8, 5), "C5_l16000": (32768, 16000, 8, 5),
}


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    t0 = time.time()
    meta = {"numpy": np.__version__, "reference": "skpower " + skpower.__version__,
            "generated_by": "tests/golden/make_golden.py"}
    import scipy
    meta["scipy"] = scipy.__version__

    # --- seeds ---------------------------------------------------------
    subs = []
    for seed, idx in [(0, (0,)), (0, (1,)), (1, (0,)), (1, (1,)), (123, (0,)), (2**64 - 1, (2, 5)),
                      (42, ()), (7, (3, 1, 4))]:
        subs.append({"seed": seed, "idx": list(idx), "value": str(substream(seed, *idx))})
    states = []
    for seed in [0, 1, 17, substream(3, 0), 2**63 + 5]:
        g = _rng(seed)
        st = g.bit_generator.state["state"]
        raw = g.bit_generator.random_raw(16)
        states.append({"seed": str(seed), "state": str(st["state"]), "inc": str(st["inc"]),
                       "raw16": [str(int(x)) for x in raw]})

    # --- CountSketch ---------------------------------------------------
    small = {}
    for i, (n, r, s, seed) in enumerate(SMALL_CS):
        seed = substream(1, 0) if seed is None else seed
        op = make_sketch("countsketch", n, r, seed, s=s)
        small[f"cs{i}_cols"] = np.asarray(op._cols, dtype=np.int64)
        small[f"cs{i}_signs"] = np.asarray(op._signs, dtype=np.int8)
        small[f"cs{i}_params"] = np.array([n, r, s, seed], dtype=np.uint64)
    big = {}
    for name, (n, r, s, cfg_seed) in BIG_CS.items():
        seed = substream(cfg_seed, 0)
        op = make_sketch("countsketch", n, r, seed, s=s)
        big[name] = {"n": n, "r": r, "s": s, "seed": str(seed),
                     "cols_sha256": sha(np.asarray(op._cols, dtype=np.int64)),
                     "signs_sha256": sha(np.asarray(op._signs, dtype=np.int8)),
                     "cols_head": np.asarray(op._cols[:4], dtype=np.int64).tolist()}
        del op
        print(name, "done", round(time.time() - t0, 1), flush=True)

    # --- end to end C1 (fp64) -------------------------------------------
    a1 = ref_io._rotate_spectrum(2000, 1000, 1.0 / np.arange(1.0, 1001.0), 1)
    assert np.array_equal(a1, datagen.c1_matrix(1)), "datagen.c1_matrix != reference generator"
    spec1 = RangeFinderSpec(k=20, l=200, r1=200, r2=30, q=2, eps=0.5, sketch_kind="countsketch",
                            seed=1, s=8)
    q1 = range_finder_sketched(a1, spec1)
    _, s1, _ = randsvd(a1, q1)
    e1 = float(np.linalg.norm(a1 - q1 @ (q1.T @ a1)) / np.linalg.norm(a1))
    c1 = {"sha256_A": sha(a1), "sigma": s1.tolist(), "rel_err": e1, "rank": int(q1.shape[1]),
          "spec": dict(k=20, l=200, r1=200, r2=30, q=2, s=8, seed=1)}

    # --- end to end C2 (fp32 input; the reference computes in fp64) -----
    a2 = datagen.c2_matrix(2)
    c2 = {"sha256_A": sha(a2), "runs": {}}
    for q in (1, 2, 3):
        spec2 = RangeFinderSpec(k=100, l=2000, r1=2000, r2=110, q=q, eps=0.5,
                                sketch_kind="countsketch", seed=2, s=8)
        q2 = range_finder_sketched(a2, spec2)
        _, s2, _ = randsvd(a2, q2)
        a2d = a2.astype(np.float64)
        e2 = float(np.linalg.norm(a2d - q2 @ (q2.T @ a2d)) / np.linalg.norm(a2d))
        c2["runs"][str(q)] = {"sigma": s2.tolist(), "rel_err": e2, "rank": int(q2.shape[1])}
        print("C2 q", q, "done", round(time.time() - t0, 1), flush=True)

    # --- literal Nystrom, small RBF -------------------------------------
    x = datagen.rbf_points(2048, 16, seed=4)
    h = datagen.rbf_bandwidth(x, 2048, seed=4)
    sq = (x * x).sum(1)
    kmat = np.exp(-np.maximum(sq[:, None] + sq[None, :] - 2 * x @ x.T, 0) / (2 * h * h))
    kmat = (kmat + kmat.T) / 2
    specn = RangeFinderSpec(k=32, l=256, r1=256, r2=32, q=2, eps=0.5, sketch_kind="countsketch",
                            seed=4, s=8)
    res = nystrom_psd(kmat, specn)
    from skpower.linalg import pinv
    en = float(np.linalg.norm(kmat - res.C @ pinv(res.W) @ res.C.T) / np.linalg.norm(kmat))
    nys = {"n": 2048, "h": h, "rel_err_literal": en,
           "W_eigs": np.linalg.eigvalsh(res.W).tolist(),
           "spec": dict(k=32, l=256, r1=256, r2=32, q=2, s=8, seed=4)}

    np.savez_compressed(os.path.join(HERE, "countsketch_small.npz"), **small)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump({"meta": meta, "substream": subs, "pcg64": states, "countsketch_big": big,
                   "C1": c1, "C2": c2, "nystrom_small": nys}, f, indent=1)
    print("wrote fixtures in", round(time.time() - t0, 1), "s")


if __name__ == "__main__":
    main()
