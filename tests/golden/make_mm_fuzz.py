"""Golden MatrixMarket cases from the LIVE reference reader (run in the
container that has /root/reference; the GPU box never reads it):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_mm_fuzz.py

Writes tests/golden/mm_fuzz.json: seeded random well-formed and malformed
files (array / coordinate, general / symmetric; bad tokens, wrong counts,
out-of-range indices, short lines, comments, blank lines, repeated
coordinates) with the reference's outcome -- the matrix, or the ValueError
message with its line number (data_io.read_matrix_market, data_io.py:99-206).
"""
import json
import os
import random

import numpy as np
from skpower import data_io

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "mm_fuzz.json")
BAD = ["0", "-1", "x", "nan", "inf", "1e3", "+2", "1_0", "%c", "2 1", "1 1 1 1", "4"]


def case(rng):
    kind = rng.choice(["array", "coordinate"])
    sym = rng.choice(["general", "symmetric"])
    lines = [f"%%MatrixMarket matrix {kind} real {sym}"]
    if rng.random() < 0.2:
        lines.append("% comment")
    r, c = rng.randint(1, 3), rng.randint(1, 3)
    if sym == "symmetric" and rng.random() < 0.8:
        c = r
    if kind == "array":
        lines.append(f"{r} {c}" if rng.random() < 0.9 else rng.choice(["1", "a 2", "0 2", "2 2 2"]))
        nv = (r * c if sym == "general" else r * (r + 1) // 2) + rng.choice([0, 0, 0, 1, -1])
        vals = [rng.choice(["1.0", "2", "-3.5", "1e-3"]) if rng.random() < 0.93 else rng.choice(BAD)
                for _ in range(max(nv, 0))]
        while vals:
            k = rng.randint(1, 3)
            lines.append(" ".join(vals[:k]))
            vals = vals[k:]
            if rng.random() < 0.1:
                lines.append("")
    else:
        nnz = rng.randint(0, 5)
        lines.append(f"{r} {c} {nnz + rng.choice([0, 0, 0, 1, -1])}" if rng.random() < 0.9
                     else rng.choice(["1 1", "a 1 1", "1 1 -1"]))
        for _ in range(nnz):
            i, j = rng.randint(1, r), rng.randint(1, c)
            if rng.random() < 0.15:
                i, j = rng.randint(0, r + 1), rng.randint(0, c + 1)
            v = rng.choice(["1.5", "-2", "3e1"]) if rng.random() < 0.9 else rng.choice(BAD)
            f = [str(i), str(j), v]
            if rng.random() < 0.05:
                f = f[:2]
            if rng.random() < 0.05:
                f[0] = rng.choice(BAD)
            lines.append(" ".join(f))
    return "\n".join(lines) + ("\n" if rng.random() < 0.7 else "")


def main():
    rng = random.Random(2026)
    path = "/tmp/_mm_fuzz.mtx"
    cases = []
    for _ in range(600):
        text = case(rng)
        with open(path, "w") as fh:
            fh.write(text)
        try:
            m = data_io.read_matrix_market(path)
            cases.append({"text": text, "ok": True, "matrix": m.tolist()})
        except ValueError as e:
            msg = str(e)
            cases.append({"text": text, "ok": False,
                          "error": msg.split(path, 1)[1] if path in msg else msg})
    with open(OUT, "w") as fh:
        json.dump(cases, fh)
    print(len(cases), "cases,", sum(c["ok"] for c in cases), "ok")


if __name__ == "__main__":
    main()
