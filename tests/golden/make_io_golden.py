"""Golden files for the device readers (paper_2605_09755_b200.io), written and
read back by the reference's own data_io in this container:
tests/golden/io_*.{skpw,mtx} and io_expected.npz.

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \\
        python tests/golden/make_io_golden.py
"""
import os

import numpy as np

from skpower import data_io

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    rng = np.random.default_rng(17)
    a = rng.standard_normal((37, 23))
    s = rng.standard_normal((9, 9))
    s = s + s.T
    out = {}
    data_io.write_binary(a, os.path.join(HERE, "io_a.skpw"))
    out["skpw"] = data_io.read_binary(os.path.join(HERE, "io_a.skpw"))
    data_io.write_matrix_market(a[:7, :5], os.path.join(HERE, "io_array_general.mtx"))
    out["array_general"] = data_io.read_matrix_market(os.path.join(HERE, "io_array_general.mtx"))
    data_io.write_matrix_market(s, os.path.join(HERE, "io_array_symmetric.mtx"), symmetric=True)
    out["array_symmetric"] = data_io.read_matrix_market(os.path.join(HERE, "io_array_symmetric.mtx"))
    with open(os.path.join(HERE, "io_coord_general.mtx"), "w") as fh:
        fh.write("%%MatrixMarket matrix coordinate real general\n% a comment\n\n6 4 5\n")
        fh.write("1 1 1.5\n6 4 -2.25\n3 2 7e-3\n% inline comment\n2 4 1e10\n5 1 -0.125\n")
    out["coord_general"] = data_io.read_matrix_market(os.path.join(HERE, "io_coord_general.mtx"))
    with open(os.path.join(HERE, "io_coord_symmetric.mtx"), "w") as fh:
        fh.write("%%MatrixMarket matrix coordinate real symmetric\n5 5 4\n")
        fh.write("1 1 2.0\n3 1 -1.0\n5 4 0.5\n4 4 3.0\n")
    out["coord_symmetric"] = data_io.read_matrix_market(os.path.join(HERE, "io_coord_symmetric.mtx"))
    np.savez(os.path.join(HERE, "io_expected.npz"), **out)
    print("ok")


if __name__ == "__main__":
    main()
