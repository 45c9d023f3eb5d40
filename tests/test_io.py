"""Direct-to-device ingestion against files written and
read by the reference's data_io (tests/golden/make_io_golden.py)."""
import os

import numpy as np
import pytest
import torch

from paper_2605_09755_b200 import io as skio

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_skpw_header_checks_without_gpu(tmp_path):
    assert skio.skpw_shape(os.path.join(GOLD, "io_a.skpw")) == (37, 23)
    p = tmp_path / "t.skpw"
    p.write_bytes(b"SKPW\x01" + b"\x00" * 5)
    with pytest.raises(ValueError, match="truncated header"):
        skio.skpw_shape(p)
    blob = open(os.path.join(GOLD, "io_a.skpw"), "rb").read()
    p.write_bytes(b"XKPW" + blob[4:])
    with pytest.raises(ValueError, match="bad magic"):
        skio.skpw_shape(p)
    p.write_bytes(blob[:4] + b"\x02" + blob[5:])
    with pytest.raises(ValueError, match="unsupported version 2"):
        skio.skpw_shape(p)
    p.write_bytes(blob[:-8])
    with pytest.raises(ValueError, match="expected"):
        skio.skpw_shape(p)


@pytest.mark.gpu
def test_read_skpw_bit_exact_and_row_ranges(tmp_path):
    ref = np.load(os.path.join(GOLD, "io_expected.npz"))["skpw"]
    path = os.path.join(GOLD, "io_a.skpw")
    t = skio.read_skpw(path, block_bytes=8 * 23 * 5)     # 5-row staging blocks
    assert np.array_equal(t.cpu().numpy(), ref)
    s = skio.read_skpw(path, rows=(11, 30))
    assert np.array_equal(s.cpu().numpy(), ref[11:30])
    f = skio.read_skpw(path, dtype=torch.float32)
    assert np.array_equal(f.cpu().numpy(), ref.astype(np.float32))
    out = tmp_path / "w.skpw"
    skio.write_skpw(t, out)
    assert out.read_bytes() == open(path, "rb").read()
    bad = np.array(ref)
    bad[3, 4] = np.nan
    with open(out, "wb") as fh:
        blob = open(path, "rb").read()
        fh.write(blob[:21] + bad.astype("<f8").tobytes())
    with pytest.raises(ValueError, match="non-finite"):
        skio.read_skpw(out)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["array_general", "array_symmetric", "coord_general",
                                  "coord_symmetric"])
def test_read_matrix_market_matches_reference(name):
    ref = np.load(os.path.join(GOLD, "io_expected.npz"))[name]
    t = skio.read_matrix_market(os.path.join(GOLD, f"io_{name}.mtx"))
    assert np.array_equal(t.cpu().numpy(), ref)


@pytest.mark.gpu
@pytest.mark.parametrize("text,msg", [
    ("%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1\n", ":1: unsupported field"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n", ":3: index (3, 1) out of bounds"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n", ":3: expected 2 entries, got 1"),
    ("%%MatrixMarket matrix array real general\n2 1\n1.0\nx\n", ":4: non-real value 'x'"),
    ("%%MatrixMarket matrix array real symmetric\n2 3\n", ":2: symmetric matrices must be square"),
    ("%%MatrixMarket vector array real general\n1 1\n1\n", ":1: malformed MatrixMarket header"),
])
def test_read_matrix_market_errors(tmp_path, text, msg):
    p = tmp_path / "bad.mtx"
    p.write_text(text)
    with pytest.raises(ValueError) as ei:
        skio.read_matrix_market(p)
    assert msg in str(ei.value)


def test_matrix_market_host_parser_matches_reference_fuzz(tmp_path):
    """600 seeded well-formed and malformed files with the LIVE reference's
    outcome (tests/golden/make_mm_fuzz.py): same matrix, or the same
    ValueError message and line number.  Host parsing only (no GPU); the
    non-finite test the reference does in as_matrix runs on the device in
    read_matrix_market, so those cases must parse to a non-finite matrix."""
    import json
    cases = json.load(open(os.path.join(GOLD, "mm_fuzz.json")))
    p = tmp_path / "f.mtx"
    for c in cases:
        p.write_text(c["text"])
        try:
            got = skio.read_matrix_market_host(p).numpy()
            err = None
        except ValueError as e:
            got, err = None, str(e).split(str(p), 1)[1]
        if c["ok"]:
            assert err is None, (c["text"], err)
            assert np.array_equal(got, np.asarray(c["matrix"])), c["text"]
        elif "non-finite" in c["error"]:
            assert err is None and not np.isfinite(got).all(), c["text"]
        else:
            assert err == c["error"], (c["text"], err, c["error"])
