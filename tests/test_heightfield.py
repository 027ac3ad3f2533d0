"""CPU: the ABHF / CSV heightfield format (heightfield_io.hpp:11-16) of the host
mirror, pinned byte-for-byte against files the reference writers produced
(tests/golden/make_golden_heightfield.py)."""
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))

from make_golden_heightfield import CASCADE, TIME, heightfield_input  # noqa: E402
from paper_2503_03326_b200 import ocean as oc  # noqa: E402

GOLD_ABHF = os.path.join(HERE, "golden", "heightfield_ref.abhf")
GOLD_CSV = os.path.join(HERE, "golden", "heightfield_ref.csv")


def test_abhf_bytes_match_reference(tmp_path):
    p = tmp_path / "f.abhf"
    oc.write_heightfield(str(p), heightfield_input(), cascade=CASCADE, t=TIME)
    assert p.read_bytes() == open(GOLD_ABHF, "rb").read()


def test_abhf_header_layout():
    buf = open(GOLD_ABHF, "rb").read()
    n = heightfield_input().shape[0]
    assert buf[:4] == b"ABHF" and len(buf) == 16 + 4 * n * n
    assert int.from_bytes(buf[4:8], "little") == n
    assert int.from_bytes(buf[8:12], "little", signed=True) == CASCADE
    assert np.frombuffer(buf[12:16], "<f4")[0] == np.float32(TIME)


def test_abhf_read_reference_file():
    f, hdr = oc.read_heightfield(GOLD_ABHF)
    assert hdr == {"resolution": 7, "cascade": CASCADE, "time": float(np.float32(TIME))}
    want = heightfield_input().astype(np.float32).astype(np.float64)
    assert np.array_equal(f, want)
    assert np.signbit(f[0, 1])  # -0.0 survives


def test_csv_matches_reference(tmp_path):
    p = tmp_path / "f.csv"
    oc.write_heightfield_csv(str(p), heightfield_input())
    assert p.read_text() == open(GOLD_CSV).read()


def test_abhf_errors(tmp_path):
    with pytest.raises(oc.IoError, match="does not match"):
        oc.write_heightfield(str(tmp_path / "x.abhf"), np.zeros((4, 4)), resolution=5)
    with pytest.raises(oc.IoError, match="cannot open for writing"):
        oc.write_heightfield(str(tmp_path / "missing" / "x.abhf"), np.zeros((4, 4)))
    bad = tmp_path / "bad.abhf"
    bad.write_bytes(b"ABHX" + bytes(12))
    with pytest.raises(oc.IoError, match="bad magic"):
        oc.read_heightfield(str(bad))
    trunc = tmp_path / "trunc.abhf"
    trunc.write_bytes(open(GOLD_ABHF, "rb").read()[:-1])
    with pytest.raises(oc.IoError, match="truncated"):
        oc.read_heightfield(str(trunc))
    zero = tmp_path / "zero.abhf"
    zero.write_bytes(b"ABHF" + bytes(12))
    with pytest.raises(oc.IoError, match="bad resolution"):
        oc.read_heightfield(str(zero))
    with pytest.raises(oc.IoError, match="cannot open"):
        oc.read_heightfield(str(tmp_path / "nope.abhf"))
