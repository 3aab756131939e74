"""BTA1 files (reference tests/test_fileio.py), plus byte-for-byte parity
with files the reference wrote (tests/golden/make_bta1.py)."""

import hashlib
import json
import os

import numpy as np
import pytest

import paper_2601_04904_b200 as bs
from paper_2601_04904_b200.fileio import MAGIC, payload_size

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
MAN = json.load(open(os.path.join(GOLDEN, "bta1_manifest.json")))


@pytest.mark.parametrize("shape", [(1, 1, 0), (1, 3, 2), (4, 2, 0), (3, 2, 1), (5, 4, 3), (2, 1, 5)])
def test_roundtrip_bitwise(tmp_path, shape):
    m = bs.generate_dd_bta(*shape, seed=sum(shape))
    path = tmp_path / "m.bta"
    bs.write_bta(m, path)
    assert m.equals_exact(bs.read_bta(path))


def test_header_layout(tmp_path):
    m = bs.generate_dd_bta(3, 2, 1, seed=0)
    path = tmp_path / "m.bta"
    bs.write_bta(m, path)
    raw = path.read_bytes()
    assert raw[:4] == MAGIC
    assert [int.from_bytes(raw[i:i + 8], "little") for i in (4, 12, 20)] == [3, 2, 1]
    assert raw[28] == 0x10
    assert len(raw) == 29 + payload_size(3, 2, 1)
    assert bs.read_bta_header(path) == (3, 2, 1)


@pytest.mark.parametrize("name", sorted(MAN))
def test_reference_files_bytewise(tmp_path, name):
    """Files written by the reference read back exactly, and re-writing them
    reproduces the reference's bytes."""
    meta = MAN[name]
    path = os.path.join(GOLDEN, f"bta1_{name}.bta")
    raw = open(path, "rb").read()
    assert hashlib.sha256(raw).hexdigest() == meta["sha256"]
    m = bs.read_bta(path)
    assert (m.n, m.b, m.a) == (meta["n"], meta["b"], meta["a"])
    if "seed" in meta:
        assert m.equals_exact(bs.generate_dd_bta(meta["n"], meta["b"], meta["a"], seed=meta["seed"]))
    out = tmp_path / "again.bta"
    bs.write_bta(m, out)
    assert out.read_bytes() == raw


def test_pinned_read(tmp_path):
    m = bs.generate_dd_bta(3, 4, 2, seed=5)
    bs.write_bta(m, tmp_path / "m.bta")
    assert bs.read_bta(tmp_path / "m.bta", pinned=True).equals_exact(m)


def test_errors(tmp_path):
    p = tmp_path / "x.bta"
    p.write_bytes(b"")
    with pytest.raises(bs.BadMagicError):
        bs.read_bta(p)
    p.write_bytes(b"NOPE" + b"\x00" * 64)
    with pytest.raises(bs.BadMagicError):
        bs.read_bta(p)
    p.write_bytes(MAGIC + b"\x01\x00")
    with pytest.raises(bs.TruncatedPayloadError):
        bs.read_bta(p)
    one, two = tmp_path / "1.bta", tmp_path / "2.bta"
    bs.write_bta(bs.generate_dd_bta(1, 2, 0, seed=0), one)
    bs.write_bta(bs.generate_dd_bta(2, 2, 0, seed=0), two)
    p.write_bytes(two.read_bytes()[:29] + one.read_bytes()[29:])
    with pytest.raises(bs.TruncatedPayloadError):
        bs.read_bta(p)
    p.write_bytes(two.read_bytes() + b"\x00" * 16)
    with pytest.raises(bs.ShapeInconsistencyError):
        bs.read_bta(p)
    raw = bytearray(two.read_bytes())
    raw[28] = 0x42
    p.write_bytes(bytes(raw))
    with pytest.raises(bs.ShapeInconsistencyError):
        bs.read_bta(p)
    p.write_bytes(MAGIC + (0).to_bytes(8, "little") * 3 + bytes([0x10]))
    with pytest.raises(bs.ShapeInconsistencyError):
        bs.read_bta(p)
    m = bs.generate_dd_bta(2, 2, 0, seed=0)
    m.diag[0][0, 0] = np.nan
    bs.write_bta(m, p)
    with pytest.raises(bs.ShapeInconsistencyError):
        bs.read_bta(p)
    assert issubclass(bs.BadMagicError, bs.FormatError) and issubclass(bs.FormatError, ValueError)
