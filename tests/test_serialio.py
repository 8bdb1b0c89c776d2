"""`.hgi` containers on CPU: reference-format round trips, corruption errors
(cghkit/serialio.py:167-238), and the library's CRC-32 combine against zlib."""

import zlib

import numpy as np
import pytest

from paper_2006_10509_b200 import serialio as S
from paper_2006_10509_b200.errors import ChecksumMismatchError, EmptyImageError, MalformedJsonError, TruncatedPayloadError


def meta():
    return S.Metadata(parameters=[("algorithm", "gs"), ("iterations", 5)], seed=7, app_version="b200",
                      timestamp="2026-01-01T00:00:00Z", algorithm="gs", error_final=0.125, iterations=5)


def test_roundtrip_bit_exact(tmp_path, rng):
    f = rng.normal(size=(5, 7)) + 1j * rng.normal(size=(5, 7))
    p = tmp_path / "a.hgi"
    S.save_field(f, meta(), p)
    g, m = S.load_field(p)
    assert np.array_equal(f, g) and m == meta()
    header, _, ok = S.inspect_field(p)
    assert ok and header["width"] == 7 and header["height"] == 5
    blob = p.read_bytes()
    assert blob[:4] == b"HGI1"
    assert header["checksum"] == zlib.crc32(blob[-5 * 7 * 16:])


def test_corruption_is_detected(tmp_path):
    p = tmp_path / "b.hgi"
    S.save_field(np.ones((3, 3), complex), meta(), p)
    blob = bytearray(p.read_bytes())
    blob[-3] ^= 0x10
    (tmp_path / "c.hgi").write_bytes(bytes(blob))
    with pytest.raises(ChecksumMismatchError):
        S.load_field(tmp_path / "c.hgi")
    assert S.inspect_field(tmp_path / "c.hgi")[2] is False
    (tmp_path / "d.hgi").write_bytes(bytes(blob[:-8]))
    with pytest.raises(TruncatedPayloadError):
        S.load_field(tmp_path / "d.hgi")
    (tmp_path / "e.hgi").write_bytes(b"XXXX" + bytes(blob[4:]))
    with pytest.raises(MalformedJsonError):
        S.load_field(tmp_path / "e.hgi")
    with pytest.raises(EmptyImageError):
        S.save_field(np.zeros((0, 4), complex), meta(), tmp_path / "f.hgi")


@pytest.mark.parametrize("na,nb", [(0, 0), (1, 0), (0, 5), (3, 17), (1000, 4096), (65536, 1)])
def test_crc32_combine_matches_zlib(na, nb, rng):
    a = rng.integers(0, 256, na, dtype=np.uint8).tobytes()
    b = rng.integers(0, 256, nb, dtype=np.uint8).tobytes()
    assert S.crc32_combine(zlib.crc32(a), zlib.crc32(b), len(b)) == zlib.crc32(a + b)
