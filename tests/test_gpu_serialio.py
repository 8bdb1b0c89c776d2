"""Device `.hgi` payload (cgh_hgi_payload): expansion states[idx] and zlib's
CRC-32 of the payload computed from the index plane, across chunk
boundaries (chunks of 256 records, blocks of 65536) and index widths; files
written from an index plane are byte-identical to save_field's."""

import zlib

import numpy as np
import pytest

from paper_2006_10509_b200 import serialio as S
from paper_2006_10509_b200.slm import PhaseOnly, states

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("shape,levels", [((1, 1), 2), ((3, 5), 8), ((256, 256), 8), ((257, 255), 4),
                                          ((512, 300), 300), ((1024, 1024), 256), ((2048, 2048), 8)])
def test_payload_and_crc_match_zlib(shape, levels):
    table = states(PhaseOnly(levels))
    rng = np.random.default_rng(shape[0] * 7 + levels)
    dt = np.uint8 if levels <= 256 else np.int32
    idx = rng.integers(0, levels, size=shape).astype(dt)
    ref = table[idx]
    want = zlib.crc32(np.ascontiguousarray(ref).astype("<c16").tobytes())
    for mode in ("host", "device"):
        holo, crc = S.hologram_payload(idx, table, expand=mode)
        assert np.array_equal(holo.view(np.uint64), ref.view(np.uint64))
        assert crc == want


def test_file_bytes_identical_to_save_field(tmp_path):
    table = states(PhaseOnly(8))
    idx = np.random.default_rng(3).integers(0, 8, size=(300, 1000)).astype(np.uint8)
    m = S.Metadata([("a", 1)], 1, "b200", "t", "gs", 0.5, 10)
    S.save_hologram(idx, table, m, tmp_path / "g.hgi")
    S.save_field(table[idx], m, tmp_path / "h.hgi")
    assert (tmp_path / "g.hgi").read_bytes() == (tmp_path / "h.hgi").read_bytes()
    f, _ = S.load_field(tmp_path / "g.hgi")
    assert np.array_equal(f, table[idx])
