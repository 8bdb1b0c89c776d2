"""numpy PCG64 stream semantics the CUDA emulation follows (oracle/pcg64_model.py)
checked against numpy itself, plus the library's host-side emulation
(cgh_permutation / cgh_random_doubles with device=-1). CPU only."""

import ctypes

import numpy as np
import pytest

from oracle.pcg64_model import Pcg64Model
from paper_2006_10509_b200 import _native


def test_model_matches_numpy_draw_types():
    g = np.random.Generator(np.random.PCG64(7))
    m = Pcg64Model.from_numpy(g.bit_generator)
    for size, levels in [(1 << 20, 2), (4096, 8), (1000, 3), (7, 5)]:
        for i in range(3000):
            assert int(g.integers(size)) == m.integers(size)
            j = int(g.integers(levels - 1))
            assert j == m.integers(levels - 1)
            if (i + j) % 3 == 0:
                assert g.random() == m.next_double()


def test_model_advance_and_fill_order():
    g = np.random.Generator(np.random.PCG64(3))
    m = Pcg64Model.from_numpy(g.bit_generator)
    x = g.random((16, 16))
    m.advance(16 * 5 + 7)
    assert m.next_double() == x[5, 7]


def test_int_seed_equals_seedsequence_seed():
    # algorithms.py:160 PCG64(seed) vs algorithms.py:423-424 PCG64(SeedSequence(seed))
    for s in (1, 3, 12345):
        assert np.random.PCG64(s).state == np.random.PCG64(np.random.SeedSequence(s)).state


def test_model_permutation():
    root = np.random.SeedSequence(9)
    for _ in range(3):
        child = root.spawn(1)[0]
        a = np.random.Generator(np.random.PCG64(child)).permutation(997)
        b = Pcg64Model.from_numpy(np.random.PCG64(child)).permutation(997)
        assert list(a) == b


lib = _native.library(required=False)


@pytest.mark.skipif(lib is None, reason="libcghb200.so not built")
def test_library_permutation_matches_numpy():
    root = np.random.SeedSequence(11)
    for n in (1, 2, 1000, 1 << 16):
        child = root.spawn(1)[0]
        want = np.random.Generator(np.random.PCG64(child)).permutation(n)
        st = _native.Pcg64State.from_bitgen(np.random.PCG64(child))
        out = np.empty(n, np.int64)
        assert lib.cgh_permutation(ctypes.byref(st), n, _native.ptr(out)) == 0
        assert np.array_equal(out, want)


@pytest.mark.skipif(lib is None, reason="libcghb200.so not built")
def test_library_host_doubles_match_numpy():
    bg = np.random.PCG64(5)
    want = np.random.Generator(np.random.PCG64(5)).random(5000)
    st = _native.Pcg64State.from_bitgen(bg)
    out = np.empty(1000, np.float64)
    assert lib.cgh_random_doubles(-1, ctypes.byref(st), 4000, 1000, _native.ptr(out)) == 0
    assert np.array_equal(out, want[4000:])
