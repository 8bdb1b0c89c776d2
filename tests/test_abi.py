"""C-ABI surface (CPU): the library loads, exports every function declared in
include/cghb200.h, and fails loudly (no CPU fallback) without a device."""

import os
import re

import numpy as np
import pytest

from paper_2006_10509_b200 import _native, errors

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "cghb200.h")


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?(?:int|void|char)\s*\**\s*(cgh_\w+)\s*\(", text, flags=re.M)
    return sorted(set(names))


def test_header_declares_the_expected_api():
    names = header_functions()
    assert len(names) >= 20
    assert set(names) == set(_native.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = _native.library()
    for name in header_functions():
        assert hasattr(lib, name), name
    assert lib.cgh_version() >= 10000


def test_library_is_sm100a_build():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.skipif(_native.device_count() > 0, reason="GPU present")
def test_no_device_fails_loudly():
    from paper_2006_10509_b200 import algorithms as A
    from paper_2006_10509_b200.image import rect_mask
    from paper_2006_10509_b200.propagation import MetricSpec, PropagationSpec, fft2
    from paper_2006_10509_b200.slm import SlmSpec, binary_phase

    cfg = A.AlgorithmConfig("gs", SlmSpec(8, 8, binary_phase()), PropagationSpec(), MetricSpec(rect_mask(8, 8)))
    with pytest.raises(errors.BackendUnavailableError):
        A.run_gs(cfg, np.ones((8, 8), complex))
    with pytest.raises(errors.BackendUnavailableError):
        fft2(np.ones((8, 8), complex))
    with pytest.raises(errors.BackendUnavailableError):
        A.run_sa(cfg, np.ones((8, 8), complex))


def test_host_expansion_into_prefaulted_arrays():
    """Host-only helpers (no GPU): cgh_prefault + cgh_expand_states into a
    caller-provided array give exactly states[idx]; bad outputs are rejected."""
    rng = np.random.default_rng(5)
    table = np.exp(2j * np.pi * np.arange(8) / 8)
    idx = rng.integers(0, 8, (1024, 1536)).astype(np.uint8)
    pre = _native.PrefaultedArrays(idx.shape, 2)    # 2 x 24 MiB: touched on a thread
    bufs = pre.take()
    assert len(bufs) == 2 and all(b.shape == idx.shape for b in bufs)
    out = _native.expand_states(idx, table, out=bufs[1])
    assert out is bufs[1] and np.array_equal(out, table[idx])
    small = _native.PrefaultedArrays((4, 4)).take()[0]   # below the thread threshold
    assert np.array_equal(_native.expand_states(idx[:4, :4], table, out=small), table[idx[:4, :4]])
    with pytest.raises(ValueError):
        _native.expand_states(idx, table, out=np.empty((3, 3), np.complex128))
    _native.check(_native.library().cgh_prefault(None, 0, 4))
    with pytest.raises(ValueError):
        _native.check(_native.library().cgh_prefault(None, 4096, 4))
