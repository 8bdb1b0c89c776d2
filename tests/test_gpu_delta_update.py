"""Full-plane rank-1 replay update on the device (propagation.py:205-218,
pinned by the reference's tests/test_propagation.py:236-267): the updated
replay equals the transform of the changed hologram."""

import numpy as np
import pytest

from paper_2006_10509_b200 import propagation as P

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("shape,m,n", [((8, 8), 3, 5), ((64, 128), 63, 0), ((256, 256), 17, 200), ((1024, 512), 1000, 511)])
def test_rank_one_update_matches_retransform(shape, m, n):
    rng = np.random.default_rng(shape[0] + m)
    h = np.exp(1j * rng.uniform(0, 2 * np.pi, shape))
    replay = np.fft.fft2(h, norm="ortho")            # uncentred unitary transform
    delta = 0.3 - 0.7j
    P.delta_replay_update(replay, m, n, delta)
    h2 = h.copy()
    h2[m, n] += delta
    ref = np.fft.fft2(h2, norm="ortho")
    assert np.max(np.abs(replay - ref)) < 1e-12


def test_bounds_and_dtype():
    r = np.zeros((4, 4), np.complex128)
    with pytest.raises(IndexError):
        P.delta_replay_update(r, 4, 0, 1.0)
    with pytest.raises(TypeError):
        P.delta_replay_update(np.zeros((4, 4), np.complex64), 0, 0, 1.0)
