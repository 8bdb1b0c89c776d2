"""Batch runner on the GPU: several host threads share the C ABI (reentrancy)
and results do not depend on how jobs are spread over worker threads."""

import numpy as np
import pytest

from paper_2006_10509_b200 import algorithms as A
from paper_2006_10509_b200.image import rect_mask
from paper_2006_10509_b200.multi import Job, derived_seed, run_batch
from paper_2006_10509_b200.propagation import MetricSpec, PropagationSpec
from paper_2006_10509_b200.slm import PhaseOnly, SlmSpec, binary_phase
from paper_2006_10509_b200.workloads import batched_target

pytestmark = pytest.mark.gpu


def jobs():
    out = []
    for i, alg in enumerate(["gs", "ospr", "sa", "dbs", "gs", "gs"]):
        n = 64 if alg in ("sa", "dbs") else 256
        scheme = binary_phase() if alg in ("sa", "dbs", "ospr") else PhaseOnly(8)
        cfg = A.AlgorithmConfig(alg, SlmSpec(n, n, scheme), PropagationSpec("fresnel" if i % 2 else "fourier"),
                                MetricSpec(rect_mask(n, n)), seed=derived_seed(7, f"j{i}"), iterations=20,
                                subframes=4, proposals=500, max_passes=2)
        out.append(Job(f"j{i}", cfg, batched_target(n, i + 1)))
    return out


def test_threads_share_the_library_deterministically():
    js = jobs()
    one = run_batch(js, devices=[0])
    three = run_batch(js, devices=[0, 0, 0])
    for a, b in zip(one, three):
        assert a.error is None and b.error is None, (a.error, b.error)
        ha = a.hologram if isinstance(a.hologram, list) else [a.hologram]
        hb = b.hologram if isinstance(b.hologram, list) else [b.hologram]
        assert all(np.array_equal(x, y) for x, y in zip(ha, hb))
        assert a.report.error_trace == b.report.error_trace


def test_device_runners_in_a_reference_style_thread_pool():
    """multi.device_runners used the way controller.run_batch uses RUNNERS
    (ThreadPoolExecutor over jobs, controller.py:345-346): per-job outputs equal
    sequential single-device runs whatever thread ran them."""
    from concurrent.futures import ThreadPoolExecutor

    import numpy as np

    from paper_2006_10509_b200 import algorithms as A
    from paper_2006_10509_b200.image import rect_mask
    from paper_2006_10509_b200.multi import derived_seed, device_runners
    from paper_2006_10509_b200.propagation import MetricSpec, PropagationSpec
    from paper_2006_10509_b200.slm import PhaseOnly, SlmSpec
    from paper_2006_10509_b200.workloads import natural_target

    n = 512
    target = natural_target(n)

    def cfg_of(job_id):
        return A.AlgorithmConfig("gs", SlmSpec(n, n, PhaseOnly(8)), PropagationSpec("fresnel"),
                                 MetricSpec(rect_mask(n, n)), seed=derived_seed(11, job_id), iterations=8)

    ids = [f"job{i}" for i in range(6)]
    runners = device_runners([0, 0, 0])
    with ThreadPoolExecutor(max_workers=3) as pool:
        got = list(pool.map(lambda j: runners["gs"](cfg_of(j), target), ids))
    for j, (holo, rep) in zip(ids, got):
        ref_h, ref = A.run_gs(cfg_of(j), target)
        assert np.array_equal(holo, ref_h)
        assert rep.error_trace == ref.error_trace
