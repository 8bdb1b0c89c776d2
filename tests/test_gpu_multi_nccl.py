"""The library's own multi-GPU data plane (cgh_multi_*: NCCL communicator,
CUDA IPC peer mappings, device barrier on peer flags; slab.NcclExchange) on a
one-rank NCCL group (this build has one GPU): collectives are identities, the
fused peer-store corner turn + device barrier run through the same code path
as at G ranks, and the C6 slab run and the sharded OSPR run equal the plain
single-GPU runs bit for bit."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(proc, out_dir):
    import ctypes

    import torch
    import torch.distributed as dist

    from paper_2006_10509_b200 import _native
    from paper_2006_10509_b200 import algorithms as A
    from paper_2006_10509_b200 import slab as SL
    from paper_2006_10509_b200.image import rect_mask
    from paper_2006_10509_b200.multi import run_ospr_sharded
    from paper_2006_10509_b200.propagation import MetricSpec, PropagationSpec
    from paper_2006_10509_b200.runtime import precision
    from paper_2006_10509_b200.slm import PhaseOnly, SlmSpec, binary_phase
    from paper_2006_10509_b200.workloads import natural_target

    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        ex = SL.NcclExchange()
        lib = _native.library()
        # collectives of a 1-rank communicator on the pass stream
        x = torch.arange(12, dtype=torch.float64, device="cuda")
        (y,) = ex.all_reduce([x.clone()])
        g = ex.gather([x])
        src = torch.arange(64, dtype=torch.uint8, device="cuda")
        dst = torch.zeros(64, dtype=torch.uint8, device="cuda")
        _native.check(lib.cgh_multi_all_to_all(ex.handle, ctypes.c_void_p(src.data_ptr()),
                                               ctypes.c_void_p(dst.data_ptr()), 64, ctypes.c_void_p(ex.stream)))
        for _ in range(3):
            _native.check(lib.cgh_multi_device_barrier(ex.handle, ctypes.c_void_p(ex.stream)))
        torch.cuda.synchronize()
        ok = bool(torch.equal(y, x)) and len(g) == 1 and bool(torch.equal(g[0], x)) and bool(torch.equal(src, dst))
        # C6 path: slab GS through the library exchange
        n = 256
        cfg = A.AlgorithmConfig("gs", SlmSpec(n, n, PhaseOnly(8)), PropagationSpec("fresnel", distance=0.05),
                                MetricSpec(rect_mask(n, n, [(32, 40, 128, 90)]), rescale=True), seed=3, iterations=5,
                                feedback_gain=0.2)
        with precision("fp64"):
            holo, rep = SL.run_gs_slab(cfg, natural_target(n), exchange=ex)
        np.save(os.path.join(out_dir, "slab.npy"), holo)
        np.save(os.path.join(out_dir, "slab_trace.npy"), np.array([e for _, e in rep.error_trace]))
        # C2 path: sharded OSPR through the library all-gather
        ocfg = A.AlgorithmConfig("ospr", SlmSpec(512, 512, binary_phase()), PropagationSpec(),
                                 MetricSpec(rect_mask(512, 512)), seed=5, subframes=6)
        with precision("fp32"):
            oh, orep = run_ospr_sharded(ocfg, natural_target(512), exchange=ex)
        np.save(os.path.join(out_dir, "ospr.npy"), np.array(oh))
        np.save(os.path.join(out_dir, "ospr_trace.npy"), np.array([e for _, e in orep.error_trace]))
        ex.close()
        with open(os.path.join(out_dir, "ok"), "w") as f:
            f.write("1" if ok else "0")
    finally:
        dist.destroy_process_group()


def test_library_exchange_single_rank(tmp_path):
    import torch.multiprocessing as mp

    from paper_2006_10509_b200 import _native
    from paper_2006_10509_b200 import algorithms as A
    from paper_2006_10509_b200 import slab as SL
    from paper_2006_10509_b200.image import rect_mask
    from paper_2006_10509_b200.propagation import MetricSpec, PropagationSpec
    from paper_2006_10509_b200.runtime import precision
    from paper_2006_10509_b200.slm import PhaseOnly, SlmSpec, binary_phase
    from paper_2006_10509_b200.workloads import natural_target

    assert _native.library().cgh_multi_available() == 1
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    mp.spawn(_worker, args=(str(tmp_path),), nprocs=1, join=True)
    assert open(tmp_path / "ok").read() == "1"
    n = 256
    cfg = A.AlgorithmConfig("gs", SlmSpec(n, n, PhaseOnly(8)), PropagationSpec("fresnel", distance=0.05),
                            MetricSpec(rect_mask(n, n, [(32, 40, 128, 90)]), rescale=True), seed=3, iterations=5,
                            feedback_gain=0.2)
    with precision("fp64"):
        holo, rep = SL.run_gs_slab(cfg, natural_target(n))
    assert np.array_equal(np.load(tmp_path / "slab.npy"), holo)
    assert np.array_equal(np.load(tmp_path / "slab_trace.npy"), np.array([e for _, e in rep.error_trace]))
    ocfg = A.AlgorithmConfig("ospr", SlmSpec(512, 512, binary_phase()), PropagationSpec(),
                             MetricSpec(rect_mask(512, 512)), seed=5, subframes=6)
    with precision("fp32"):
        oh, orep = A.run_ospr(ocfg, natural_target(512))
    assert np.array_equal(np.load(tmp_path / "ospr.npy"), np.array(oh))
    e1, e0 = np.load(tmp_path / "ospr_trace.npy"), np.array([e for _, e in orep.error_trace])
    assert np.max(np.abs(e1 - e0) / e0) < 1e-5
