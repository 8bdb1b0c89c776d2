"""GPU parity for the SA / DBS persistent search kernel and the kernel seam.

Bar (north star): accept/reject (SA) and commit (DBS) sequences identical to
the reference for the first 10^4 decisions; holograms bit-exact; traces
within 1e-9 relative (float64 incremental state).
"""

import threading

import numpy as np
import pytest

import golden_cases as G
from oracle import cgh_oracle as O
from paper_2006_10509_b200 import algorithms as A
from paper_2006_10509_b200 import kernels as K
from paper_2006_10509_b200.search import dbs_call, sa_call
from paper_2006_10509_b200.slm import binary_phase, states

pytestmark = pytest.mark.gpu

MAN = G.manifest()["cases"]
SEARCH_CASES = sorted(k for k in MAN if k.startswith(("sa_", "dbs_")))


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300))


@pytest.mark.parametrize("name", SEARCH_CASES)
def test_golden_search_bit_exact(name):
    rec = MAN[name]
    cfg, target, illum = G.build(rec)
    arrs = G.load_arrays(name)
    holo, rep = A.RUNNERS[rec["algorithm"]](cfg, target, illum)
    assert np.array_equal(holo, states(cfg.slm.scheme)[arrs["idx0"]])
    trace = np.array([e for _, e in rep.error_trace])
    assert len(trace) == len(arrs["trace"])
    assert rel(trace, arrs["trace"]) < 1e-9
    assert [k for k, _ in rep.error_trace] == list(arrs["trace_k"])
    assert rep.termination == rec["termination"]
    assert rep.iterations_executed == rec["iterations_executed"]
    assert abs(rep.efficiency - rec["efficiency"]) < 1e-9


def test_sa_decisions_match_oracle():
    rec = MAN["sa_32_bin_auto"]
    cfg, target, illum = G.build(rec)
    _, ref = O.sa(cfg, target, illum, log_limit=3000)
    _, rep = sa_call(cfg, target, illum, None, None, None, log_cap=3000)
    pix, lev, acc = rep.decisions
    want = np.array(ref.log)
    assert np.array_equal(pix, want[:, 0].astype(np.int64))
    assert np.array_equal(lev, want[:, 1].astype(np.int32))
    assert np.array_equal(acc.astype(bool), want[:, 2].astype(bool))


@pytest.mark.slow
def test_c4_sa_first_10k_decisions_match_reference():
    """C4: SA 1024x1024 binary, seed 3: golden log from the real reference
    (100 warm-up draws then 10^4 proposals with their accept flags)."""
    rec = MAN["C4_sa_1024_bin_1e4"]
    cfg, target, illum = G.build(rec)
    log = G.load_arrays("C4_sa_1024_bin_1e4")["log"]
    gold = log[100:100 + 10000]
    holo, rep = sa_call(cfg, target, illum, None, None, None, log_cap=10000)
    pix, lev, acc = rep.decisions
    assert np.array_equal(pix, gold[:, 0].astype(np.int64))
    assert np.array_equal(lev, gold[:, 1].astype(np.int32))
    assert np.array_equal(acc.astype(np.int64), gold[:, 2].astype(np.int64))
    assert np.array_equal(holo, states(cfg.slm.scheme)[G.load_arrays("C4_sa_1024_bin_1e4")["idx0"]])
    assert abs(rep.final_error - rec["final_error"]) / rec["final_error"] < 1e-9


@pytest.mark.slow
def test_c4_dbs_first_10k_visits_match_reference():
    """C4: DBS 1024x1024 binary raster, seed 3: commits among the first 10^4
    pixel visits equal the reference's (golden commit log)."""
    rec = MAN["C4_dbs_1024_bin_raster_1e4"]
    cfg, target, illum = G.build(rec)
    gold = G.load_arrays("C4_dbs_1024_bin_raster_1e4")["log"]   # (pixel, level, change) per commit
    cfg.max_passes = 1
    _, rep = dbs_call(cfg, target, illum, None, None, None, log_cap=10000)
    pix, lev, ch = rep.decisions
    assert np.array_equal(pix, np.arange(10000))
    took = lev >= 0
    assert np.array_equal(pix[took], gold[:, 0].astype(np.int64))
    assert np.array_equal(lev[took], gold[:, 1].astype(np.int32))
    assert np.max(np.abs(ch[took] - gold[:, 2])) < 1e-10   # sums over 2^20 samples: absolute


def test_sa_audit_matches_full_repropagation():
    rec = MAN["sa_16_pl4_fresnel_mask"]
    cfg, target, illum = G.build(rec)
    worst = []

    def audit(k, inc, holo):
        full = O.amplitude_error(O.to_replay(holo, cfg.propagation), target, cfg.metric.mask, False)
        worst.append(abs(inc - full))

    A.run_sa(cfg, target, illum, audit=audit)
    interval = max(1, cfg.proposals // 1000)
    assert len(worst) == cfg.proposals // interval
    assert max(worst) < 1e-9


def test_dbs_toy_descent_optimum_and_determinism():
    for seed in (1, 2, 3, 4, 5):
        rec = MAN[f"dbs_toy_2x2_seed{seed}"]
        cfg, target, illum = G.build(rec)
        holo, rep = A.run_dbs(cfg, target)
        ref_h, ref = O.dbs(cfg, target)
        assert np.array_equal(holo, ref_h)
        assert abs(rep.final_error - ref.final_error) < 1e-12
    rec = MAN["dbs_16_pl4_random_fresnel"]
    cfg, target, illum = G.build(rec)
    a, ra = A.run_dbs(cfg, target, illum)
    b, rb = A.run_dbs(cfg, target, illum)
    assert np.array_equal(a, b) and ra.error_trace == rb.error_trace


def test_sa_cancellation_via_progress():
    rec = MAN["sa_16_bin_t0"]
    cfg, target, _ = G.build(rec)
    cfg.proposals = 100000
    cancel = threading.Event()

    def progress(k, err):
        if k >= 50:
            cancel.set()

    _, rep = A.run_sa(cfg, target, progress=progress, cancel=cancel)
    assert rep.termination == A.CANCELLED
    assert rep.iterations_executed < 100000


def test_dbs_cancel_before_start():
    rec = MAN["dbs_16_bin_raster"]
    cfg, target, _ = G.build(rec)
    ev = threading.Event()
    ev.set()
    holo, rep = A.run_dbs(cfg, target, cancel=ev)
    assert rep.termination == A.CANCELLED and rep.iterations_executed == 0
    assert np.all(np.isin(holo, states(binary_phase())))


def test_kernel_seam_matches_c_oracle():
    gen = np.random.default_rng(3)
    h, w = 12, 10
    holo = gen.normal(size=(h, w)) + 1j * gen.normal(size=(h, w))
    replay = np.fft.fft2(holo, norm="ortho")
    mask = gen.random((h, w)) < 0.6
    mask[0, 0] = True
    mu, mv = np.nonzero(mask)
    mu = mu.astype(np.int32)
    mv = mv.astype(np.int32)
    rm = np.ascontiguousarray(replay[mu, mv])
    tm = np.ascontiguousarray(gen.random((h, w))[mu, mv])
    rows = np.exp(-2j * np.pi * np.outer(np.arange(h), np.arange(h)) / h)
    cols = np.exp(-2j * np.pi * np.outer(np.arange(w), np.arange(w)) / w) / np.sqrt(h * w)
    d = 0.37 - 1.1j
    got = K.delta_error(rm, tm, rows[5], cols[7], mu, mv, d)
    st = O.PixelSearchState.__new__(O.PixelSearchState)
    lib = O._incr_lib()
    if lib:
        want = lib.oracle_delta_error(O._ptr(rm), O._ptr(tm), O._ptr(rows[5].copy()), O._ptr(cols[7].copy()),
                                      O._ptr(mu), O._ptr(mv), len(tm), d.real, d.imag)
        assert abs(got - want) < 1e-12
    deltas = np.array([0.3 + 0.1j, 0.0, -1.2 + 0.4j, 0.8j])
    bj, bc = K.best_delta(rm, tm, rows[2], cols[4], mu, mv, deltas)
    changes = [K.delta_error(rm, tm, rows[2], cols[4], mu, mv, x) if x != 0 else np.inf for x in deltas]
    j = int(np.argmin(changes))
    if changes[j] < 0:
        assert bj == j and abs(bc - changes[j]) < 1e-12
    else:
        assert bj == -1 and bc == 0.0
    before = rm.copy()
    K.commit_update(rm, rows[3], cols[3], mu, mv, d)
    modified = holo.copy()
    modified[3, 3] += d
    assert np.max(np.abs(rm - np.fft.fft2(modified, norm="ortho")[mu, mv])) < 1e-12
    assert not np.array_equal(rm, before)
    del st
