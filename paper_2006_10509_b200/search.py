"""Host side of the SA / DBS runners: validation in the reference's order,
numpy seed-state derivation, result materialisation. The search itself runs
in ``csrc/search.cu`` (persistent cooperative kernel, float64 state)."""

from __future__ import annotations

import ctypes
import time

import numpy as np

from . import _native
from .algorithms import (
    RANDOM,
    RunReport,
    _check_inputs,
    _elapsed_ms,
    _Hooks,
    _illum,
    _index_plane,
    _init_code,
    _mask_bytes,
    _problem,
    _TERMINATION,
    _trace,
)
from .slm import states


def _prep(cfg, target, illumination):
    target = np.asarray(target, dtype=np.complex128)
    _check_inputs(cfg, target, illumination)
    init = _init_code(cfg.init_mode)
    pb, keep = _problem(cfg, target)
    pb.precision = _native.FP64
    _mask_bytes(cfg, target)
    lib = _native.library()
    _native.require_device()
    return target, init, lib, pb, keep


def sa_call(cfg, target, illumination, progress, cancel, audit, log_cap=0):
    """run_sa (algorithms.py:343-404). ``log_cap`` > 0 also returns the first
    decisions as arrays (pixel, level, accepted) in ``report.decisions``."""
    start = time.perf_counter()
    target, init, lib, pb, keep = _prep(cfg, target, illumination)
    mask = _mask_bytes(cfg, target)
    tgt = _native.c128(target)
    ill = _illum(illumination)
    sp = _native.SaParams()
    sp.proposals = int(cfg.proposals)
    t0 = cfg.initial_temperature
    sp.initial_temperature = -1.0 if t0 is None else float(t0)
    sp.cooling_factor = float(cfg.cooling_factor)
    sp.init_mode = init
    sp.rng = _native.Pcg64State.from_bitgen(np.random.PCG64(cfg.seed))
    logs = None
    if log_cap > 0:
        logs = (np.zeros(log_cap, np.int64), np.zeros(log_cap, np.int32), np.zeros(log_cap, np.uint8))
        sp.log_cap = log_cap
        sp.log_pixel = logs[0].ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
        sp.log_level = logs[1].ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
        sp.log_accept = logs[2].ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))
    idx = _index_plane(pb.n_states, target.shape)
    interval = max(1, int(cfg.proposals) // 1000)
    cap = int(cfg.proposals) // interval + 3
    tk = np.zeros(cap, np.int64)
    tv = np.zeros(cap, np.float64)
    rep = _native.Report()
    hooks = _Hooks(progress, cancel, audit, target.shape[1], target.shape[0])
    table = states(cfg.slm.scheme)
    if audit is not None:
        user_audit = audit
        hooks.audit = lambda k, e, ix: user_audit(k, e, table[ix])
    st = lib.cgh_sa_run(ctypes.byref(pb), ctypes.byref(sp), _native.ptr(tgt), _native.ptr(mask), _native.ptr(ill),
                        _native.ptr(idx), _native.ptr(tk), _native.ptr(tv), cap, ctypes.byref(rep),
                        ctypes.byref(hooks.cb))
    hooks.raise_pending()
    _native.check(st)
    del keep
    report = RunReport(
        error_trace=_trace(tk, tv, rep.trace_len),
        final_error=float(rep.final_error),
        efficiency=float(rep.efficiency),
        iterations_executed=int(rep.iterations_executed),
        runtime_ms=_elapsed_ms(start),
        seed_used=cfg.seed,
        termination=_TERMINATION[rep.termination],
    )
    if logs is not None:
        report.decisions = logs
    return table[idx], report


def dbs_call(cfg, target, illumination, progress, cancel, audit, log_cap=0):
    """run_dbs (algorithms.py:410-467). ``log_cap`` > 0 returns the first pixel
    visits (pixel, committed level or -1, best change) in ``report.decisions``."""
    start = time.perf_counter()
    target, init, lib, pb, keep = _prep(cfg, target, illumination)
    mask = _mask_bytes(cfg, target)
    tgt = _native.c128(target)
    ill = _illum(illumination)
    dp = _native.DbsParams()
    dp.max_passes = int(cfg.max_passes)
    dp.scan_random = 1 if cfg.scan_order == RANDOM else 0
    dp.init_mode = init
    root = np.random.SeedSequence(cfg.seed)
    dp.rng = _native.Pcg64State.from_bitgen(np.random.PCG64(root))
    npass = max(1, int(cfg.max_passes))
    pass_rng = (_native.Pcg64State * npass)()
    if dp.scan_random:
        # one child stream per pass, spawned in order (algorithms.py:437-439)
        for i in range(int(cfg.max_passes)):
            pass_rng[i] = _native.Pcg64State.from_bitgen(np.random.PCG64(root.spawn(1)[0]))
    dp.pass_rng = ctypes.cast(pass_rng, ctypes.POINTER(_native.Pcg64State))
    logs = None
    if log_cap > 0:
        logs = (np.zeros(log_cap, np.int64), np.zeros(log_cap, np.int32), np.zeros(log_cap, np.float64))
        dp.log_cap = log_cap
        dp.log_pixel = logs[0].ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
        dp.log_level = logs[1].ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
        dp.log_change = logs[2].ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    idx = _index_plane(pb.n_states, target.shape)
    cap = int(cfg.max_passes) + 3
    tk = np.zeros(cap, np.int64)
    tv = np.zeros(cap, np.float64)
    rep = _native.Report()
    hooks = _Hooks(progress, cancel, audit, target.shape[1], target.shape[0])
    table = states(cfg.slm.scheme)
    if audit is not None:
        user_audit = audit
        hooks.audit = lambda k, e, ix: user_audit(k, e, table[ix])
    st = lib.cgh_dbs_run(ctypes.byref(pb), ctypes.byref(dp), _native.ptr(tgt), _native.ptr(mask), _native.ptr(ill),
                         _native.ptr(idx), _native.ptr(tk), _native.ptr(tv), cap, ctypes.byref(rep),
                         ctypes.byref(hooks.cb))
    hooks.raise_pending()
    _native.check(st)
    del keep
    report = RunReport(
        error_trace=_trace(tk, tv, rep.trace_len),
        final_error=float(rep.final_error),
        efficiency=float(rep.efficiency),
        iterations_executed=int(rep.iterations_executed),
        runtime_ms=_elapsed_ms(start),
        seed_used=cfg.seed,
        termination=_TERMINATION[rep.termination],
    )
    if logs is not None:
        report.decisions = logs
    return table[idx], report
