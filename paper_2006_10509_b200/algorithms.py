"""The four hologram generators — drop-in for ``cghkit/algorithms.py``.

Same entry points, parameter objects, return values and exceptions as the
reference (``algorithms.py:57-137,147,343,410,473,533``); the work runs in
``libcghb200.so`` (hand-written sm_100a CUDA) through the C ABI:

* ``run_gs``   -> ``cgh_gs_run``   two fused FFT passes per iteration
* ``run_ospr`` -> ``cgh_ospr_run`` three batched passes per frame group
* ``run_sa``   -> ``cgh_sa_run``   persistent pixel-flip kernel, fp64 state
* ``run_dbs``  -> ``cgh_dbs_run``  same kernel with windowed speculation

The host side only validates inputs in the reference's order, derives the
numpy PCG64 seed states (``SeedSequence``) the device emulates, and
materialises ``states[indices]`` so returned holograms are bitwise members
of the state set. There is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import threading
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .errors import DimensionMismatchError
from .propagation import FRESNEL, MetricSpec, PropagationSpec, fill_propagation, propagate_inverse  # noqa: F401 (FRESNEL: reference namespace)
from .runtime import current_device, runner_precision
from .slm import SlmSpec, problem_for, states

GS = "gs"
SA = "sa"
DBS = "dbs"
OSPR = "ospr"

RANDOM_PHASE = "random-phase"
BACKPROPAGATE = "backpropagate"

RASTER = "raster"
RANDOM = "random"

COMPLETED = "completed"
CONVERGED = "converged"
CANCELLED = "cancelled"

_TERMINATION = {_native.COMPLETED: COMPLETED, _native.CONVERGED: CONVERGED, _native.CANCELLED: CANCELLED}


@dataclass
class AlgorithmConfig:
    """Everything a runner needs (algorithms.py:57-81)."""

    algorithm: str
    slm: SlmSpec
    propagation: PropagationSpec
    metric: MetricSpec
    seed: int = 1
    init_mode: str = RANDOM_PHASE
    iterations: int = 100
    feedback_gain: float = 0.0
    quantize_each_iteration: bool = False
    proposals: int = 20000
    initial_temperature: float | None = None
    cooling_factor: float = 0.99995
    max_passes: int = 10
    scan_order: str = RASTER
    subframes: int = 8
    params: list = field(default_factory=list)


@dataclass
class RunReport:
    """Per-run trace and final metrics (algorithms.py:84-94)."""

    error_trace: list
    final_error: float
    efficiency: float
    iterations_executed: int
    runtime_ms: float
    seed_used: int
    termination: str


def _check_inputs(cfg, target, illumination):
    # algorithms.py:97-108
    shape = (cfg.slm.height, cfg.slm.width)
    if target.shape != shape:
        raise DimensionMismatchError(f"target {target.shape} does not match SLM {shape}")
    if illumination is not None and illumination.shape != shape:
        raise DimensionMismatchError(f"illumination {illumination.shape} does not match SLM {shape}")


def _illumination_amplitude(target, illumination):
    if illumination is None:
        return np.ones(target.shape, dtype=np.float64)
    return np.abs(illumination)


def initial_hologram(target, illumination, mode, rng, propagation=PropagationSpec()):
    """Starting hologram (algorithms.py:117-137).

    Public helper kept for API parity (tests build expected start states
    with it); the runners generate the same field on the device.
    """
    target = np.asarray(target, dtype=np.complex128)
    if illumination is not None and illumination.shape != target.shape:
        raise DimensionMismatchError(
            f"illumination {illumination.shape} does not match target {target.shape}")
    amp = _illumination_amplitude(target, illumination)
    if mode == RANDOM_PHASE:
        theta = 2.0 * np.pi * rng.random(target.shape)
        return amp * np.exp(1j * theta)
    if mode == BACKPROPAGATE:
        back = propagate_inverse(target, propagation)
        return amp * np.exp(1j * np.angle(back))
    raise ValueError(f"unknown init mode {mode!r}")


def _elapsed_ms(start):
    return (time.perf_counter() - start) * 1000.0


class _Hooks:
    """ctypes callbacks around the caller's progress/cancel; an exception in
    ``progress`` stops the device loop and is re-raised after the call."""

    def __init__(self, progress, cancel, audit=None, width=None, height=None):
        self.progress = progress
        self.cancel = cancel
        self.audit = audit
        self.error = None
        self.shape = (height, width)
        cb = _native.Callbacks()
        if cancel is not None or progress is not None or audit is not None:
            cb.cancel = _native.CANCEL_FN(self._cancel)
        if progress is not None:
            cb.progress = _native.PROGRESS_FN(self._progress)
        if audit is not None:
            cb.audit = _native.AUDIT_FN(self._audit)
        self.cb = cb

    def _cancel(self, _user):
        if self.error is not None:
            return 1
        try:
            return 1 if (self.cancel is not None and self.cancel.is_set()) else 0
        except BaseException as exc:  # noqa: BLE001 - re-raised after the call
            self.error = exc
            return 1

    def _progress(self, _user, k, err):
        if self.error is not None:
            return
        try:
            self.progress(int(k), float(err))
        except BaseException as exc:  # noqa: BLE001
            self.error = exc

    def _audit(self, _user, k, inc_err, idx_ptr):
        if self.error is not None:
            return
        try:
            h, w = self.shape
            idx = np.ctypeslib.as_array(idx_ptr, shape=(h * w,)).reshape(h, w).copy()
            self.audit(int(k), float(inc_err), idx)
        except BaseException as exc:  # noqa: BLE001
            self.error = exc

    def raise_pending(self):
        if self.error is not None:
            raise self.error


def _problem(cfg, target):
    """C problem + keepalives for a runner call (validates the propagation spec)."""
    h, w = target.shape
    pb, keep = problem_for(cfg.slm.scheme, h, w, runner_precision(), current_device())
    fill_propagation(pb, cfg.propagation)
    pb.rescale = 1 if cfg.metric.rescale else 0
    return pb, keep


def _mask_bytes(cfg, target):
    mask = np.asarray(cfg.metric.mask)
    if mask.shape != target.shape:
        raise DimensionMismatchError(f"mask {mask.shape} does not match target {target.shape}")
    if mask.dtype == np.bool_ and mask.flags.c_contiguous:
        return mask.view(np.uint8)            # numpy bools are bytes 0/1: no copy
    return np.ascontiguousarray(mask != 0, dtype=np.uint8)


def _illum(illumination):
    return None if illumination is None else _native.c128(illumination)


def _index_plane(n_states, shape, frames=None):
    dt = np.uint8 if n_states <= 256 else np.int32
    return np.empty(shape if frames is None else (frames,) + tuple(shape), dtype=dt)


def _init_code(mode):
    if mode == RANDOM_PHASE:
        return _native.INIT_RANDOM
    if mode == BACKPROPAGATE:
        return _native.INIT_BACKPROP
    raise ValueError(f"unknown init mode {mode!r}")


def _trace(tk, tv, n):
    return [(int(tk[i]), float(tv[i])) for i in range(n)]


_plans = threading.local()
_MAX_PLANS = 4


def _cached_plan(cfg, shape):
    """Per-thread cache of device plans (stream, buffers, tables) keyed by
    everything a plan bakes in; reentrant because each thread owns its plans."""
    from .plan import GenerationPlan, plan_key

    prec, dev = runner_precision(), current_device()
    key = plan_key(cfg, shape, prec, dev)
    cache = getattr(_plans, "d", None)
    if cache is None:
        cache = _plans.d = {}
    plan = cache.get(key)
    if plan is None:
        if len(cache) >= _MAX_PLANS:
            old = cache.pop(next(iter(cache)))
            old.close()
        plan = GenerationPlan(cfg, shape, precision=prec, device=dev)
        cache[key] = plan
    else:
        cache[key] = cache.pop(key)   # most recently used last
    return plan


# --- Gerchberg-Saxton ---------------------------------------------------------


def run_gs(cfg, target, illumination=None, progress=None, cancel=None):
    """Alternating-projection phase retrieval (algorithms.py:147-202) on the GPU."""
    start = time.perf_counter()
    target = np.asarray(target, dtype=np.complex128)
    _check_inputs(cfg, target, illumination)
    _init_code(cfg.init_mode)
    pb, keep = _problem(cfg, target)      # validates the propagation spec
    _mask_bytes(cfg, target)
    _native.library()
    _native.require_device()
    plan = _cached_plan(cfg, target.shape)
    plan.set_target(target, illumination, cfg=cfg, amplitude_only=cfg.init_mode == RANDOM_PHASE)
    hooks = _Hooks(progress, cancel) if (progress is not None or cancel is not None) else None
    out = _native.PrefaultedArrays(target.shape)    # faulted in while the device iterates
    rep, (tk, tv) = plan.gs(cfg=cfg, hooks=hooks)
    idx = plan.download_indices(1)[0]
    del keep
    holo = _native.expand_states(idx, states(cfg.slm.scheme), out=out.take()[0])
    return holo, RunReport(
        error_trace=_trace(tk, tv, rep.trace_len),
        final_error=float(rep.final_error),
        efficiency=float(rep.efficiency),
        iterations_executed=int(rep.iterations_executed),
        runtime_ms=_elapsed_ms(start),
        seed_used=cfg.seed,
        termination=_TERMINATION[rep.termination],
    )


def gs_field(cfg, target, illumination=None):
    """Parity helper: (index plane, pre-snap hologram field, report) of run_gs."""
    target = np.asarray(target, dtype=np.complex128)
    _check_inputs(cfg, target, illumination)
    pb, keep = _problem(cfg, target)
    mask = _mask_bytes(cfg, target)
    lib = _native.library()
    _native.require_device()
    tgt = _native.c128(target)
    ill = _illum(illumination)
    gp = _native.GsParams(int(cfg.iterations), float(cfg.feedback_gain), 1 if cfg.quantize_each_iteration else 0,
                          _init_code(cfg.init_mode), _native.Pcg64State.from_bitgen(np.random.PCG64(cfg.seed)))
    idx = _index_plane(pb.n_states, target.shape)
    fld = np.empty(target.shape, np.complex128)
    cap = max(0, int(cfg.iterations)) + 1
    tk = np.zeros(cap, np.int64)
    tv = np.zeros(cap, np.float64)
    rep = _native.Report()
    _native.check(lib.cgh_gs_run(ctypes.byref(pb), ctypes.byref(gp), _native.ptr(tgt), _native.ptr(mask),
                                 _native.ptr(ill), _native.ptr(idx), _native.ptr(fld), _native.ptr(tk),
                                 _native.ptr(tv), cap, ctypes.byref(rep), None))
    del keep
    return idx, fld, rep, _trace(tk, tv, rep.trace_len)


# --- one-step phase retrieval ---------------------------------------------------


def run_ospr(cfg, target, illumination=None, progress=None, cancel=None):
    """Randomised quantized backpropagations averaged in intensity (algorithms.py:473-530)."""
    start = time.perf_counter()
    target = np.asarray(target, dtype=np.complex128)
    _check_inputs(cfg, target, illumination)
    pb, keep = _problem(cfg, target)
    _mask_bytes(cfg, target)
    _native.library()
    _native.require_device()
    plan = _cached_plan(cfg, target.shape)
    plan.set_target(target, illumination, cfg=cfg, amplitude_only=True)   # OSPR never backpropagates
    hooks = _Hooks(progress, cancel) if (progress is not None or cancel is not None) else None
    out = _native.PrefaultedArrays(target.shape, max(0, int(cfg.subframes)))
    rep, (tk, tv) = plan.ospr(cfg=cfg, hooks=hooks)
    n = int(rep.iterations_executed)
    frames = []
    if n:
        idx = plan.download_indices(n)
        table = states(cfg.slm.scheme)
        bufs = out.take()
        frames = [_native.expand_states(idx[i], table, out=bufs[i]) for i in range(n)]
    del keep
    return frames, RunReport(
        error_trace=_trace(tk, tv, rep.trace_len),
        final_error=float(rep.final_error),
        efficiency=float(rep.efficiency),
        iterations_executed=n,
        runtime_ms=_elapsed_ms(start),
        seed_used=cfg.seed,
        termination=_TERMINATION[rep.termination],
    )


# --- simulated annealing / direct binary search ----------------------------------


def run_sa(cfg, target, illumination=None, progress=None, cancel=None, audit=None):
    """Simulated annealing over quantized pixel states (algorithms.py:343-404)."""
    from .search import sa_call

    return sa_call(cfg, target, illumination, progress, cancel, audit)


def run_dbs(cfg, target, illumination=None, progress=None, cancel=None, audit=None):
    """Direct binary search (algorithms.py:410-467)."""
    from .search import dbs_call

    return dbs_call(cfg, target, illumination, progress, cancel, audit)


RUNNERS = {GS: run_gs, SA: run_sa, DBS: run_dbs, OSPR: run_ospr}
