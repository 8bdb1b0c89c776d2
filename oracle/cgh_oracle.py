"""numpy restatement of the reference hologram-generation hot path.

TEST INFRASTRUCTURE ONLY — the checker, never the product. Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (CPU baseline / ``--impl
reference``) may import this module.

Every function restates one reference function and cites it. Citations are
relative to ``/root/reference/pkg/src/cghkit/``. The arithmetic deliberately
uses the same numpy calls in the same order as the reference so that the
oracle reproduces it bit-for-bit; this is checked against vectors produced by
the real reference (``tests/golden/make_golden.py``, ``tests/test_oracle.py``).

Parameter objects are duck-typed: anything with the attributes of the
reference's ``AlgorithmConfig`` / ``SlmSpec`` / ``PropagationSpec`` /
``MetricSpec`` works (the reference's own objects, the drop-in's mirrors, or
``types.SimpleNamespace``).
"""

from __future__ import annotations

import ctypes
import math
import os
import time
from dataclasses import dataclass, field

import numpy as np

# --------------------------------------------------------------------------
# scheme helpers (slm.py)
# --------------------------------------------------------------------------


def scheme_kind(scheme):
    """'phase' | 'amplitude' | 'multi' from attributes (slm.py:18-68)."""
    scheme = getattr(scheme, "scheme", scheme)
    if hasattr(scheme, "state_values"):
        return "multi"
    if hasattr(scheme, "phase_offset"):
        return "phase"
    if hasattr(scheme, "levels"):
        return "amplitude"
    raise TypeError(f"not a modulation scheme: {scheme!r}")


def state_table(scheme):
    """Allowed states as complex128 in index order — slm.py:71-79 (``states``)."""
    scheme = getattr(scheme, "scheme", scheme)
    kind = scheme_kind(scheme)
    if kind == "phase":
        k = np.arange(scheme.levels)
        return np.exp(1j * (scheme.phase_offset + 2.0 * np.pi * k / scheme.levels))
    if kind == "amplitude":
        return (np.arange(scheme.levels) / (scheme.levels - 1)).astype(np.complex128)
    return np.asarray(scheme.state_values, dtype=np.complex128)


def nearest_state_index(values, scheme):
    """Nearest-state index plane — slm.py:86-108 (``quantize_indices``).

    Phase-only: closed-form level from the angle with the half-way tie kept
    on the lower index (wrapping to 0). Other schemes: first argmin of |z - s|.
    """
    scheme = getattr(scheme, "scheme", scheme)
    values = np.asarray(values, dtype=np.complex128)
    if scheme_kind(scheme) == "phase":
        levels = scheme.levels
        step = 2.0 * np.pi / levels
        frac = np.mod((np.angle(values) - scheme.phase_offset) / step, levels)
        low = np.floor(frac)
        rem = frac - low
        low = low.astype(np.int64)
        high = (low + 1) % levels
        pick = np.where(rem < 0.5, low, high)
        pick = np.where(rem == 0.5, np.minimum(low, high), pick)
        return np.mod(pick, levels).astype(np.int32)
    table = state_table(scheme)
    dist = np.abs(values.reshape(-1, 1) - table[None, :])
    return np.argmin(dist, axis=1).astype(np.int32).reshape(values.shape)


def snap(values, scheme):
    """slm.py:111-116 (``quantize``) for arrays."""
    return state_table(scheme)[nearest_state_index(values, scheme)]


# --------------------------------------------------------------------------
# propagation (propagation.py)
# --------------------------------------------------------------------------


class OracleInputError(Exception):
    """Raised where the reference raises one of its CghError subclasses.

    ``kind`` holds the reference class name (errors.py:79-108).
    """

    def __init__(self, kind, message):
        super().__init__(f"{kind}: {message}")
        self.kind = kind


def _finite_or_raise(arr):
    # propagation.py:66-68
    if not np.all(np.isfinite(arr)):
        raise OracleInputError("NonFiniteError", "field contains NaN or Inf")


def centred_dft(field, direction="forward"):
    """Unitary centred 2-D DFT — propagation.py:81-94 (``fft2``)."""
    field = np.asarray(field, dtype=np.complex128)
    _finite_or_raise(field)
    if direction == "forward":
        return np.fft.fftshift(np.fft.fft2(field, norm="ortho"))
    if direction == "inverse":
        return np.fft.ifft2(np.fft.ifftshift(field), norm="ortho")
    raise ValueError(f"bad direction {direction!r}")


def _check_spec(spec):
    # propagation.py:48-55
    if spec.kind not in ("fourier", "fresnel"):
        raise OracleInputError("InvalidSpecError", f"unknown propagation kind {spec.kind!r}")
    if spec.kind == "fresnel":
        if spec.wavelength <= 0 or spec.pitch_x <= 0 or spec.pitch_y <= 0:
            raise OracleInputError("InvalidSpecError", "positive wavelength and pitches")
        if spec.distance == 0:
            raise OracleInputError("InvalidSpecError", "nonzero distance")


def quadratic_phase(shape, spec):
    """Fresnel prefactor — propagation.py:97-107 (``fresnel_prefactor``)."""
    height, width = shape
    m = np.arange(height) - height / 2.0
    n = np.arange(width) - width / 2.0
    quad = (
        np.pi
        * ((m * m * spec.pitch_y**2)[:, None] + (n * n * spec.pitch_x**2)[None, :])
        / (spec.wavelength * spec.distance)
    )
    return np.exp(1j * quad)


def to_replay(field, spec):
    """propagation.py:110-115 (``propagate``)."""
    _check_spec(spec)
    if spec.kind == "fourier":
        return centred_dft(field, "forward")
    return centred_dft(np.asarray(field, dtype=np.complex128) * quadratic_phase(field.shape, spec), "forward")


def to_hologram(replay, spec):
    """propagation.py:118-123 (``propagate_inverse``)."""
    _check_spec(spec)
    if spec.kind == "fourier":
        return centred_dft(replay, "inverse")
    return np.conj(quadratic_phase(replay.shape, spec)) * centred_dft(replay, "inverse")


def amplitude_error(replay, target, mask, rescale):
    """Masked amplitude MSE — propagation.py:164-192 (``mse_error``)."""
    replay = np.asarray(replay)
    target = np.asarray(target)
    if replay.shape != target.shape or mask.shape != target.shape:
        raise OracleInputError("DimensionMismatchError", "shapes differ")
    if not mask.any():
        raise OracleInputError("EmptyMaskError", "empty mask")
    r = np.abs(replay[mask])
    t = np.abs(target[mask])
    denom = float(np.sum(t * t))
    if denom == 0.0:
        raise OracleInputError("ZeroTargetError", "target zero in mask")
    if rescale:
        rr = float(np.sum(r * r))
        s = float(np.sum(r * t)) / rr if rr > 0.0 else 1.0
    else:
        s = 1.0
    diff = s * r - t
    return float(np.sum(diff * diff) / denom)


def in_mask_energy_fraction(replay, mask):
    """propagation.py:195-202 (``efficiency``)."""
    replay = np.asarray(replay)
    inten = replay.real**2 + replay.imag**2
    total = float(np.sum(inten))
    if total == 0.0:
        raise OracleInputError("ZeroFieldError", "replay field is zero")
    return float(np.sum(inten[mask]) / total)


def rank_one_update(replay, m, n, delta):
    """propagation.py:205-218 (``delta_replay_update``), in place."""
    height, width = replay.shape
    row = np.exp(-2j * np.pi * m / height * np.arange(height))
    col = np.exp(-2j * np.pi * n / width * np.arange(width))
    replay += (delta / np.sqrt(height * width)) * np.outer(row, col)


# --------------------------------------------------------------------------
# runners (algorithms.py)
# --------------------------------------------------------------------------


@dataclass
class OracleReport:
    """Mirror of RunReport (algorithms.py:84-94) plus checker extras."""

    error_trace: list
    final_error: float
    efficiency: float
    iterations_executed: int
    runtime_ms: float
    seed_used: int
    termination: str
    indices: object = None          # final index plane(s)
    fields: dict = field(default_factory=dict)   # GS: iteration -> pre-quantization field
    log: list = field(default_factory=list)      # SA/DBS decision log


def _shape_check(cfg, target, illumination):
    # algorithms.py:97-108
    shape = (cfg.slm.height, cfg.slm.width)
    if target.shape != shape:
        raise OracleInputError("DimensionMismatchError", f"target {target.shape} vs {shape}")
    if illumination is not None and illumination.shape != shape:
        raise OracleInputError("DimensionMismatchError", "illumination shape")


def _beam(target, illumination):
    # algorithms.py:111-114
    if illumination is None:
        return np.ones(target.shape, dtype=np.float64)
    return np.abs(illumination)


def start_field(target, illumination, mode, rng, spec):
    """algorithms.py:117-137 (``initial_hologram``)."""
    target = np.asarray(target, dtype=np.complex128)
    if illumination is not None and illumination.shape != target.shape:
        raise OracleInputError("DimensionMismatchError", "illumination shape")
    amp = _beam(target, illumination)
    if mode == "random-phase":
        theta = 2.0 * np.pi * rng.random(target.shape)
        return amp * np.exp(1j * theta)
    if mode == "backpropagate":
        back = to_hologram(target, spec)
        return amp * np.exp(1j * np.angle(back))
    raise ValueError(f"unknown init mode {mode!r}")


def _elapsed(t0):
    return (time.perf_counter() - t0) * 1000.0


def gs(cfg, target, illumination=None, progress=None, cancel=None, keep_fields=()):
    """Gerchberg-Saxton — algorithms.py:147-202 (``run_gs``).

    ``keep_fields``: iteration counts k (1-based, after the k-th hologram
    update) whose complex hologram-plane field is stored in ``report.fields``.
    """
    t0 = time.perf_counter()
    target = np.asarray(target, dtype=np.complex128)
    _shape_check(cfg, target, illumination)
    rng = np.random.Generator(np.random.PCG64(cfg.seed))
    holo = start_field(target, illumination, cfg.init_mode, rng, cfg.propagation)
    beam = _beam(target, illumination)
    tamp = np.abs(target)
    mask = cfg.metric.mask
    keep = set(keep_fields)
    stored = {}

    trace = []
    done = 0
    stopped = False
    for k in range(cfg.iterations):
        if cancel is not None and cancel.is_set():
            stopped = True
            break
        replay = to_replay(holo, cfg.propagation)
        err = amplitude_error(replay, target, mask, cfg.metric.rescale)
        trace.append((k, err))
        if progress is not None:
            progress(k, err)
        want = tamp + cfg.feedback_gain * (tamp - np.abs(replay))
        np.clip(want, 0.0, None, out=want)
        projected = np.where(mask, want * np.exp(1j * np.angle(replay)), replay)
        holo = to_hologram(projected, cfg.propagation)
        holo = beam * np.exp(1j * np.angle(holo))
        if cfg.quantize_each_iteration:
            holo = snap(holo, cfg.slm)
        done = k + 1
        if done in keep:
            stored[done] = holo.copy()

    idx = nearest_state_index(holo, cfg.slm)
    holo = state_table(cfg.slm)[idx]
    replay = to_replay(holo, cfg.propagation)
    final = amplitude_error(replay, target, mask, cfg.metric.rescale)
    trace.append((done, final))
    if progress is not None:
        progress(done, final)
    return holo, OracleReport(
        error_trace=trace,
        final_error=final,
        efficiency=in_mask_energy_fraction(replay, mask),
        iterations_executed=done,
        runtime_ms=_elapsed(t0),
        seed_used=cfg.seed,
        termination="cancelled" if stopped else "completed",
        indices=idx,
        fields=stored,
    )


# ---- incremental search state (algorithms.py:208-306) ---------------------

_LIB = None


def _incr_lib():
    """The C restatement of _core.pyx (oracle/incremental.c), or None."""
    global _LIB
    if _LIB is None:
        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_build", "liboracle_incr.so")
        if not os.path.exists(path):
            _LIB = False
        else:
            lib = ctypes.CDLL(path)
            p = ctypes.c_void_p
            i64 = ctypes.c_int64
            d = ctypes.c_double
            lib.oracle_delta_error.argtypes = [p, p, p, p, p, p, i64, d, d]
            lib.oracle_delta_error.restype = d
            lib.oracle_commit.argtypes = [p, p, p, p, p, i64, d, d]
            lib.oracle_commit.restype = None
            lib.oracle_best_delta.argtypes = [p, p, p, p, p, p, i64, p, i64, p]
            lib.oracle_best_delta.restype = i64
            _LIB = lib
    return _LIB or None


def build_incremental_lib():
    """Compile oracle/incremental.c with oracle/Makefile (gcc only)."""
    import subprocess

    here = os.path.dirname(os.path.abspath(__file__))
    subprocess.run(["make", "-s", "-C", here], check=True)
    global _LIB
    _LIB = None
    return _incr_lib() is not None


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


class PixelSearchState:
    """Masked uncentred replay kept in sync with a quantized pixel grid.

    Restates ``_IncrementalState`` (algorithms.py:208-306); the three kernel
    calls go to the C restatement of ``_core.pyx`` (bit-exact with the
    reference's compiled backend) or, if it is not built, to a numpy
    restatement of ``_pure.py`` (not bit-exact: np.abs uses hypot).
    """

    def __init__(self, cfg, target, start):
        self.height, self.width = target.shape
        self.size = self.height * self.width
        self.table = state_table(cfg.slm)
        self.n_states = len(self.table)
        self.idx = nearest_state_index(start, cfg.slm)
        self.q = quadratic_phase(target.shape, cfg.propagation) if cfg.propagation.kind == "fresnel" else None
        pix = self.table[self.idx]
        if self.q is not None:
            pix = pix * self.q
        replay = np.fft.fft2(pix, norm="ortho")
        mu, mv = np.nonzero(np.fft.ifftshift(cfg.metric.mask))
        self.mu = np.ascontiguousarray(mu, dtype=np.int32)
        self.mv = np.ascontiguousarray(mv, dtype=np.int32)
        tu = np.fft.ifftshift(np.abs(target))
        self.t = np.ascontiguousarray(tu[mu, mv], dtype=np.float64)
        self.r = np.ascontiguousarray(replay[mu, mv], dtype=np.complex128)
        self.denom = float(np.sum(self.t * self.t))
        if self.denom == 0.0:
            raise OracleInputError("ZeroTargetError", "target is zero inside the mask")
        d = np.abs(self.r) - self.t
        self.num = float(np.sum(d * d))
        hi = np.arange(self.height)
        wi = np.arange(self.width)
        self.rows = np.exp(-2j * np.pi * np.outer(hi, hi) / self.height)
        self.cols = np.exp(-2j * np.pi * np.outer(wi, wi) / self.width)
        self.cols /= math.sqrt(self.size)
        self.lib = _incr_lib()

    def _delta(self, m, n, j):
        # algorithms.py:253-257
        dv = self.table[j] - self.table[self.idx[m, n]]
        if self.q is not None:
            dv = dv * self.q[m, n]
        return dv

    def change(self, m, n, j):
        # algorithms.py:259-268 -> _core.pyx:20-34
        dv = complex(self._delta(m, n, j))
        row = self.rows[m]
        col = self.cols[n]
        if self.lib:
            return float(self.lib.oracle_delta_error(
                _ptr(self.r), _ptr(self.t), _ptr(row), _ptr(col),
                _ptr(self.mu), _ptr(self.mv), len(self.t), dv.real, dv.imag))
        w = row[self.mu] * col[self.mv]
        d0 = np.abs(self.r) - self.t
        d1 = np.abs(self.r + dv * w) - self.t
        return float(np.sum(d1 * d1 - d0 * d0))

    def best(self, m, n):
        # algorithms.py:270-282 -> _core.pyx:47-83
        deltas = self.table - self.table[self.idx[m, n]]
        if self.q is not None:
            deltas = deltas * self.q[m, n]
        deltas = np.ascontiguousarray(deltas)
        row = self.rows[m]
        col = self.cols[n]
        if self.lib:
            out = ctypes.c_double(0.0)
            j = self.lib.oracle_best_delta(
                _ptr(self.r), _ptr(self.t), _ptr(row), _ptr(col),
                _ptr(self.mu), _ptr(self.mv), len(self.t), _ptr(deltas), len(deltas),
                ctypes.byref(out))
            if j == -2:
                raise MemoryError()
            return int(j), float(out.value)
        w = row[self.mu] * col[self.mv]
        d0 = np.abs(self.r) - self.t
        best_j, best_c = -1, 0.0
        for j, dv in enumerate(deltas):
            if dv == 0:
                continue
            d1 = np.abs(self.r + dv * w) - self.t
            c = float(np.sum(d1 * d1 - d0 * d0))
            if c < best_c:
                best_j, best_c = j, c
        return best_j, best_c

    def apply(self, m, n, j, change):
        # algorithms.py:284-294 -> _core.pyx:37-44
        dv = complex(self._delta(m, n, j))
        row = self.rows[m]
        col = self.cols[n]
        if self.lib:
            self.lib.oracle_commit(_ptr(self.r), _ptr(row), _ptr(col),
                                   _ptr(self.mu), _ptr(self.mv), len(self.t), dv.real, dv.imag)
        else:
            self.r += dv * (row[self.mu] * col[self.mv])
        self.idx[m, n] = j
        self.num += change

    def reported(self, rescale):
        # algorithms.py:296-303
        if not rescale:
            return self.num / self.denom
        r = np.abs(self.r)
        rr = float(np.sum(r * r))
        s = float(np.sum(r * self.t)) / rr if rr > 0.0 else 1.0
        d = s * r - self.t
        return float(np.sum(d * d) / self.denom)

    def hologram(self):
        return self.table[self.idx]


def _finish(cfg, st, trace, done, t0, how, progress, log):
    """algorithms.py:309-328 (``_final_report``)."""
    final = st.reported(cfg.metric.rescale)
    if not trace or trace[-1][1] != final:
        trace.append((done, final))
        if progress is not None:
            progress(done, final)
    holo = st.hologram()
    replay = to_replay(holo, cfg.propagation)
    return holo, OracleReport(
        error_trace=trace,
        final_error=final,
        efficiency=in_mask_energy_fraction(replay, cfg.metric.mask),
        iterations_executed=done,
        runtime_ms=_elapsed(t0),
        seed_used=cfg.seed,
        termination=how,
        indices=st.idx.copy(),
        log=log,
    )


def _propose(rng, st):
    """algorithms.py:334-340 (``_draw_proposal``)."""
    p = int(rng.integers(st.size))
    m, n = divmod(p, st.width)
    j = int(rng.integers(st.n_states - 1))
    if j >= st.idx[m, n]:
        j += 1
    return m, n, j


def sa(cfg, target, illumination=None, progress=None, cancel=None, audit=None,
       log_limit=0, stop_after=None):
    """Simulated annealing — algorithms.py:343-404 (``run_sa``).

    ``log_limit``: record (pixel, level, accepted) for the first N proposals.
    ``stop_after``: checker-only shortcut ending the run after N proposals
    (reported as completed with the trace so far), for bounded CPU samples.
    """
    t0 = time.perf_counter()
    target = np.asarray(target, dtype=np.complex128)
    _shape_check(cfg, target, illumination)
    rng = np.random.Generator(np.random.PCG64(cfg.seed))
    start = start_field(target, illumination, cfg.init_mode, rng, cfg.propagation)
    st = PixelSearchState(cfg, target, start)
    trace = [(0, st.reported(cfg.metric.rescale))]
    if progress is not None:
        progress(0, trace[0][1])

    temp = cfg.initial_temperature
    if temp is None or temp < 0:
        acc = 0.0
        for _ in range(100):                      # algorithms.py:54, 369-375
            m, n, j = _propose(rng, st)
            acc += abs(st.change(m, n, j)) / st.denom
        temp = acc / 100

    every = max(1, cfg.proposals // 1000)
    done = 0
    stopped = False
    log = []
    total = cfg.proposals if stop_after is None else min(cfg.proposals, stop_after)
    for k in range(total):
        if cancel is not None and cancel.is_set():
            stopped = True
            break
        m, n, j = _propose(rng, st)
        ch = st.change(m, n, j)
        x = ch / st.denom
        ok = x < 0.0
        if not ok and temp > 0.0:
            ok = rng.random() < math.exp(-x / temp)
        if ok:
            st.apply(m, n, j, ch)
        if k < log_limit:
            log.append((m * st.width + n, j, bool(ok)))
        temp *= cfg.cooling_factor
        done = k + 1
        if done % every == 0:
            e = st.reported(cfg.metric.rescale)
            trace.append((done, e))
            if progress is not None:
                progress(done, e)
            if audit is not None:
                audit(done, st.num / st.denom, st.hologram())
    return _finish(cfg, st, trace, done, t0, "cancelled" if stopped else "completed", progress, log)


def dbs(cfg, target, illumination=None, progress=None, cancel=None, audit=None,
        log_limit=0, stop_after=None):
    """Direct binary search — algorithms.py:410-467 (``run_dbs``).

    ``log_limit``: record (pixel, level, change) for the first N pixel visits
    (level -1 = no commit). ``stop_after``: checker-only bound on pixel visits.
    """
    t0 = time.perf_counter()
    target = np.asarray(target, dtype=np.complex128)
    _shape_check(cfg, target, illumination)
    root = np.random.SeedSequence(cfg.seed)
    rng = np.random.Generator(np.random.PCG64(root))
    start = start_field(target, illumination, cfg.init_mode, rng, cfg.propagation)
    st = PixelSearchState(cfg, target, start)
    trace = [(0, st.reported(cfg.metric.rescale))]
    if progress is not None:
        progress(0, trace[0][1])

    passes = 0
    stopped = False
    settled = False
    visits = 0
    log = []
    for _ in range(cfg.max_passes):
        if cfg.scan_order == "random":
            prng = np.random.Generator(np.random.PCG64(root.spawn(1)[0]))
            order = prng.permutation(st.size)
        else:
            order = range(st.size)
        commits = 0
        for p in order:
            if cancel is not None and cancel.is_set():
                stopped = True
                break
            if stop_after is not None and visits >= stop_after:
                stopped = True
                break
            m, n = divmod(int(p), st.width)
            j, ch = st.best(m, n)
            took = j >= 0 and ch < 0.0
            if took:
                st.apply(m, n, j, ch)
                commits += 1
            if visits < log_limit:
                log.append((int(p), j if took else -1, ch))
            visits += 1
        if stopped:
            break
        passes += 1
        if commits > 0:
            e = st.reported(cfg.metric.rescale)
            trace.append((passes, e))
            if progress is not None:
                progress(passes, e)
            if audit is not None:
                audit(passes, st.num / st.denom, st.hologram())
        else:
            settled = True
            break
    how = "cancelled" if stopped else ("converged" if settled else "completed")
    return _finish(cfg, st, trace, passes, t0, how, progress, log)


def ospr(cfg, target, illumination=None, progress=None, cancel=None):
    """One-step phase retrieval — algorithms.py:473-530 (``run_ospr``)."""
    t0 = time.perf_counter()
    target = np.asarray(target, dtype=np.complex128)
    _shape_check(cfg, target, illumination)
    beam = _beam(target, illumination)
    tamp = np.abs(target)
    children = np.random.SeedSequence(cfg.seed).spawn(cfg.subframes)

    frames = []
    idxs = []
    acc = np.zeros(target.shape, dtype=np.float64)
    trace = []
    stopped = False
    for child in children:
        if cancel is not None and cancel.is_set():
            stopped = True
            break
        rng = np.random.Generator(np.random.PCG64(child))
        theta = 2.0 * np.pi * rng.random(target.shape)
        sub = tamp * np.exp(1j * theta)
        holo = to_hologram(sub, cfg.propagation)
        idx = nearest_state_index(beam * np.exp(1j * np.angle(holo)), cfg.slm)
        holo = state_table(cfg.slm)[idx]
        frames.append(holo)
        idxs.append(idx)
        replay = to_replay(holo, cfg.propagation)
        acc += replay.real**2 + replay.imag**2
        seen = np.sqrt(acc / len(frames))
        e = amplitude_error(seen, target, cfg.metric.mask, cfg.metric.rescale)
        trace.append((len(frames), e))
        if progress is not None:
            progress(len(frames), e)
    if frames:
        seen = np.sqrt(acc / len(frames))
        eta = in_mask_energy_fraction(seen, cfg.metric.mask)
        final = trace[-1][1]
    else:
        seen = np.zeros(target.shape)
        eta = 0.0
        final = amplitude_error(seen, target, cfg.metric.mask, cfg.metric.rescale)
        trace.append((0, final))
    return frames, OracleReport(
        error_trace=trace,
        final_error=final,
        efficiency=eta,
        iterations_executed=len(frames),
        runtime_ms=_elapsed(t0),
        seed_used=cfg.seed,
        termination="cancelled" if stopped else "completed",
        indices=idxs,
    )


RUN = {"gs": gs, "sa": sa, "dbs": dbs, "ospr": ospr}
