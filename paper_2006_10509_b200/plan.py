"""Device-resident generation plans (``cgh_plan_*``): the target stays in HBM
across runs, index planes stay on the device until downloaded. Used by the
batched / multi-GPU layer and by bench.py for the inputs-resident timing."""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .algorithms import _init_code, _mask_bytes
from .propagation import fill_propagation
from .runtime import current_device, runner_precision
from .slm import problem_for

# pass ids reported by cgh_plan_profile
PASS_NAMES = {0: "row_fwd", 1: "row_inv", 2: "row_holo", 3: "row_init", 4: "ospr_gen", 5: "ospr_acc",
              8: "col_fwd", 9: "col_inv", 10: "col_gs", 11: "col_final", 12: "col_holo", 22: "ospr_loop", 23: "gs_loop"}


def plan_key(cfg, shape, precision, device):
    """Everything a plan bakes in: shape, precision, device, state table,
    propagation parameters, rescale flag."""
    from .slm import states

    p = cfg.propagation
    return (tuple(shape), int(precision), int(device), states(cfg.slm.scheme).tobytes(),
            float(getattr(cfg.slm.scheme, "phase_offset", 0.0)), p.kind, float(p.wavelength), float(p.distance),
            float(p.pitch_x), float(p.pitch_y), bool(cfg.metric.rescale))


class GenerationPlan:
    def __init__(self, cfg, shape, precision=None, device=None):
        self.lib = _native.library()
        _native.require_device()
        h, w = shape
        prec = runner_precision() if precision is None else precision
        dev = current_device() if device is None else device
        self.pb, self._keep = problem_for(cfg.slm.scheme, h, w, prec, dev)
        fill_propagation(self.pb, cfg.propagation)
        self.pb.rescale = 1 if cfg.metric.rescale else 0
        self.cfg = cfg
        self.shape = (h, w)
        self.handle = ctypes.c_void_p()
        _native.check(self.lib.cgh_plan_create(ctypes.byref(self.pb), ctypes.byref(self.handle)))
        self.idx_dtype = np.uint8 if self.pb.n_states <= 256 else np.int32

    def close(self):
        if self.handle:
            self.lib.cgh_plan_destroy(self.handle)
            self.handle = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    def set_target(self, target, illumination=None, cfg=None, amplitude_only=False):
        """Upload a target. ``amplitude_only``: the runs will not start from the
        backpropagated target (fp32 plans then upload only the shifted,
        mask-signed amplitude, built by host threads)."""
        target = _native.c128(target)
        mask = _mask_bytes(cfg or self.cfg, target)
        ill = None if illumination is None else _native.c128(illumination)
        _native.check(self.lib.cgh_plan_set_target_ex(self.handle, _native.ptr(target), _native.ptr(mask),
                                                      _native.ptr(ill), 1 if amplitude_only else 0))

    def gs(self, seed=None, iterations=None, with_trace=True, cfg=None, hooks=None):
        cfg = cfg or self.cfg
        gp = _native.GsParams()
        gp.iterations = int(cfg.iterations if iterations is None else iterations)
        gp.feedback_gain = float(cfg.feedback_gain)
        gp.quantize_each_iteration = 1 if cfg.quantize_each_iteration else 0
        gp.init_mode = _init_code(cfg.init_mode)
        gp.rng = _native.Pcg64State.from_bitgen(np.random.PCG64(cfg.seed if seed is None else seed))
        rep = _native.Report()
        cap = gp.iterations + 1
        tk = np.zeros(cap, np.int64) if with_trace else None
        tv = np.zeros(cap, np.float64) if with_trace else None
        st = self.lib.cgh_plan_gs(self.handle, ctypes.byref(gp), _native.ptr(tk), _native.ptr(tv),
                                  cap if with_trace else 0, ctypes.byref(rep),
                                  None if hooks is None else ctypes.byref(hooks.cb))
        if hooks is not None:
            hooks.raise_pending()
        _native.check(st)
        return rep, (tk, tv)

    def ospr(self, seed=None, subframes=None, cfg=None, hooks=None):
        cfg = cfg or self.cfg
        nsub = int(cfg.subframes if subframes is None else subframes)
        streams = np.random.SeedSequence(cfg.seed if seed is None else seed).spawn(nsub)
        fr = (_native.Pcg64State * max(1, nsub))()
        for i, s in enumerate(streams):
            fr[i] = _native.Pcg64State.from_bitgen(np.random.PCG64(s))
        op = _native.OsprParams(nsub, ctypes.cast(fr, ctypes.POINTER(_native.Pcg64State)))
        rep = _native.Report()
        tk = np.zeros(max(1, nsub), np.int64)
        tv = np.zeros(max(1, nsub), np.float64)
        st = self.lib.cgh_plan_ospr(self.handle, ctypes.byref(op), _native.ptr(tk), _native.ptr(tv),
                                    max(1, nsub), ctypes.byref(rep),
                                    None if hooks is None else ctypes.byref(hooks.cb))
        if hooks is not None:
            hooks.raise_pending()
        _native.check(st)
        return rep, (tk, tv)

    def ospr_part(self, streams, frame0, nframes_total, phase):
        """One contiguous part of a subframe-sharded OSPR run
        (cgh_plan_ospr_part): ``streams`` = the numpy SeedSequence children of
        these frames. Returns (report, per-frame error list)."""
        m = len(streams)
        fr = (_native.Pcg64State * max(1, m))()
        for i, sq in enumerate(streams):
            fr[i] = _native.Pcg64State.from_bitgen(np.random.PCG64(sq))
        op = _native.OsprParams(m, ctypes.cast(fr, ctypes.POINTER(_native.Pcg64State)))
        rep = _native.Report()
        tk = np.zeros(max(1, m), np.int64)
        tv = np.zeros(max(1, m), np.float64)
        _native.check(self.lib.cgh_plan_ospr_part(self.handle, ctypes.byref(op), int(frame0), int(nframes_total),
                                                  int(phase), _native.ptr(tk), _native.ptr(tv), max(1, m),
                                                  ctypes.byref(rep)))
        return rep, [(int(k), float(v)) for k, v in zip(tk[:m], tv[:m])]

    def intensity_ptr(self):
        """(device address, bytes) of the plan's carried intensity plane."""
        p, nbytes = ctypes.c_void_p(), ctypes.c_int64()
        _native.check(self.lib.cgh_plan_intensity(self.handle, ctypes.byref(p), ctypes.byref(nbytes)))
        return int(p.value or 0), int(nbytes.value)

    def copy_intensity(self, dst_ptr):
        """Copy the intensity plane to device address ``dst_ptr`` (H*W reals)."""
        _native.check(self.lib.cgh_plan_copy_intensity(self.handle, ctypes.c_void_p(int(dst_ptr))))

    def set_intensity(self, plane_ptrs):
        """intensity := sum of the device planes at ``plane_ptrs`` (fixed order)."""
        arr = (ctypes.c_void_p * max(1, len(plane_ptrs)))(*[ctypes.c_void_p(int(q)) for q in plane_ptrs])
        _native.check(self.lib.cgh_plan_set_intensity(self.handle, arr, len(plane_ptrs)))

    def sa(self, seed=None, proposals=None):
        """run_sa on the resident target (plan must be FP64)."""
        cfg = self.cfg
        sp = _native.SaParams()
        sp.proposals = int(cfg.proposals if proposals is None else proposals)
        t0 = cfg.initial_temperature
        sp.initial_temperature = -1.0 if t0 is None else float(t0)
        sp.cooling_factor = float(cfg.cooling_factor)
        sp.init_mode = _init_code(cfg.init_mode)
        sp.rng = _native.Pcg64State.from_bitgen(np.random.PCG64(cfg.seed if seed is None else seed))
        rep = _native.Report()
        cap = sp.proposals // max(1, sp.proposals // 1000) + 3
        tk = np.zeros(cap, np.int64)
        tv = np.zeros(cap, np.float64)
        _native.check(self.lib.cgh_plan_sa(self.handle, ctypes.byref(sp), _native.ptr(tk), _native.ptr(tv), cap,
                                           ctypes.byref(rep), None))
        return rep, (tk, tv)

    def dbs(self, seed=None, max_passes=None):
        """run_dbs (raster order) on the resident target (plan must be FP64)."""
        cfg = self.cfg
        dp = _native.DbsParams()
        dp.max_passes = int(cfg.max_passes if max_passes is None else max_passes)
        dp.scan_random = 0
        dp.init_mode = _init_code(cfg.init_mode)
        dp.rng = _native.Pcg64State.from_bitgen(np.random.PCG64(cfg.seed if seed is None else seed))
        rep = _native.Report()
        cap = dp.max_passes + 3
        tk = np.zeros(cap, np.int64)
        tv = np.zeros(cap, np.float64)
        _native.check(self.lib.cgh_plan_dbs(self.handle, ctypes.byref(dp), _native.ptr(tk), _native.ptr(tv), cap,
                                            ctypes.byref(rep), None))
        return rep, (tk, tv)

    def download_indices(self, frames=1):
        out = np.empty((frames,) + self.shape, self.idx_dtype)
        _native.check(self.lib.cgh_plan_download_idx(self.handle, _native.ptr(out), frames))
        return out

    def stream(self):
        return self.lib.cgh_plan_stream(self.handle)

    def sync(self):
        _native.check(self.lib.cgh_plan_sync(self.handle))

    def profile(self, enable):
        """Switch per-pass event timing; returns {pass: (ms_total, launches)} since the last call."""
        ms = np.zeros(24, np.float64)
        cnt = np.zeros(24, np.int64)
        _native.check(self.lib.cgh_plan_profile(self.handle, 1 if enable else 0, _native.ptr(ms), _native.ptr(cnt), 24))
        return {PASS_NAMES.get(i, f"pass{i}"): (float(ms[i]), int(cnt[i])) for i in range(24) if cnt[i]}
