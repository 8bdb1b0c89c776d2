#!/usr/bin/env python3
"""Generate golden vectors by running the REAL reference (cghkit) here.

Run in the build container only (needs /root/reference):

    python tests/golden/make_golden.py [--big]

The reference is built from a writable copy (the mount is read-only) with its
compiled incremental kernels; the script asserts ``BACKEND == "compiled"``.
It writes ``tests/golden/<case>.npz`` (index planes, traces, decision logs)
and ``tests/golden/manifest.json`` (configs + scalar results + sha256 of
every index plane). The reference itself is only read and called; SA/DBS
decision logs are captured by wrapping the reference's own methods from this
script (the reference source is not modified).

``--big`` adds the full-size BASELINE configs (C1-C4; ~10 min on one core).
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import shutil
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

from paper_2006_10509_b200.workloads import aperture_beam, gaussian_beam, natural_target, square_target  # noqa: E402

REF_COPY = os.environ.get("CGHKIT_BUILD", "/tmp/cghkit_golden_build")


def load_reference():
    src = os.path.join(REF_COPY, "src")
    if not os.path.exists(os.path.join(src, "cghkit")):
        shutil.rmtree(REF_COPY, ignore_errors=True)
        shutil.copytree("/root/reference/pkg", REF_COPY)
        subprocess.run([sys.executable, "setup.py", "build_ext", "--inplace"], cwd=REF_COPY,
                       check=True, stdout=subprocess.DEVNULL)
    sys.path.insert(0, src)
    import cghkit.kernels

    assert cghkit.kernels.BACKEND == "compiled", cghkit.kernels.BACKEND
    return cghkit


def sha(arr):
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()


def scheme_desc(s):
    if hasattr(s, "state_values"):
        return {"kind": "multi", "states": [[complex(v).real, complex(v).imag] for v in s.state_values]}
    if hasattr(s, "phase_offset"):
        return {"kind": "phase", "levels": s.levels, "offset": s.phase_offset}
    return {"kind": "amplitude", "levels": s.levels}


def small_cases(ck):
    from cghkit.image import rect_mask
    from cghkit.propagation import MetricSpec, PropagationSpec
    from cghkit.slm import AmplitudeOnly, MultiAmp, PhaseOnly, SlmSpec, binary_phase

    fres = PropagationSpec("fresnel", distance=0.05)
    cases = []

    def add(name, alg, n, scheme, target, *, prop=None, mask=None, rescale=False, illum=None,
            target_kind="natural", mask_rects=(), **kw):
        cfg = dict(algorithm=alg, slm=SlmSpec(n, n, scheme), propagation=prop or PropagationSpec(),
                   metric=MetricSpec(rect_mask(n, n, list(mask_rects)), rescale=rescale), **kw)
        cases.append(dict(name=name, cfg=cfg, target=target, illum=illum, target_kind=target_kind,
                          mask_rects=list(mask_rects), n=n))

    nat64 = natural_target(64)
    add("gs_fourier_64_pl256", "gs", 64, PhaseOnly(256), nat64, seed=1, iterations=30)
    add("gs_fresnel_64_pl8_gain_mask", "gs", 64, PhaseOnly(8), nat64, prop=fres, rescale=True,
        mask_rects=[(8, 10, 40, 36)], illum="beam", seed=2, iterations=25, feedback_gain=0.4)
    add("gs_binary_qeach_32", "gs", 32, binary_phase(), square_target(32), target_kind="square",
        seed=7, iterations=10, quantize_each_iteration=True)
    add("gs_backprop_fresnel_32_pl16", "gs", 32, PhaseOnly(16, 0.3), natural_target(32),
        prop=PropagationSpec("fresnel", distance=0.08), seed=4, iterations=12, init_mode="backpropagate")
    add("gs_amplitude_32", "gs", 32, AmplitudeOnly(4), natural_target(32), seed=5, iterations=8)
    add("gs_multiamp_32", "gs", 32, MultiAmp((0.2 + 0.1j, -0.5, 1j, 0.9)), natural_target(32),
        seed=6, iterations=8)
    add("gs_rect_128x64", "gs", 64, PhaseOnly(32), None, target_kind="rect128x64", seed=8, iterations=15)
    add("ospr_fourier_64_bin_8", "ospr", 64, binary_phase(), nat64, rescale=True, seed=1, subframes=8)
    add("ospr_fresnel_32_pl4_3", "ospr", 32, PhaseOnly(4), natural_target(32), prop=fres,
        mask_rects=[(4, 4, 20, 24)], illum="beam", seed=9, subframes=3)
    add("sa_32_bin_auto", "sa", 32, binary_phase(), square_target(32), target_kind="square",
        seed=5, proposals=3000)
    add("sa_16_pl4_fresnel_mask", "sa", 16, PhaseOnly(4), square_target(16), target_kind="square",
        prop=fres, rescale=True, mask_rects=[(2, 3, 9, 8)], seed=11, proposals=1500,
        initial_temperature=0.2, cooling_factor=0.999)
    add("sa_16_bin_t0", "sa", 16, binary_phase(), square_target(16), target_kind="square",
        seed=7, proposals=800, initial_temperature=0.0)
    add("dbs_16_bin_raster", "dbs", 16, binary_phase(), square_target(16), target_kind="square",
        seed=7, max_passes=6)
    add("dbs_16_pl4_random_fresnel", "dbs", 16, PhaseOnly(4), square_target(16), target_kind="square",
        prop=fres, mask_rects=[(2, 2, 12, 10)], seed=3, max_passes=4, scan_order="random")
    # exact-zero illumination (aperture): the reference snaps beam * exp(i angle)
    # with beam = 0 to the phase of a signed zero (complex multiply by 0 + 0j)
    add("gs_aperture_32_pl8", "gs", 32, PhaseOnly(8), natural_target(32), illum="aperture", seed=12,
        iterations=6)
    add("gs_aperture_32_bin_qeach", "gs", 32, binary_phase(), natural_target(32), illum="aperture",
        prop=fres, seed=13, iterations=5, quantize_each_iteration=True)
    add("ospr_aperture_32_bin_4", "ospr", 32, binary_phase(), natural_target(32), illum="aperture",
        seed=14, subframes=4)
    add("ospr_aperture_32_pl4_fresnel_3", "ospr", 32, PhaseOnly(4), natural_target(32), illum="aperture",
        prop=fres, seed=15, subframes=3)
    add("sa_16_aperture_bin", "sa", 16, binary_phase(), square_target(16), target_kind="square",
        illum="aperture", seed=16, proposals=600)
    add("dbs_16_aperture_pl4", "dbs", 16, PhaseOnly(4), square_target(16), target_kind="square",
        illum="aperture", seed=17, max_passes=3)
    for seed in (1, 2, 3, 4, 5):
        t = np.zeros((2, 2), complex)
        t[1, 1] = 1.0
        add(f"dbs_toy_2x2_seed{seed}", "dbs", 2, binary_phase(), t, target_kind="delta2", seed=seed,
            max_passes=20)
    return cases


def big_cases(ck):
    from cghkit.image import rect_mask
    from cghkit.propagation import MetricSpec, PropagationSpec
    from cghkit.slm import PhaseOnly, SlmSpec, binary_phase

    def mk(alg, n, scheme, prop, **kw):
        return dict(algorithm=alg, slm=SlmSpec(n, n, scheme), propagation=prop,
                    metric=MetricSpec(rect_mask(n, n), rescale=False), **kw)

    return [
        dict(name="C1_gs_fourier_512_pl256_100", n=512, target_kind="natural", illum=None, mask_rects=[],
             cfg=mk("gs", 512, PhaseOnly(256), PropagationSpec(), seed=1, iterations=100), target=None),
        dict(name="C2_ospr_1024_bin_24", n=1024, target_kind="natural", illum=None, mask_rects=[],
             cfg=mk("ospr", 1024, binary_phase(), PropagationSpec(), seed=1, subframes=24), target=None),
        dict(name="C3_gs_fresnel_2048_pl8_200", n=2048, target_kind="natural", illum=None, mask_rects=[],
             cfg=mk("gs", 2048, PhaseOnly(8), PropagationSpec("fresnel"), seed=1, iterations=200),
             target=None),
        dict(name="C4_sa_1024_bin_1e4", n=1024, target_kind="natural", illum=None, mask_rects=[],
             cfg=mk("sa", 1024, binary_phase(), PropagationSpec(), seed=3, proposals=10000), target=None,
             log=True),
        dict(name="C4_dbs_1024_bin_raster_1e4", n=1024, target_kind="natural", illum=None, mask_rects=[],
             cfg=mk("dbs", 1024, binary_phase(), PropagationSpec(), seed=3, max_passes=1), target=None,
             log=True, visits=10000),
    ]


class CountingCancel:
    """cancel.is_set() becomes True after ``limit`` polls (bounds a DBS run)."""

    def __init__(self, limit):
        self.limit = limit
        self.polls = 0

    def is_set(self):
        self.polls += 1
        return self.polls > self.limit


def make_target(case):
    n = case["n"]
    kind = case["target_kind"]
    if case["target"] is not None:
        return case["target"]
    if kind == "natural":
        return natural_target(n)
    if kind == "rect128x64":
        return natural_target(128, 64)
    raise ValueError(kind)


def run_case(ck, case, outdir):
    from cghkit import algorithms as A
    from cghkit.slm import SlmSpec

    target = make_target(case)
    cfgd = dict(case["cfg"])
    if case["target_kind"] == "rect128x64":
        cfgd["slm"] = SlmSpec(128, 64, cfgd["slm"].scheme)
        from cghkit.image import rect_mask
        from cghkit.propagation import MetricSpec
        cfgd["metric"] = MetricSpec(rect_mask(128, 64), rescale=False)
    cfg = A.AlgorithmConfig(**cfgd)
    h, w = target.shape
    illum = {"beam": gaussian_beam, "aperture": aperture_beam}.get(case["illum"])
    illum = None if illum is None else illum(h, w)
    log = []
    cancel = None
    undo = []
    if case.get("log") and cfg.algorithm == "sa":
        orig_draw = A._draw_proposal
        orig_commit = A._IncrementalState.commit

        def draw(rng, state):
            m, n, j = orig_draw(rng, state)
            log.append([m * state.width + n, j, 0])
            return m, n, j

        def commit(self, m, n, j, change):
            log[-1][2] = 1
            return orig_commit(self, m, n, j, change)

        A._draw_proposal = draw
        A._IncrementalState.commit = commit
        undo = [(A, "_draw_proposal", orig_draw), (A._IncrementalState, "commit", orig_commit)]
    if case.get("log") and cfg.algorithm == "dbs":
        orig_commit = A._IncrementalState.commit

        def commit(self, m, n, j, change):
            log.append([m * self.width + n, j, change])
            return orig_commit(self, m, n, j, change)

        A._IncrementalState.commit = commit
        undo = [(A._IncrementalState, "commit", orig_commit)]
        cancel = CountingCancel(case["visits"])
    try:
        out, rep = A.RUNNERS[cfg.algorithm](cfg, target, illum, cancel=cancel)
    finally:
        for obj, name, val in undo:
            setattr(obj, name, val)

    from cghkit.slm import quantize_indices

    frames = out if isinstance(out, list) else [out]
    idx = [quantize_indices(f, cfg.slm.scheme) for f in frames]
    # The returned holograms are bitwise state members; recover exact indices.
    from cghkit.slm import states

    st = states(cfg.slm.scheme)
    for f, ix in zip(frames, idx):
        assert np.array_equal(st[ix], f)
    dtype = np.uint8 if len(st) <= 256 else np.int32
    arrays = {f"idx{i}": ix.astype(dtype) for i, ix in enumerate(idx)}
    arrays["trace"] = np.array([e for _, e in rep.error_trace], dtype=np.float64)
    arrays["trace_k"] = np.array([k for k, _ in rep.error_trace], dtype=np.int64)
    if log:
        arrays["log"] = np.array(log, dtype=np.float64)
    big = case["n"] >= 512
    if big and cfg.algorithm == "ospr":
        keep = {k: v for k, v in arrays.items() if not k.startswith("idx")}
        keep["idx0"] = arrays["idx0"]
        keep[f"idx{len(idx) - 1}"] = arrays[f"idx{len(idx) - 1}"]
        arrays = keep
    np.savez_compressed(os.path.join(outdir, case["name"] + ".npz"), **arrays)
    rec = {
        "algorithm": cfg.algorithm,
        "height": h,
        "width": w,
        "scheme": scheme_desc(cfg.slm.scheme),
        "propagation": {k: getattr(cfg.propagation, k) for k in
                        ("kind", "wavelength", "distance", "pitch_x", "pitch_y")},
        "rescale": cfg.metric.rescale,
        "mask_rects": case["mask_rects"],
        "target": case["target_kind"],
        "illumination": case["illum"],
        "params": {k: getattr(cfg, k) for k in ("seed", "init_mode", "iterations", "feedback_gain",
                                                 "quantize_each_iteration", "proposals",
                                                 "initial_temperature", "cooling_factor",
                                                 "max_passes", "scan_order", "subframes")},
        "final_error": rep.final_error,
        "efficiency": rep.efficiency,
        "iterations_executed": rep.iterations_executed,
        "termination": rep.termination,
        "idx_sha256": [sha(ix.astype(dtype)) for ix in idx],
        "visits": case.get("visits"),
        "runtime_ms": rep.runtime_ms,
    }
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true")
    ap.add_argument("--only", default=None)
    args = ap.parse_args()
    ck = load_reference()
    import numpy

    man_path = os.path.join(HERE, "manifest.json")
    manifest = {"cases": {}}
    if os.path.exists(man_path):
        manifest = json.load(open(man_path))
    manifest["numpy"] = numpy.__version__
    manifest["generator"] = "tests/golden/make_golden.py (real reference, compiled backend)"
    cases = small_cases(ck) + (big_cases(ck) if args.big else [])
    for case in cases:
        if args.only and args.only not in case["name"]:
            continue
        rec = run_case(ck, case, HERE)
        manifest["cases"][case["name"]] = rec
        print(case["name"], rec["final_error"], f"{rec['runtime_ms']:.0f} ms", flush=True)
        json.dump(manifest, open(man_path, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
