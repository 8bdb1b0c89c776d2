#!/usr/bin/env python3
"""Golden record of the REFERENCE batch driver (cghkit.controller.run_batch,
controller.py:303-356) for the drop-in batch test (tests/test_gpu_batch_golden.py).

Run in the build container only (needs /root/reference):

    python tests/golden/make_batch_golden.py

A 6-job manifest in the shape of the reference's own acceptance test
(pkg/tests/test_acceptance.py:292-345: gs / sa / dbs / ospr jobs on a 32x32
binary-phase SLM, one job whose target file is missing, one job with an
explicit seed) is run by the reference's load_manifest + run_batch with
base seed 7 and 2 workers. Recorded in tests/golden/batch_manifest.json:
the results.csv rows (manifest order, the ERROR row), every job's resolved
configuration (the reference's own build_schema / apply_values /
configure_run, with the derived seed of controller.py:95-97), and for every
output .hgi the sha256 of its decoded payload (reference load_field) and its
metadata. The decoded targets go to tests/golden/batch_targets.npz.
"""

from __future__ import annotations

import csv
import hashlib
import json
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, HERE)
sys.path.insert(0, REPO)

from make_golden import load_reference, scheme_desc  # noqa: E402

from paper_2006_10509_b200.workloads import natural_target  # noqa: E402

BASE_SEED = 7
N = 32


def main():
    load_reference()
    from PIL import Image

    from cghkit import controller as C
    from cghkit.serialio import load_field

    tmp = tempfile.mkdtemp(prefix="cgh_batch_golden_")
    gray = np.clip(np.abs(natural_target(N)) * 255.0 + 0.5, 0, 255).astype(np.uint8)
    target_png = os.path.join(tmp, "target.png")
    Image.fromarray(gray, mode="L").save(target_png)
    small = {
        "projector/slm/slm-resolution-x": N,
        "projector/slm/slm-resolution-y": N,
        "projector/slm/slm-type": "binary-phase",
    }
    entries = [
        {"id": "gs-a", "target": target_png, "output": "gs-a",
         "overrides": {**small, "algorithm/run/algorithm/gs/iterations": 10}},
        {"id": "sa-a", "target": target_png, "output": "sa-a",
         "overrides": {**small, "algorithm/run/algorithm": "sa", "algorithm/run/algorithm/sa/proposals": 300}},
        {"id": "dbs-a", "target": target_png, "output": "dbs-a",
         "overrides": {**small, "algorithm/run/algorithm": "dbs", "algorithm/run/algorithm/dbs/max-passes": 2}},
        {"id": "ospr-a", "target": target_png, "output": "ospr-a",
         "overrides": {**small, "algorithm/run/algorithm": "ospr", "algorithm/run/algorithm/ospr/subframes": 2}},
        {"id": "broken", "target": os.path.join(tmp, "missing.png"), "output": "broken", "overrides": small},
        {"id": "gs-b", "target": target_png, "output": "gs-b",
         "overrides": {**small, "algorithm/run/algorithm/gs/iterations": 7, "algorithm/run/seed": 1234}},
    ]
    manifest = os.path.join(tmp, "manifest.json")
    with open(manifest, "w") as f:
        json.dump(entries, f)
    jobs = C.load_manifest(manifest)
    out_dir = os.path.join(tmp, "out")
    summary = C.run_batch(jobs, workers=2, out_dir=out_dir, base_seed=BASE_SEED)
    with open(os.path.join(out_dir, C.RESULTS_FILENAME), newline="") as fh:
        rows = list(csv.DictReader(fh))

    records, targets = [], {}
    for job, row in zip(jobs, rows):
        rec = {"id": job.id, "row": row}
        if row["output_file"].startswith("ERROR:"):
            records.append(rec)
            continue
        # the job's configuration exactly as _run_job resolves it (controller.py:303-313)
        tree = C.build_schema()
        C.apply_values(tree, job.overrides)
        if tree.get(C.PATH_SEED) == C.AUTO_SEED:
            tree.set(C.PATH_SEED, C._derived_seed(BASE_SEED, job.id))
        resolution = (tree.get(C.PATH_RESOLUTION_X), tree.get(C.PATH_RESOLUTION_Y))
        cfg = C.configure_run(tree)
        targets[job.id] = C.load_target(job.target_path, resolution)
        assert bool(np.all(cfg.metric.mask)), "the manifest uses the default full mask"
        rec["config"] = {
            "algorithm": cfg.algorithm,
            "width": cfg.slm.width,
            "height": cfg.slm.height,
            "scheme": scheme_desc(cfg.slm.scheme),
            "propagation": {k: getattr(cfg.propagation, k)
                            for k in ("kind", "wavelength", "distance", "pitch_x", "pitch_y")},
            "rescale": cfg.metric.rescale,
            "params": {k: getattr(cfg, k) for k in ("seed", "init_mode", "iterations", "feedback_gain",
                                                     "quantize_each_iteration", "proposals",
                                                     "initial_temperature", "cooling_factor",
                                                     "max_passes", "scan_order", "subframes")},
        }
        outs = []
        stem = job.output_name   # save_outputs: <stem>.hgi, or <stem>.frame<i>.hgi per OSPR subframe
        files = [f"{stem}.hgi"] if cfg.algorithm != "ospr" else [f"{stem}.frame{i}.hgi" for i in range(cfg.subframes)]
        for p in files:
            field, meta = load_field(os.path.join(out_dir, p))
            outs.append({"file": p,
                         "payload_sha256": hashlib.sha256(np.ascontiguousarray(field).tobytes()).hexdigest(),
                         "seed": meta.seed, "algorithm": meta.algorithm, "error_final": meta.error_final,
                         "iterations": meta.iterations})
        rec["outputs"] = outs
        records.append(rec)

    doc = {"generator": "tests/golden/make_batch_golden.py", "base_seed": BASE_SEED, "workers": 2,
           "numpy": np.__version__, "summary": {"total": summary.total, "succeeded": summary.succeeded,
                                               "failed": summary.failed},
           "jobs": records}
    with open(os.path.join(HERE, "batch_manifest.json"), "w") as f:
        json.dump(doc, f, indent=1)
    np.savez_compressed(os.path.join(HERE, "batch_targets.npz"), **targets)
    print(json.dumps(doc["summary"]), [r["id"] for r in records])


if __name__ == "__main__":
    main()
