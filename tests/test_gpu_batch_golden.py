"""The drop-in batch path against the REFERENCE batch driver.

tests/golden/batch_manifest.json records what cghkit.controller.run_batch
(controller.py:303-356) produced for a 6-job manifest shaped like the
reference's own acceptance test (pkg/tests/test_acceptance.py:292-345; script:
tests/golden/make_batch_golden.py): gs / sa / dbs / ospr on a 32x32 binary-phase
SLM, a job whose target file is missing, a job with an explicit seed; base seed
7, 2 workers. Here the same jobs run through multi.run_batch on the GPU in the
fp64 parity mode, two worker threads on one device: seeds derived from
(base seed, job id) as controller.py:95-97, one result per job in manifest
order, the failing job isolated as an error entry, and every output hologram
(each OSPR subframe) byte-identical to the reference's .hgi payload, also after
a round trip through the drop-in .hgi writer/reader.
"""

import hashlib
import json
import os

import numpy as np
import pytest

from paper_2006_10509_b200 import algorithms as A
from paper_2006_10509_b200.image import rect_mask
from paper_2006_10509_b200.multi import Job, derived_seed, run_batch
from paper_2006_10509_b200.propagation import MetricSpec, PropagationSpec
from paper_2006_10509_b200.runtime import device, precision
from paper_2006_10509_b200.serialio import Metadata, load_field, save_field
from paper_2006_10509_b200.slm import SlmSpec

from golden_cases import GOLDEN, scheme_from


def _doc():
    with open(os.path.join(GOLDEN, "batch_manifest.json")) as f:
        return json.load(f)


def _cfg(rec):
    c = rec["config"]
    p = c["propagation"]
    w, h = c["width"], c["height"]
    return A.AlgorithmConfig(algorithm=c["algorithm"], slm=SlmSpec(w, h, scheme_from(c["scheme"])),
                             propagation=PropagationSpec(p["kind"], p["wavelength"], p["distance"], p["pitch_x"],
                                                         p["pitch_y"]),
                             metric=MetricSpec(rect_mask(w, h), c["rescale"]), **c["params"])


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _fp64_runner(job, dev):
    with device(dev), precision("fp64"):
        if job.target is None:
            raise FileNotFoundError(job.meta["target"])
        return A.RUNNERS[job.cfg.algorithm](job.cfg, job.target, job.illumination)


def test_batch_golden_seeds_and_order():
    """Host side (no GPU): the drop-in's derived seeds reproduce the seeds the
    reference batch wrote, and the fixture holds one record per manifest job."""
    doc = _doc()
    ids = [rec["id"] for rec in doc["jobs"]]
    assert ids == [rec["row"]["job_id"] for rec in doc["jobs"]]
    for rec in doc["jobs"]:
        if "config" in rec and rec["id"] != "gs-b":
            assert derived_seed(doc["base_seed"], rec["id"]) == int(rec["row"]["seed"]) == rec["config"]["params"]["seed"]


@pytest.mark.gpu
def test_batch_matches_reference_controller(tmp_path):
    doc = _doc()
    targets = np.load(os.path.join(GOLDEN, "batch_targets.npz"))
    jobs = []
    for rec in doc["jobs"]:
        if "config" in rec:
            cfg = _cfg(rec)
            jobs.append(Job(rec["id"], cfg, targets[rec["id"]]))
        else:
            jobs.append(Job(rec["id"], None, None, meta={"target": "missing.png"}))
    results = run_batch(jobs, devices=[0, 0], runner=_fp64_runner)

    assert [r.job_id for r in results] == [rec["id"] for rec in doc["jobs"]]   # manifest order
    assert sum(r.error is not None for r in results) == doc["summary"]["failed"]
    for rec, res in zip(doc["jobs"], results):
        row = rec["row"]
        if "config" not in rec:
            assert row["output_file"].startswith("ERROR:") and res.error is not None
            continue
        assert res.error is None, (rec["id"], res.error)
        rep = res.report
        # seeds: the derived per-job seed (or the explicit one) the reference used
        if rec["id"] != "gs-b":
            assert derived_seed(doc["base_seed"], rec["id"]) == int(row["seed"])
        assert rep.seed_used == int(row["seed"])
        assert rep.iterations_executed == int(row["iterations"])
        assert abs(rep.final_error - float(row["final_error"])) <= 1e-10 * abs(float(row["final_error"])) + 1e-11
        assert abs(rep.efficiency - float(row["efficiency"])) <= 1e-11
        fields = res.hologram if isinstance(res.hologram, list) else [res.hologram]
        assert len(fields) == len(rec["outputs"])
        for field, out in zip(fields, rec["outputs"]):
            assert _sha(field) == out["payload_sha256"], (rec["id"], out["file"])
            assert abs(rep.final_error - out["error_final"]) <= 1e-10 * abs(out["error_final"])
            path = tmp_path / out["file"]
            save_field(field, Metadata([], rep.seed_used, "b200", "2026-01-01T00:00:00Z", rep_alg(rec),
                                       rep.final_error, rep.iterations_executed), str(path))
            back, meta = load_field(str(path))
            assert _sha(back) == out["payload_sha256"] and meta.seed == out["seed"]


def rep_alg(rec):
    return rec["config"]["algorithm"]
