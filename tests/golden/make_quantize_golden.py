#!/usr/bin/env python3
"""Golden vectors for the standalone quantizer (slm.py:86-116) from the REAL
reference: the eight schemes of the reference's own test_slm.py:15-24, each
on the random values those tests draw (random_values, test_slm.py:27-29, seeds
0, 3, 4, 5) plus edge values: exact half-way ties between every pair of
neighbouring phase levels (including the wrap between L-1 and 0), the state
values themselves, signed zeros in every combination, angles of +-pi, pure
real / imaginary values and extreme magnitudes.

Run in the build container only (needs /root/reference):

    python tests/golden/make_quantize_golden.py
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

from make_golden import load_reference  # noqa: E402


def random_values(count, seed=0):
    gen = np.random.default_rng(seed)
    return (gen.normal(size=count) + 1j * gen.normal(size=count)).reshape(-1)


def edge_values(scheme, states):
    v = [complex(0.0, 0.0), complex(-0.0, 0.0), complex(0.0, -0.0), complex(-0.0, -0.0),
         complex(-1.0, 0.0), complex(-1.0, -0.0), complex(1.0, 0.0), complex(1.0, -0.0),
         complex(0.0, 1.0), complex(-0.0, 1.0), complex(0.0, -1.0), complex(-0.0, -1.0),
         complex(1e-300, 1e-300), complex(-1e300, 1e-300), complex(5e-324, -5e-324),
         complex(0.5, 0.0), complex(0.25, 0.0), complex(0.75, 0.0), complex(0.4999999999999999, 0.0)]
    v.extend(states)
    v.extend(-states)
    v.extend(0.5 * states)
    if hasattr(scheme, "phase_offset"):
        step = 2.0 * np.pi / scheme.levels
        k = np.arange(scheme.levels + 1)
        v.extend(np.exp(1j * (scheme.phase_offset + (k + 0.5) * step)))   # exact ties (as computed)
        v.extend(np.exp(1j * (scheme.phase_offset + k * step)))
        v.extend(np.exp(1j * (scheme.phase_offset + (k + 0.5) * step + np.array([[1e-15], [-1e-15]]))).ravel())
    return np.asarray(v, dtype=np.complex128)


def main():
    load_reference()
    from cghkit.slm import AmplitudeOnly, MultiAmp, PhaseOnly, quantize_indices, states

    schemes = [PhaseOnly(2), PhaseOnly(4), PhaseOnly(7, phase_offset=0.3), PhaseOnly(256), AmplitudeOnly(2),
               AmplitudeOnly(5), MultiAmp((0, 1)), MultiAmp((0.2 + 0.1j, -0.5, 1j, 0.9))]
    out = {}
    for i, s in enumerate(schemes):
        st = states(s)
        vals = np.concatenate([random_values(2000, 0), random_values(2000, 3), random_values(500, 4),
                               random_values(300, 5), edge_values(s, st)])
        out[f"values{i}"] = vals
        out[f"idx{i}"] = quantize_indices(vals, s).astype(np.int32)
        out[f"desc{i}"] = np.array(repr(s))
    np.savez_compressed(os.path.join(HERE, "quantize_golden.npz"), **out)
    print("schemes:", [str(out[f"desc{i}"]) for i in range(len(schemes))])


if __name__ == "__main__":
    main()
