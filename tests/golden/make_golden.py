#!/usr/bin/env python3
"""Regenerates tests/golden/*.npz from the REFERENCE itself (oracle/_ref/libmagfd_ref.so,
compiled from /root/reference/proj by oracle/Makefile).  Run here, where the reference
exists; the GPU box only reads the committed fixtures.

fields_small.npz: for each case, the spec, the input M (seeded), and the reference's
H_demag / H_eff (DemagConvolution::field, EffectiveFieldProvider::compute) in that
precision, plus 5-step torques and final M (Simulation::step).
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from oracle import oracle as O  # noqa: E402

CASES = [  # name, grid, precision
    ("g553_f64", (5, 3, 2, 1e-9, 2e-9, 3e-9), 64),
    ("g553_f32", (5, 3, 2, 1e-9, 2e-9, 3e-9), 32),
    ("g881_f64", (8, 8, 1, 2e-9, 2e-9, 2e-9), 64),
    ("g444_f64", (4, 4, 4, 2e-9, 2e-9, 2e-9), 64),
    ("g111_f64", (1, 1, 1, 2e-9, 2e-9, 2e-9), 64),
    ("sp4_f64", (128, 32, 1, 3.90625e-9, 3.90625e-9, 3e-9), 64),
    ("sp4_f32", (128, 32, 1, 3.90625e-9, 3.90625e-9, 3e-9), 32),
]


def spec(g):
    nx, ny, nz, dx, dy, dz = g
    return O.Spec(nx, ny, nz, dx, dy, dz, A=1.3e-11, Ku=4e4, Ms=8e5, alpha=0.5,
                  easy_axis=(0.6, 0.0, 0.8), h_ext=(2e4, -1e4, 3e4), dt=1e-14)


def main():
    assert O.ref_available(), "build oracle/_ref first (make -C oracle ref)"
    out = {}
    for i, (name, g, prec) in enumerate(CASES):
        s = spec(g)
        m = O.random_unit_field(s.n, s.Ms, 100 + i)
        if prec == 32:
            m = m.astype(np.float32).astype(np.float64)
        r = O.Ref(s, prec)
        r.set_m(m)
        out[name + "_spec"] = np.array(list(g) + [prec], dtype=np.float64)
        out[name + "_m"] = m
        out[name + "_hdemag"] = r.hdemag()
        out[name + "_heff"] = r.heff()
        out[name + "_torque5"] = r.step(5)
        out[name + "_m5"] = r.get_m()
    np.savez_compressed(os.path.join(os.path.dirname(os.path.abspath(__file__)), "fields_small.npz"), **out)


if __name__ == "__main__":
    main()
