"""Shared test helpers: build matching engine / oracle instances from one Spec."""
import numpy as np

from oracle import oracle as O


def engine_sim(spec: O.Spec, precision: int):
    import paper_1406_7459_b200 as E
    g = E.Grid(spec.nx, spec.ny, spec.nz, spec.dx, spec.dy, spec.dz)
    m = E.Material(spec.A, spec.Ku, spec.Ms, spec.alpha, spec.gamma, tuple(spec.easy_axis))
    f = E.FieldConfig(spec.exchange, spec.anisotropy, spec.demag, spec.zeeman, tuple(spec.h_ext))
    s = E.StepperConfig(spec.dt, spec.renorm_every, spec.max_steps, spec.torque_tol, spec.sample_every)
    return E.Simulation(g, m, f, s, precision=precision)


def checker(spec: O.Spec, precision: int):
    """The reference itself when its .so is present, else the C restatement (bitwise equal)."""
    return O.Ref(spec, precision) if O.ref_available() else O.Port(spec, precision)


def pair(spec: O.Spec, precision: int, m=None, seed=42):
    sim = engine_sim(spec, precision)
    ref = checker(spec, precision)
    if m is None:
        m = O.random_unit_field(spec.n, spec.Ms, seed)
    if precision == 32:
        m = m.astype(np.float32).astype(np.float64)
    sim.set_m(m)
    ref.set_m(m)
    return sim, ref, m
