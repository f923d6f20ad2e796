"""Write-overrun and determinism checks of the production kernels (the B200 pool
has compute-sanitizer closed, so the kernels are checked by guard bands and by
bitwise run-to-run repeatability instead).

* MFD_GUARD=1: every device buffer of the engine is bracketed by 4 KB of 0xA5;
  after fields, graph-chunked steps, asynchronous chunks, sampling (K5's
  last-block combine) and relax (device skip flags), no guard byte may have
  changed (mfd_debug_guard_check).
* Determinism: two engines fed the same input give bitwise identical M,
  torques, fields and sample sums (a shared-memory race or an unordered
  reduction would show up as run-to-run differences).
"""
import os

import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import engine_sim

pytestmark = pytest.mark.gpu

BENCH = dict(A=1.3e-11, Ku=4e4, Ms=8e5, alpha=0.02, easy_axis=(0.0, 0.0, 1.0), h_ext=(1e4, 0.0, 0.0), dt=1e-14)

CASES = [  # (grid, precision, env): the production variants of C1-C4 at test sizes
    ((128, 128, 64), 32, {}),                          # fused K1-in-K5 RS=0, C4 K3, K4 TMA L=256
    ((512, 512, 4), 32, {"MFD_FUSE_K1": "0"}),        # C4 x / y instantiations (K2/K4 TMA at 1024)
    ((512, 512, 4), 64, {"MFD_FUSE_K1": "0"}),
    ((512, 128, 4), 32, {}),                           # C2 (few-row K1/K5)
    ((128, 32, 1), 32, {}),                            # C1 SP4 (one-kernel y-z pass)
    ((128, 128, 128), 32, {}),                         # C3 (K3 at Pz = 256)
    ((33, 17, 5), 64, {}),                             # odd sizes, generic paths
]


def make(g, prec, env, guard=True):
    old = {}
    env = dict(env, MFD_GUARD="1" if guard else "0")
    for k, v in env.items():
        old[k] = os.environ.get(k)
        os.environ[k] = v
    try:
        s = O.Spec(*g, 2.5e-9, 2.5e-9, 2.5e-9, **BENCH, max_steps=150, torque_tol=1e-9, sample_every=50)
        return engine_sim(s, prec), s
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def exercise(sim, s, prec):
    m = O.random_unit_field(s.n, s.Ms, 77)
    sim.set_m(m)
    out = {"he": sim.effective_field(), "hd": sim.demag_field(),
           "he32": sim.effective_field(dtype=np.float32), "t": sim.step(20, return_all=True)}
    sim.step_async(70)
    sim.sync()
    out["m"] = sim.get_m()
    smp = sim.sample_now()
    out["smp"] = np.array(list(smp.m) + [smp.e_total, smp.max_torque_deg_per_ns])
    conv, log = sim.relax()
    out["relax"] = np.array([[x.step, x.e_total, x.max_torque_deg_per_ns] for x in log])
    out["m_relax"] = sim.get_m()
    return out


@pytest.mark.parametrize("g,prec,env", CASES)
def test_guard_bands_intact(g, prec, env):
    sim, s = make(g, prec, env)
    assert sim.guard_check() == 0
    exercise(sim, s, prec)
    assert sim.guard_check() == 0


@pytest.mark.parametrize("g,prec,env", CASES[:4])
def test_run_to_run_bitwise(g, prec, env):
    a, s = make(g, prec, env, guard=False)
    b, _ = make(g, prec, env, guard=False)
    ra, rb = exercise(a, s, prec), exercise(b, s, prec)
    for k in ra:
        assert np.array_equal(ra[k], rb[k]), k


def test_guard_bands_virtual_ranks():
    import paper_1406_7459_b200 as E
    os.environ["MFD_GUARD"] = "1"
    try:
        sim = E.Simulation(E.Grid(64, 32, 16, 2e-9, 2e-9, 2e-9), E.Material(A=1.3e-11, Ku=4e4, Ms=8e5, alpha=0.5),
                           E.FieldConfig(extern_field=(1e4, 0, 0)), E.StepperConfig(dt=1e-14), precision=32,
                           world=4, virtual_ranks=True)
    finally:
        os.environ.pop("MFD_GUARD", None)
    sim.set_m(O.random_unit_field(64 * 32 * 16, 8e5, 3))
    sim.step(5)
    sim.sample_now()
    assert sim.guard_check() == 0
