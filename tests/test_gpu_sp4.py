"""muMAG standard problem 4 trajectory parity (BASELINE north_star: <m>(t)
within 1e-4 of the reference over the standard-problem trajectory).

Fixtures from the reference itself (tests/golden/make_sp4.py):
* relax from uniform (1,1,1)/sqrt3, alpha = 1, to 0.01 deg/ns (dynamics::relax),
  in f64 (sp4_relax.npz) and in the reference's own f32 (sp4_relax_f32.npz);
* field 1 from the reference s-state, 200 ps.  SP4 field 1 is chaotic
  (a 1e-15 perturbation reaches 1e-4 at ~0.21-0.26 ns
  f64-vs-f64, f32-vs-f64 at 87 ps), so the windows are [0, 200 ps] in f64 and
  [0, 80 ps] in f32.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
GRID = (128, 32, 1, 500e-9 / 128, 125e-9 / 32, 3e-9)
MU0 = 4e-7 * np.pi


def sim(prec, alpha, h, **st):
    import paper_1406_7459_b200 as E
    return E.Simulation(E.Grid(*GRID), E.Material(A=1.3e-11, Ku=0.0, Ms=8e5, alpha=alpha),
                        E.FieldConfig(True, False, True, h is not None, h or (0.0, 0.0, 0.0)),
                        E.StepperConfig(dt=5e-14, **st), precision=prec)


def test_sp4_relax_trajectory_f64():
    path = os.path.join(HERE, "sp4_relax.npz")
    if not os.path.exists(path):
        pytest.skip("fixture not generated")
    z = np.load(path)
    ref = z["samples"]                        # step, t, mx, my, mz, torque, E_total
    s = sim(64, 1.0, None, max_steps=200000, torque_tol_deg_per_ns=0.01, sample_every=100)
    s.set_m(np.full((3, 4096), 8e5 / np.sqrt(3.0)))
    conv, log = s.relax()
    assert conv == bool(z["converged"])
    mine = {x.step: x for x in log}
    common = [int(r[0]) for r in ref if int(r[0]) in mine]
    assert len(common) >= 0.95 * len(ref)
    worst = max(np.max(np.abs(mine[k].m - ref[ref[:, 0] == k][0, 2:5])) for k in common)
    assert worst <= 1e-4, worst
    assert log[-1].step == int(ref[-1, 0])    # same convergence step
    assert np.max(np.abs(log[-1].m - ref[-1, 2:5])) <= 1e-4


def test_sp4_relax_trajectory_f32():
    """The reference's own f32 relax never reaches 0.01 deg/ns: its torque
    settles on an f32 rounding floor (~0.063 deg/ns, sp4_relax_f32.npz) and the
    run ends at max_steps.  Parity: same outcome, <m> within 1e-4 of the f64
    trajectory while it runs and of the reference f32 state at the end."""
    p64, p32 = os.path.join(HERE, "sp4_relax.npz"), os.path.join(HERE, "sp4_relax_f32.npz")
    if not (os.path.exists(p64) and os.path.exists(p32)):
        pytest.skip("fixture not generated")
    ref64, z32 = np.load(p64)["samples"], np.load(p32)
    ref32 = z32["samples"]
    s = sim(32, 1.0, None, max_steps=200000, torque_tol_deg_per_ns=0.01, sample_every=1000)
    s.set_m(np.full((3, 4096), 8e5 / np.sqrt(3.0)))
    conv, log = s.relax()
    assert conv == bool(z32["converged"]) and not conv
    assert log[-1].step == int(ref32[-1, 0])
    mine = {x.step: x for x in log}
    common = [int(r[0]) for r in ref64 if int(r[0]) in mine]
    assert len(common) >= 50
    worst = max(np.max(np.abs(mine[k].m - ref64[ref64[:, 0] == k][0, 2:5])) for k in common)
    assert worst <= 1e-4, worst
    worst32 = max(np.max(np.abs(mine[int(r[0])].m - r[2:5])) for r in ref32 if int(r[0]) in mine)
    assert worst32 <= 1e-4, worst32
    # the torque floor: same order as the reference's (rounding-noise dominated)
    tail = np.array([x.max_torque_deg_per_ns for x in log if x.step >= 100000])
    rtail = ref32[ref32[:, 0] >= 100000, 5]
    assert 0.2 * rtail.mean() <= tail.mean() <= 5 * rtail.mean(), (tail.mean(), rtail.mean())


@pytest.mark.parametrize("prec,window_ps", [(64, 200), (32, 80)])
def test_sp4_field1_window(prec, window_ps):
    p1, p0 = os.path.join(HERE, "sp4_field1.npz"), os.path.join(HERE, "sp4_relax.npz")
    if not (os.path.exists(p1) and os.path.exists(p0)):
        pytest.skip("fixture not generated")
    ref = np.load(p1)["samples"]              # step, mx, my, mz
    s = sim(prec, 0.02, (-24.6e-3 / MU0, 4.3e-3 / MU0, 0.0))
    s.set_m(np.load(p0)["s_state"])
    worst = 0.0
    for row in ref:
        step = int(row[0])
        if step * 5e-14 > window_ps * 1e-12 + 1e-18:
            break
        if step > 0:
            s.step(200)
        m = s.get_m().sum(axis=1) / (8e5 * 4096)
        worst = max(worst, float(np.max(np.abs(m - row[1:4]))))
    assert worst <= 1e-4, worst
