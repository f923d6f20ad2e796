"""GPU parity of the B200 engine against the CPU oracle (the reference's own
code, oracle/_ref, or its bitwise-equal C restatement, oracle/build).

Tolerances (BASELINE.json north_star):
  * H_demag / H_eff: rel L-inf <= 1e-5 in f32; <= 1e-10 in f64 where the
    reference tensor is itself accurate (small grids), and <= 1e-11 for the
    FFT pipeline alone when the reference's tensor is injected (any grid).
  * demag-free local path: bitwise in f32 and f64 (no FMA, reference order).
  * device tensor vs the __float128 truth: <= 5e-12 relative per entry.
"""
import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import checker, engine_sim, pair

pytestmark = pytest.mark.gpu

MS = 8e5

# acceptance.cpp:65-71 grid set + degenerate and odd shapes
SMALL_GRIDS = [
    (2, 2, 2, 2e-9, 2e-9, 2e-9), (4, 4, 4, 2e-9, 2e-9, 2e-9), (5, 3, 2, 1e-9, 2e-9, 3e-9),
    (8, 8, 1, 2e-9, 2e-9, 2e-9), (8, 8, 8, 2e-9, 2e-9, 2e-9), (3, 3, 1, 2e-9, 2e-9, 2e-9),
    (1, 1, 1, 2e-9, 2e-9, 2e-9), (1, 1, 4, 2e-9, 2e-9, 1e-9), (7, 1, 1, 1e-9, 1e-9, 1e-9),
    (16, 8, 4, 3e-9, 2e-9, 1e-9), (33, 17, 5, 2e-9, 2e-9, 3e-9),
]
# every FFT length of every pass, incl. the 3-stage plans
SIZE_GRIDS = [
    (128, 32, 1, 3.90625e-9, 3.90625e-9, 3e-9),     # SP4 C1
    (512, 4, 2, 1e-9, 1e-9, 1e-9), (1024, 2, 1, 1e-9, 1e-9, 1e-9), (2048, 2, 1, 1e-9, 1e-9, 1e-9),
    (4, 512, 2, 1e-9, 1e-9, 1e-9), (2, 1024, 1, 1e-9, 1e-9, 1e-9),
    (2, 2, 256, 1e-9, 1e-9, 1e-9), (2, 3, 1024, 1e-9, 1e-9, 1e-9),
    (64, 48, 40, 2e-9, 2e-9, 2e-9), (200, 100, 3, 2e-9, 2e-9, 2e-9),
    (20, 12, 100, 2e-9, 2e-9, 1e-9),                # Pz = 256 with nz < Pz/2 (K3 non-FZ, radix 32 x 8)
    (3, 768, 1, 1e-9, 1e-9, 1e-9),                  # Py = 2048 with ny < Py/2 (three-stage TMA K2, FY=0)
    (6, 200, 2, 1e-9, 1e-9, 1e-9),                  # Py = 512: TMA y passes, three-stage in f64
]


def spec_of(g, **kw):
    nx, ny, nz, dx, dy, dz = g
    base = dict(A=1.3e-11, Ku=4e4, Ms=MS, alpha=0.5, easy_axis=(0.6, 0.0, 0.8),
                h_ext=(2e4, -1e4, 3e4), dt=1e-14)
    base.update(kw)
    return O.Spec(nx, ny, nz, dx, dy, dz, **base)


# ------------------------------------------------------------------ tensor
@pytest.mark.parametrize("g", [(8, 8, 8, 2e-9, 2e-9, 2e-9), (128, 32, 1, 3.90625e-9, 3.90625e-9, 3e-9),
                               (40, 20, 8, 0.9765625e-9, 0.9765625e-9, 0.75e-9),
                               (24, 24, 24, 3.90625e-9, 3.90625e-9, 3.90625e-9),
                               (5, 3, 2, 1e-9, 2e-9, 3e-9), (300, 2, 2, 1e-9, 1e-9, 1e-9)])
def test_device_tensor_vs_quad_truth(g):
    if not O.quad_available():
        pytest.skip("quad oracle not built")
    s = spec_of(g)
    sim = engine_sim(s, 64)
    dev = sim.demag_octant()
    truth = O.tensor_octant(*g, which="quad")
    # per entry: 1e-10 relative, or 5e-13 of the component's largest entry for the
    # entries that nearly vanish by symmetry (where fp64 Newell cancels absolutely)
    for c in range(6):
        scale = np.max(np.abs(truth[c]))
        if scale == 0:
            assert np.all(dev[c] == 0)
            continue
        err = np.abs(dev[c] - truth[c])
        rel = err / np.maximum(np.abs(truth[c]), 1e-300)
        bad = (err > 1e-10 * np.abs(truth[c])) & (err > 5e-13 * scale)
        assert not bad.any(), (c, float(rel[bad].max()), np.argwhere(bad)[:3])


def test_tensor_self_identities():
    """acceptance.cpp:120-135: trace -1, cubic -1/3 (device tensor)."""
    for asp in [(1, 1, 1), (1, 1, 5), (2, 3, 4)]:
        s = spec_of((1, 1, 1, asp[0] * 1e-9, asp[1] * 1e-9, asp[2] * 1e-9))
        o = engine_sim(s, 64).demag_octant()[:, 0, 0, 0]
        assert abs(o[0] + o[1] + o[2] + 1.0) <= 1e-12
        if asp == (1, 1, 1):
            assert np.all(np.abs(o[:3] + 1 / 3) <= 1e-12) and np.all(o[3:] == 0)


# --------------------------------------------------------------- spectrum
@pytest.mark.parametrize("g", [(5, 3, 2, 1e-9, 2e-9, 3e-9), (8, 4, 1, 2e-9, 2e-9, 2e-9),
                               (6, 6, 6, 2e-9, 2e-9, 2e-9), (33, 17, 5, 2e-9, 2e-9, 3e-9)])
def test_spectrum_octant_vs_reference(g):
    if not O.ref_available():
        pytest.skip("reference .so not built")
    s = spec_of(g)
    sim = engine_sim(s, 64)
    sim.set_demag_octant(O.tensor_octant(*g, which="ref"))
    mine = sim.spectrum_octant()                         # [6][v][w][u]
    ref, max_imag = O.ref_spectrum_octant(*g)            # [6][w][v][u]
    ref = np.transpose(ref, (0, 2, 1, 3))
    for c in range(6):
        assert O.rel_linf(mine[c], ref[c]) <= 1e-12, c
    assert max_imag <= 1e-12 * np.max(np.abs(ref))       # E6: spectra are real


# ---------------------------------------------------------------- H_demag
@pytest.mark.parametrize("g", SMALL_GRIDS)
@pytest.mark.parametrize("prec", [64, 32])
def test_demag_field_small(g, prec):
    s = spec_of(g)
    sim, ref, m = pair(s, prec)
    tol = 1e-10 if prec == 64 else 1e-5
    assert O.rel_linf(sim.demag_field(), ref.hdemag()) <= tol


@pytest.mark.parametrize("g", SIZE_GRIDS)
def test_demag_fft_pipeline_with_reference_tensor(g):
    """FFT machinery at every pass length, isolated from tensor accuracy."""
    if not O.ref_available():
        pytest.skip("reference .so not built")
    s = spec_of(g)
    sim, ref, m = pair(s, 64, seed=7)
    sim.set_demag_octant(O.tensor_octant(*g, which="ref"))
    assert O.rel_linf(sim.demag_field(), ref.hdemag()) <= 1e-11


@pytest.mark.parametrize("g", SIZE_GRIDS)
def test_demag_field_f32_sizes(g):
    s = spec_of(g)
    sim, ref, m = pair(s, 32, seed=8)
    assert O.rel_linf(sim.demag_field(), ref.hdemag()) <= 1e-5


def test_demag_matches_direct_sum():
    """acceptance criterion 1 against the long-double direct sum."""
    for g in [(2, 2, 2, 2e-9, 2e-9, 2e-9), (4, 4, 4, 2e-9, 2e-9, 2e-9), (5, 3, 2, 1e-9, 2e-9, 3e-9),
              (8, 8, 1, 2e-9, 2e-9, 2e-9), (8, 8, 8, 2e-9, 2e-9, 2e-9)]:
        s = spec_of(g)
        m = O.random_unit_field(s.n, MS, 42)
        direct = O.direct_demag(s, m, "port")
        sim = engine_sim(s, 64)
        sim.set_m(m)
        assert O.rel_linf(sim.demag_field(), direct) <= 1e-11
        sim32 = engine_sim(s, 32)
        sim32.set_m(m)
        assert O.rel_linf(sim32.demag_field(), direct) <= 1e-3


def test_uniform_cube_demag_factor():
    """acceptance criterion 4: <Hz> = -Ms/3 for a uniform 8^3 cube."""
    s = spec_of((8, 8, 8, 2e-9, 2e-9, 2e-9))
    sim = engine_sim(s, 64)
    sim.set_m(np.stack([np.zeros(s.n), np.zeros(s.n), np.full(s.n, MS)]))
    h = sim.demag_field()
    assert abs(h[2].mean() + MS / 3) / (MS / 3) <= 1e-9


def test_demag_disabled_raises_logic_error():
    s = spec_of((4, 4, 4, 2e-9, 2e-9, 2e-9), demag=False)
    sim = engine_sim(s, 64)
    with pytest.raises(LookupError, match="lastDemagField: demag term is disabled"):
        sim.demag_field()


# ---------------------------------------------------------------- H_eff
@pytest.mark.parametrize("g", SMALL_GRIDS + SIZE_GRIDS[:2])
@pytest.mark.parametrize("prec", [64, 32])
def test_effective_field(g, prec):
    s = spec_of(g)
    sim, ref, m = pair(s, prec, seed=3)
    tol = 1e-10 if prec == 64 else 1e-5
    if prec == 64 and max(g[:3]) >= 100:
        tol = 1e-9   # reference long-double tensor error at >= 100 cells
    assert O.rel_linf(sim.effective_field(), ref.heff()) <= tol


@pytest.mark.parametrize("prec", [64, 32])
@pytest.mark.parametrize("g", [(8, 8, 8, 5e-9, 5e-9, 5e-9), (33, 17, 5, 2e-9, 2e-9, 3e-9),
                               (1, 1, 1, 2e-9, 2e-9, 2e-9), (128, 32, 1, 3.90625e-9, 3.90625e-9, 3e-9)])
def test_local_path_bitwise(g, prec):
    """terms.demag = false: H_eff, torque and Euler steps bitwise equal to the reference."""
    s = spec_of(g, demag=False)
    sim, ref, m = pair(s, prec, seed=5)
    assert np.array_equal(sim.effective_field(), ref.heff())
    t_mine = sim.step(7, return_all=True)
    t_ref = ref.step(7)
    assert np.array_equal(t_mine, t_ref)
    assert np.array_equal(sim.get_m(), ref.get_m())
    assert sim.time() == ref.time()


def test_renorm_every_cadence_bitwise():
    """renormalise iff (step+1) % k == 0 (sim.hpp:38), k = 3, starting mid-count."""
    s = spec_of((6, 5, 4, 2e-9, 2e-9, 2e-9), demag=False, renorm_every=3, dt=2e-14)
    sim, ref, m = pair(s, 64, seed=9)
    sim.set_time(1e-12, 4)
    ref.set_time(1e-12, 4)
    assert np.array_equal(sim.step(8, return_all=True), ref.step(8))
    assert np.array_equal(sim.get_m(), ref.get_m())


# ------------------------------------------------------------- dynamics
@pytest.mark.parametrize("prec", [64, 32])
@pytest.mark.parametrize("g", [(8, 8, 8, 5e-9, 5e-9, 5e-9), (16, 8, 4, 3e-9, 2e-9, 1e-9),
                               (128, 32, 1, 3.90625e-9, 3.90625e-9, 3e-9)])
def test_steps_with_demag(g, prec):
    s = spec_of(g, alpha=0.02, dt=5e-14)
    sim, ref, m = pair(s, prec, seed=11)
    t_mine = sim.step(20, return_all=True)
    t_ref = ref.step(20)
    tol = 1e-9 if prec == 64 else 2e-5
    assert np.max(np.abs(t_mine - t_ref) / np.abs(t_ref)) <= tol
    assert O.rel_linf(sim.get_m(), ref.get_m()) <= tol
    assert sim.time() == ref.time()


def test_sample_and_energies():
    s = spec_of((8, 8, 8, 5e-9, 5e-9, 5e-9))
    sim, ref, m = pair(s, 64, seed=13)
    e_ref = ref.energies()
    smp = sim.sample_now()
    got = np.array([smp.e_exchange, smp.e_anisotropy, smp.e_demag, smp.e_zeeman, smp.e_total])
    assert np.allclose(got, e_ref, rtol=1e-10, atol=0)
    m_ref = m.sum(axis=1) / (MS * s.n)
    assert np.allclose(smp.m, m_ref, rtol=0, atol=1e-14)


def test_relax_stops_at_reference_step():
    """dynamics::relax: same converged flag, stop step, samples (acceptance 10 analogue)."""
    if not O.ref_available():
        pytest.skip("reference .so not built")
    s = spec_of((8, 8, 2, 5e-9, 5e-9, 5e-9), alpha=1.0, dt=1e-13, torque_tol=50.0,
                max_steps=5000, sample_every=50, h_ext=(0, 0, 0), zeeman=False)
    sim, ref, m = pair(s, 64, seed=17)
    conv, log = sim.relax()
    rconv, rlog = ref.relax()
    assert conv == rconv
    assert [x.step for x in log] == [x.step for x in rlog]
    for a, b in zip(log, rlog):
        assert abs(a.t - b.t) == 0
        assert np.max(np.abs(a.m - np.array(b.m[:]))) <= 1e-9
        assert abs(a.max_torque_deg_per_ns - b.torque) <= 1e-8 * b.torque
        assert abs(a.e_total - b.e_total) <= 1e-9 * abs(b.e_total)
    assert O.rel_linf(sim.get_m(), ref.get_m()) <= 1e-9


def test_relax_exhausts_max_steps():
    if not O.ref_available():
        pytest.skip("reference .so not built")
    s = spec_of((4, 4, 4, 5e-9, 5e-9, 5e-9), alpha=1.0, dt=1e-13, torque_tol=1e-12,
                max_steps=300, sample_every=100)
    sim, ref, m = pair(s, 64, seed=19)
    conv, log = sim.relax()
    rconv, rlog = ref.relax()
    assert (conv, [x.step for x in log]) == (rconv, [x.step for x in rlog])
    assert sim.time()[1] == 300


def test_nonfinite_update_raises_runtime_error():
    s = spec_of((4, 4, 4, 2e-9, 2e-9, 2e-9), dt=1e-6, renorm_every=1000)
    sim, ref, m = pair(s, 64, seed=21)
    with pytest.raises(RuntimeError, match="eulerUpdate: non-finite magnetization"):
        for _ in range(200):
            sim.step(1)
    t, step = sim.time()
    assert np.all(np.isfinite(sim.get_m()))


def test_set_get_roundtrip_and_uniform():
    s = spec_of((5, 3, 2, 1e-9, 2e-9, 3e-9))
    sim = engine_sim(s, 64)
    m = O.random_unit_field(s.n, MS, 1)
    sim.set_m(m)
    assert np.array_equal(sim.get_m(), m)
    import paper_1406_7459_b200 as E
    g = E.Grid(4, 4, 4, 1e-9, 1e-9, 1e-9)
    u = E.Simulation(g, E.Material(Ms=MS), init_direction=(0.6, 0.0, 0.8))
    mm = u.get_m()
    assert np.all(mm[0] == MS * 0.6) and np.all(mm[2] == MS * 0.8)


def test_step_async_error_rolls_back_clock():
    """A non-finite update inside an asynchronous chunk: sync() raises the reference's
    runtime_error and t / step stop at the last completed step (dynamics.hpp:115-120),
    across several 64-step graph chunks."""
    s = spec_of((4, 4, 4, 2e-9, 2e-9, 2e-9), dt=2e-12, renorm_every=100000)
    # |M| grows under Euler without renormalisation; from 3% of Ms it overflows at
    # step 97 of the reference, i.e. inside the second 64-step graph chunk
    m0 = 0.03 * np.full((3, s.n), MS / 3 ** 0.5)
    sim, ref, m = pair(s, 64, m=m0)
    n_ok = 0
    with pytest.raises(RuntimeError):
        for _ in range(400):
            ref.step(1)
            n_ok += 1
    sim.step_async(400)
    with pytest.raises(RuntimeError, match="eulerUpdate: non-finite magnetization"):
        sim.sync()
    assert sim.time() == ref.time()
    assert sim.time()[1] == n_ok
    assert np.all(np.isfinite(sim.get_m()))
    sim.sync()   # error consumed


@pytest.mark.parametrize("prec", [64, 32])
def test_staged_upload_pipeline_equals_serial(prec):
    """mfd_stage_m (overlapped H2D on a copy stream) + step_async + sync_torque gives
    bitwise the states and torques of set_m + step; staging twice installs the last."""
    s = spec_of((33, 17, 5, 2e-9, 2e-9, 3e-9), alpha=0.1)
    dt = np.float32 if prec == 32 else np.float64
    ins = [O.random_unit_field(s.n, MS, 40 + i).astype(dt) for i in range(4)]
    a, b = engine_sim(s, prec), engine_sim(s, prec)
    ta, tb = [], []
    for m in ins:
        a.set_m(m)
        ta.append(a.step(1))
    b.stage_m(ins[0])
    for i in range(len(ins)):
        b.step_async(1)
        if i + 1 < len(ins):
            b.stage_m(ins[i + 1])
        tb.append(b.sync_torque())
    assert ta == tb
    assert np.array_equal(a.get_m(dt), b.get_m(dt))
    b.stage_m(ins[1])
    b.stage_m(ins[2])                       # the later staged state wins
    assert np.array_equal(b.get_m(dt), ins[2])


def test_set_stepper_equals_fresh_context():
    """mfd_set_stepper on a live context (captured graphs dropped) == a context built with it."""
    import paper_1406_7459_b200 as E
    s1 = spec_of((16, 8, 4, 3e-9, 2e-9, 1e-9), dt=1e-14)
    s2 = spec_of((16, 8, 4, 3e-9, 2e-9, 1e-9), dt=3e-14, renorm_every=2)
    m = O.random_unit_field(s1.n, MS, 51)
    a, b = engine_sim(s1, 64), engine_sim(s2, 64)
    a.set_m(m)
    b.set_m(m)
    a.step(5)
    a.set_stepper(E.StepperConfig(dt=3e-14, renormalize_every=2))
    a.set_time(0.0, 0)
    a.set_m(m)
    assert np.array_equal(a.step(9, return_all=True), b.step(9, return_all=True))
    assert np.array_equal(a.get_m(), b.get_m())
    with pytest.raises(ValueError, match="dt must be > 0"):
        a.set_stepper(E.StepperConfig(dt=0.0))


@pytest.mark.parametrize("prec", [64, 32])
def test_f32_field_readouts(prec):
    s = spec_of((33, 17, 5, 2e-9, 2e-9, 3e-9))
    sim, ref, m = pair(s, prec, seed=52)
    h64, h32 = sim.effective_field(), sim.effective_field(dtype=np.float32)
    assert h32.dtype == np.float32 and np.array_equal(h32, h64.astype(np.float32))
    assert np.array_equal(sim.demag_field(dtype=np.float32), sim.demag_field().astype(np.float32))


def test_prepare_async_captures_the_timed_graphs():
    s = spec_of((64, 32, 8, 2e-9, 2e-9, 2e-9))
    a, b = engine_sim(s, 32), engine_sim(s, 32)
    m = O.random_unit_field(s.n, MS, 53)
    a.set_m(m)
    b.set_m(m)
    launches = a.prepare_async(150)   # chunks of 64 + 64 + 22
    assert launches >= 3 * 4
    a.step_async(150)
    a.sync()
    b.step(150)
    assert np.array_equal(a.get_m(), b.get_m())
