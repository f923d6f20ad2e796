"""Multi-GPU z-slab decomposition, exercised on one B200 with virtual ranks
(mfd_exec.virtual_ranks = 1): every rank is a full engine with its own slab,
halo planes, blocked spectra and tensor block, and the group moves exactly the
blocks the NCCL transport moves.  The per-column FFT arithmetic is unchanged
by the decomposition, so fields and trajectories must equal the one-rank
engine bitwise; only the sample sums reassociate."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

MS = 8e5


def make(g, prec, world, **kw):
    import paper_1406_7459_b200 as E
    nx, ny, nz, dx, dy, dz = g
    base = dict(A=1.3e-11, Ku=4e4, Ms=MS, alpha=0.5, easy_axis=(0.6, 0.0, 0.8))
    base.update({k: v for k, v in kw.items() if k in base})
    fields = E.FieldConfig(kw.get("exchange", True), True, kw.get("demag", True), True, (2e4, -1e4, 3e4))
    st = E.StepperConfig(dt=kw.get("dt", 1e-14), max_steps=kw.get("max_steps", 500000),
                         torque_tol_deg_per_ns=kw.get("torque_tol", 0.01), sample_every=kw.get("sample_every", 100))
    return E.Simulation(E.Grid(nx, ny, nz, dx, dy, dz), E.Material(**base), fields, st, precision=prec,
                        world=world, virtual_ranks=world > 1)


GRIDS = [(16, 12, 8, 2e-9, 2e-9, 2e-9), (33, 17, 4, 2e-9, 3e-9, 2e-9), (64, 32, 16, 2e-9, 2e-9, 2e-9),
         (4, 512, 4, 1e-9, 1e-9, 1e-9),     # Py = 1024: two-stage TMA y passes (f32), three-stage (f64)
         (4, 1024, 4, 1e-9, 1e-9, 1e-9),    # Py = 2048: three-stage TMA y passes
         (4, 4, 128, 2e-9, 2e-9, 1e-9)]     # Pz = 256: K3 radix 32 x 8


@pytest.mark.parametrize("prec", [64, 32])
@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("g", GRIDS)
def test_virtual_ranks_match_single_rank(g, world, prec):
    if g[2] % world:
        pytest.skip("nz not divisible")
    m = O.random_unit_field(g[0] * g[1] * g[2], MS, 23)
    one, many = make(g, prec, 1), make(g, prec, world)
    one.set_m(m)
    many.set_m(m)
    assert np.array_equal(many.get_m(), one.get_m())
    assert np.array_equal(many.demag_field(), one.demag_field())
    assert np.array_equal(many.effective_field(), one.effective_field())
    assert np.array_equal(many.step(6, return_all=True), one.step(6, return_all=True))
    assert np.array_equal(many.get_m(), one.get_m())
    assert many.time() == one.time()
    a, b = many.sample_now(), one.sample_now()
    assert np.allclose(a.m, b.m, rtol=0, atol=1e-13)
    assert abs(a.e_total - b.e_total) <= 1e-12 * abs(b.e_total)


@pytest.mark.parametrize("world", [2, 4])
def test_virtual_ranks_demag_off_halo(world):
    """demag off: only the one-plane halo crosses ranks (exchange stencil)."""
    g = (20, 10, 8, 2e-9, 2e-9, 2e-9)
    m = O.random_unit_field(g[0] * g[1] * g[2], MS, 29)
    one, many = make(g, 64, 1, demag=False), make(g, 64, world, demag=False)
    one.set_m(m)
    many.set_m(m)
    assert np.array_equal(many.effective_field(), one.effective_field())
    assert np.array_equal(many.step(4, return_all=True), one.step(4, return_all=True))
    assert np.array_equal(many.get_m(), one.get_m())


def test_virtual_ranks_relax_matches_reference():
    g = (8, 8, 4, 5e-9, 5e-9, 5e-9)
    spec = O.Spec(*g, A=1.3e-11, Ku=4e4, Ms=MS, alpha=1.0, easy_axis=(0.6, 0.0, 0.8), h_ext=(2e4, -1e4, 3e4),
                  dt=1e-13, torque_tol=50.0, max_steps=3000, sample_every=50)
    m = O.random_unit_field(spec.n, MS, 31)
    many = make(g, 64, 2, alpha=1.0, dt=1e-13, torque_tol=50.0, max_steps=3000, sample_every=50)
    many.set_m(m)
    conv, log = many.relax()
    if not O.ref_available():
        pytest.skip("reference .so not built")
    ref = O.Ref(spec, 64)
    ref.set_m(m)
    rconv, rlog = ref.relax()
    assert conv == rconv and [s.step for s in log] == [s.step for s in rlog]
    assert O.rel_linf(many.get_m(), ref.get_m()) <= 1e-9


def test_uneven_slab_rejected():
    with pytest.raises(ValueError, match="divisible"):
        make((8, 8, 6, 2e-9, 2e-9, 2e-9), 64, 4)
