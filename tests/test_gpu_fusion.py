"""Fused next-step x pass (K5 also runs the following step's K1 inside a graph
chunk): a 64-step chunk must be bitwise identical to 64 single-step calls
(single-step chunks never fuse), in both precisions, with sampling on."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("prec", [32, 64])
@pytest.mark.parametrize("dims", [(32, 16, 4), (128, 32, 1), (20, 12, 3)])
def test_fused_chunk_equals_single_steps(prec, dims):
    import paper_1406_7459_b200 as E
    from oracle import oracle as O
    g = E.Grid(*dims, 3e-9, 3e-9, 3e-9)
    mat = E.Material(A=1.3e-11, Ku=4e4, Ms=8e5, alpha=0.1)
    f = E.FieldConfig(extern_field=(1e4, 0.0, 0.0))
    st = E.StepperConfig(dt=1e-14)
    m0 = O.random_unit_field(g.cell_count, 8e5, 11)
    a = E.Simulation(g, mat, f, st, precision=prec)
    b = E.Simulation(g, mat, f, st, precision=prec)
    a.set_m(m0)
    b.set_m(m0)
    ta = a.step(64, return_all=True)
    tb = [b.step(1) for _ in range(64)]
    assert np.array_equal(np.asarray(ta), np.asarray(tb))
    dt = np.float32 if prec == 32 else np.float64
    assert np.array_equal(a.get_m(dt), b.get_m(dt))
    assert np.array_equal(a.sample_now().m, b.sample_now().m)
