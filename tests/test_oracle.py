"""CPU tests pinning the oracle before it is trusted as the GPU checker.

* the 12 Maple Newell golden values (proj/tests/test_demag.cpp:26-44);
* tensor identities (acceptance.cpp:119-163; test_demag.cpp:46-120);
* the C restatement is bitwise equal to the reference itself (oracle/_ref) on
  fields, steps, energies (both precisions);
* FFT pipeline vs long-double direct sum (acceptance criterion 1);
* the committed golden fixtures (tests/golden, made by tests/golden/make_golden.py).
"""
import os

import numpy as np
import pytest

from oracle import oracle as O

MAPLE = [  # (fn, X, Y, Z, dx, dy, dz, value, tol) — test_demag.cpp:32-43
    ("xx", 0, 0, 0, 1, 1, 1, 1.0 / 3.0, 1e-12),
    ("xx", 0, 0, 0, 1, 1, 2, 0.40084192360558096752690050789034, 1e-12),
    ("xx", 0, 0, 0, 2, 1, 1, 0.19831615278883806494619898421931, 1e-12),
    ("xx", 0, 0, 0, 50, 10, 1, 0.021829576458713811627717362556500, 1e-12),
    ("xx", 1, 0, 0, 1, 1, 1, -0.13501718054449526838713434911401, 1e-12),
    ("xx", 0, 1, 0, 1, 1, 1, 0.067508590272247634193567174557006, 1e-12),
    ("xx", 1, 1, 1, 1, 2, 3, -0.056075776617493854142226134670956, 1e-12),
    ("xx", 10, 1, 1, 1, 2, 3, -0.00085675752896240944969766580856030, 1e-10),
    ("xy", 1, 1, 1, 1, 1, 1, -0.016062127810508233979724830686189, 1e-12),
    ("xy", 1, 1, 0, 1, 2, 3, -0.077258075615212400146921495217230, 1e-12),
    ("xy", 1, 2, 3, 1, 2, 3, -0.0088226536707711039322880437795490, 1e-12),
    ("xy", 10, 4, 6, 1, 2, 3, -0.00020004764005741154294387738750612, 1e-10),
]


@pytest.mark.parametrize("row", MAPLE)
@pytest.mark.parametrize("which", ["port", "ref"])
def test_maple_goldens(row, which):
    if which == "ref" and not O.ref_available():
        pytest.skip("oracle/_ref not built")
    fn, X, Y, Z, a, b, c, want, tol = row
    f = O.newell_nxx if fn == "xx" else O.newell_nxy
    got = f(X, Y, Z, a, b, c, which=which)
    assert abs(got - want) <= tol * abs(want)


def test_tensor_identities_port():
    for asp in [(1, 1, 1), (1, 1, 5), (2, 3, 4)]:
        e = O.tensor_entry(0, 0, 0, *(v * 1e-9 for v in asp))
        assert abs(e[0] + e[1] + e[2] + 1.0) <= 1e-12
    e = O.tensor_entry(0, 0, 0, 2e-9, 2e-9, 2e-9)
    assert np.all(np.abs(e[:3] + 1 / 3) <= 1e-12) and np.all(e[3:] == 0)
    # far displacement vs point dipole within 1% (test_demag.cpp:63-71)
    d = 3e-9
    e = O.tensor_entry(10, 0, 0, d, d, d)
    r = 10 * d
    dip = -(d ** 3 / (4 * np.pi)) * (r * r - 3 * r * r) / r ** 5
    assert abs(e[0] - dip) / abs(dip) <= 0.01 and dip > 0


def test_quad_truth_agrees_with_reference_near_field():
    if not O.quad_available():
        pytest.skip("quad oracle not built")
    for d in [(0, 0, 0), (1, 0, 0), (2, 1, 0), (3, 2, 1), (5, 5, 5)]:
        q = O.tensor_entry(*d, 3.90625e-9, 3.90625e-9, 3e-9, which="quad")
        p = O.tensor_entry(*d, 3.90625e-9, 3.90625e-9, 3e-9, which="port")
        assert np.all(np.abs(q - p) <= 1e-12 * np.max(np.abs(q)))


def _spec(g, **kw):
    nx, ny, nz, dx, dy, dz = g
    base = dict(A=1.3e-11, Ku=4e4, Ms=8e5, alpha=0.5, easy_axis=(0.6, 0.0, 0.8),
                h_ext=(2e4, -1e4, 3e4), dt=1e-14)
    base.update(kw)
    return O.Spec(nx, ny, nz, dx, dy, dz, **base)


@pytest.mark.parametrize("prec", [64, 32])
@pytest.mark.parametrize("g", [(5, 3, 2, 1e-9, 2e-9, 3e-9), (8, 8, 1, 2e-9, 2e-9, 2e-9),
                               (1, 1, 1, 2e-9, 2e-9, 2e-9), (7, 6, 5, 2e-9, 1e-9, 3e-9)])
def test_port_bitwise_equals_reference(g, prec):
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    s = _spec(g)
    m = O.random_unit_field(s.n, s.Ms, 1)
    r, p = O.Ref(s, prec), O.Port(s, prec)
    r.set_m(m)
    p.set_m(m)
    assert np.array_equal(r.hdemag(), p.hdemag())
    assert np.array_equal(r.heff(), p.heff())
    assert np.array_equal(r.step(5), p.step(5))
    assert np.array_equal(r.get_m(), p.get_m())
    assert np.array_equal(r.energies(), p.energies())


def test_port_pipeline_vs_direct_sum():
    """acceptance criterion 1 (f64 1e-11, f32 1e-3)."""
    for g in [(2, 2, 2, 2e-9, 2e-9, 2e-9), (4, 4, 4, 2e-9, 2e-9, 2e-9), (5, 3, 2, 1e-9, 2e-9, 3e-9),
              (8, 8, 1, 2e-9, 2e-9, 2e-9)]:
        s = _spec(g)
        m = O.random_unit_field(s.n, s.Ms, 42)
        direct = O.direct_demag(s, m, "port")
        for prec, tol in ((64, 1e-11), (32, 1e-3)):
            p = O.Port(s, prec)
            p.set_m(m)
            assert O.rel_linf(p.hdemag(), direct) <= tol


def test_nonfinite_raises_runtime_error():
    s = _spec((4, 4, 4, 2e-9, 2e-9, 2e-9), dt=1e-6, renorm_every=1000)
    p = O.Port(s, 64)
    p.set_m(O.random_unit_field(s.n, s.Ms, 3))
    with pytest.raises(RuntimeError, match="eulerUpdate"):
        for _ in range(200):
            p.step(1)


GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_golden_fixtures_reproduce():
    """The committed fixtures (generated from the reference) are reproduced by the port."""
    path = os.path.join(GOLDEN, "fields_small.npz")
    if not os.path.exists(path):
        pytest.skip("fixtures not generated")
    z = np.load(path, allow_pickle=False)
    for key in z.files:
        if not key.endswith("_spec"):
            continue
        name = key[:-5]
        vals = z[key]
        g = tuple(vals[:6])
        prec = int(vals[6])
        s = _spec((int(g[0]), int(g[1]), int(g[2]), g[3], g[4], g[5]))
        p = O.Port(s, prec)
        p.set_m(z[name + "_m"])
        assert np.array_equal(p.hdemag(), z[name + "_hdemag"]), name
        assert np.array_equal(p.heff(), z[name + "_heff"]), name
