"""CPU tests of the drop-in boundary: libmagfd_b200.so loads, exports every
symbol include/mfd.h declares, validates arguments with the reference's
exception messages before touching a device, and refuses to run without an
sm_100 GPU (there is no CPU fallback)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mfd.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mfd_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ["mfd_create", "mfd_destroy", "mfd_step", "mfd_relax", "mfd_effective_field_f64",
              "mfd_demag_field_f64", "mfd_set_m_f64", "mfd_get_m_f64", "mfd_sample_now",
              "mfd_last_error"]:
        assert s in syms


def test_library_exports_every_declared_symbol():
    import paper_1406_7459_b200 as E
    lib = E.load_library()
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert b"sm_100a" in lib.mfd_version()


def _mk(**over):
    import paper_1406_7459_b200 as E
    g = dict(nx=4, ny=4, nz=4, dx=1e-9, dy=1e-9, dz=1e-9)
    m = dict(A=1.3e-11, Ku=0.0, Ms=8e5, alpha=0.5)
    s = dict(dt=1e-14)
    for k, v in over.items():
        (g if k in g else m if k in m or k in ("gamma", "easy_axis") else s)[k] = v
    return E.Simulation(E.Grid(**g), E.Material(**m), stepper=E.StepperConfig(
        dt=s.get("dt", 1e-14), renormalize_every=s.get("renormalize_every", 1),
        torque_tol_deg_per_ns=s.get("torque_tol_deg_per_ns", 0.01)))


@pytest.mark.parametrize("over,msg", [
    (dict(nx=0), "Grid: cell counts must be >= 1"),
    (dict(dz=0.0), "Grid: cell sizes must be > 0"),
    (dict(Ms=0.0), "MaterialParams: Ms must be > 0"),
    (dict(A=-1.0), "MaterialParams: A must be >= 0"),
    (dict(alpha=-0.1), "MaterialParams: alpha must be >= 0"),
    (dict(gamma=0.0), "MaterialParams: gamma must be > 0"),
    (dict(easy_axis=(1.0, 1.0, 0.0)), "MaterialParams: easyAxis must be a unit vector"),
    (dict(dt=0.0), "StepperConfig: dt must be > 0"),
    (dict(renormalize_every=0), "StepperConfig: renormalizeEvery must be >= 1"),
    (dict(torque_tol_deg_per_ns=0.0), "StepperConfig: torque tolerance must be > 0"),
])
def test_validation_matches_reference_messages(over, msg):
    with pytest.raises(ValueError, match=re.escape(msg)):
        _mk(**over)


def test_no_cpu_fallback():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    with pytest.raises(OSError, match="no CUDA device"):
        _mk()


def test_stability_limit_matches_reference_formula():
    import paper_1406_7459_b200 as E
    g = E.Grid(4, 4, 4, 3.90625e-9, 3.90625e-9, 3e-9)
    m = E.Material(A=1.3e-11, Ms=8e5, alpha=0.02)
    want = (1 + 0.02 ** 2) * 8e5 * 3e-9 ** 2 / (E.GAMMA_E * 4 * 1.3e-11 * 10)
    assert abs(E.Simulation.stability_dt_limit(g, m) - want) <= 1e-15 * want
